"""Build the in-tree CUDA extension `_gazemap_b200.so` (sm_100a).

    python -m paper_2601_07571_b200.build [-v]

nvcc compiles the kernels for `-gencode arch=compute_100a,code=sm_100a` with
`-fmad=false` (the reference's numba kernels contain no FMA; the explicit
__fma_rn BLAS chains are unaffected).  The host fixation setup is plain g++
with -ffp-contract=off -fno-builtin (see gm_setup.cpp for why).  The result
is written next to this file so it travels with the repository snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
SO = PKG / "_gazemap_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _tool(name: str, fallback: str) -> str:
    for cand in (f"/usr/bin/{name}", shutil.which(name) or "", fallback):
        if cand and os.path.exists(cand):
            return cand
    return name


def _nvcc() -> str:
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    p = Path(cuda) / "bin" / "nvcc"
    return str(p) if p.exists() else "nvcc"


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp")) + sorted(CSRC.glob("*.h")) + sorted(
        CSRC.glob("*.cuh"))


def needs_build() -> bool:
    if not SO.exists():
        return True
    t = SO.stat().st_mtime
    return any(s.stat().st_mtime > t for s in _sources()) or Path(__file__).stat().st_mtime > t


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """Compile the extension; `defines`/`out` build an experimental variant
    (e.g. defines=["-DKS_MINB=4"], out=PKG / "_variant.so") without touching
    the production library."""
    so = Path(out) if out else SO
    if not force and not defines and out is None and not needs_build():
        return SO
    build_dir = BUILD if out is None else BUILD / so.stem
    build_dir.mkdir(parents=True, exist_ok=True)
    gxx = _tool("g++", "g++")
    nvcc = _nvcc()
    objs = []
    cmds = []
    for cu in sorted(CSRC.glob("*.cu")):
        obj = build_dir / (cu.stem + ".o")
        cmds.append([nvcc, "-c", str(cu), "-o", str(obj), *ARCH, "-O3", "-std=c++17", "-lineinfo", "-fmad=false",
                     "-Xptxas", "-v", "-ccbin", gxx, "-Xcompiler", "-fPIC", "-I", str(CSRC), *defines])
        objs.append(obj)
    for cpp in sorted(CSRC.glob("*.cpp")):
        obj = build_dir / (cpp.stem + ".o")
        cmds.append([gxx, "-c", str(cpp), "-o", str(obj), "-O2", "-std=c++17", "-fPIC", "-fopenmp",
                     "-ffp-contract=off", "-fno-fast-math", "-fno-builtin", "-I", str(CSRC)])
        objs.append(obj)
    tmp = so.with_suffix(".so.tmp")
    cmds.append([nvcc, "-shared", *ARCH, "-o", str(tmp), *map(str, objs), "-ccbin", gxx, "-Xcompiler", "-fopenmp",
                 "-lgomp"])
    for c in cmds:
        r = subprocess.run(c, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(" ".join(c) + "\n" + r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"build failed: {' '.join(c[:3])} ...")
        if "-Xptxas" in c:
            (build_dir / (Path(c[2]).stem + ".ptxas.txt")).write_text(r.stderr)
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv))
