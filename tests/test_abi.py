"""The C-ABI library loads and exports every symbol include/gazemap_b200.h
declares; without a GPU every compute entry point fails loudly (no CPU
fallback).  CPU-only."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "gazemap_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gm_[a-z0-9_]+)\s*\(", text)) - {"gm_progress_fn"})


def test_library_exports_every_declared_symbol():
    from paper_2601_07571_b200 import _native

    lib = _native.load()
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes signature table covers the header
    assert set(names) <= set(_native.SIGNATURES), set(names) - set(_native.SIGNATURES)


def test_symbols_visible_with_nm():
    import subprocess

    from paper_2601_07571_b200 import _native

    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.SO_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gm_\w+)", out))
    assert set(_declared()) <= exported


def test_sm100a_code_present():
    import subprocess

    from paper_2601_07571_b200 import _native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.SO_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    from paper_2601_07571_b200 import _native
    import paper_2601_07571_b200 as gm

    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    mesh = gm.Mesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    with pytest.raises(_native.NativeUnavailableError):
        gm.build_sampled_mesh(mesh, 100.0)
    scene = gm.Scene((gm.SceneObject("t", mesh),))
    sm = {"t": gm.SampledMesh("t", np.ones(1, np.int64), np.full(1, 3, np.int64), np.zeros(1, np.int64), 3, 1.0)}
    with pytest.raises(_native.NativeUnavailableError):
        gm.generate(scene, sm, [], gm.GenerationConfig(k=1.0))


def test_last_error_is_a_string():
    from paper_2601_07571_b200 import _native

    lib = _native.load()
    assert isinstance(lib.gm_last_error(), bytes)
    assert lib.gm_abi_version() == 1
