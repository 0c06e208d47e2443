"""Self-check run: a whole fixation stream through the GM_CHECK build of the
extension (every float32-bound / conservative-cull decision re-done in exact
float64 and compared on the device, gm_plan_check), one JSON line out.

    GAZEMAP_B200_SO=paper_2601_07571_b200/_gazemap_b200_check.so \
        python tools/check_run.py --config c2 [--fixations N] [--start S] [--unfiltered]

Counters (GM_CHK_*, csrc/gm_kernels.cu): texels / candidate pairs / depth tests
checked, and the "wrong" counts -- decisions the exact reference arithmetic
contradicts.  A clean run has every *_wrong counter at 0.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3k30", "c3k100", "c4", "c5"])
    ap.add_argument("--fixations", type=int, default=0)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--unfiltered", action="store_true")
    ap.add_argument("--chunk", type=int, default=8192, help="fixations per generate call")
    ap.add_argument("--any-build", action="store_true",
                    help="run on the production build too (no counters; e.g. under compute-sanitizer)")
    a = ap.parse_args()

    import bench
    import paper_2601_07571_b200 as gm
    from paper_2601_07571_b200 import _native, density

    scene, k, fx, filtering, desc = bench.workload(a.config, 0, 0)
    if a.unfiltered:
        filtering = False
    fx = fx[a.start:]
    if a.fixations:
        fx = fx[:a.fixations]
    cfg = gm.GenerationConfig(k=k, filtering_enabled=filtering)
    sampled = gm.build_sampled_meshes(scene, k)
    plan = density.get_plan(scene, sampled, cfg, 0)
    lib = _native.load()
    out = (ctypes.c_uint64 * len(_native.CHECK_NAMES))()
    is_check = ctypes.c_int(0)
    _native.check(lib.gm_plan_check(plan._h, out, 1, ctypes.byref(is_check)))
    if not is_check.value and not a.any_build:
        raise SystemExit("not a GM_CHECK build: set GAZEMAP_B200_SO to the _gazemap_b200_check.so variant")
    t0 = time.perf_counter()
    for c0 in range(0, len(fx), a.chunk):
        plan.accumulate(fx[c0:c0 + a.chunk], cfg, reset=(c0 == 0))
    plan.sync()
    dt = time.perf_counter() - t0
    _native.check(lib.gm_plan_check(plan._h, out, 0, ctypes.byref(is_check)))
    counts = {n: int(v) for n, v in zip(_native.CHECK_NAMES, out) if not n.startswith("reserved")}
    vals = plan.read()
    wrong = sum(v for n, v in counts.items() if n.endswith("_wrong"))
    print(json.dumps({"config": a.config, "workload": desc, "filtering": filtering, "start": a.start,
                      "fixations": int(len(fx)), "samples": int(plan.n_samples), "seconds": round(dt, 1),
                      "library": os.environ.get("GAZEMAP_B200_SO", "default"), "check_build": bool(is_check.value),
                      "max": float(vals.max()) if len(vals) else 0.0, "sum": float(vals.sum()),
                      "nonzero": int((vals != 0).sum()), "counters": counts,
                      "violations": wrong, "clean": wrong == 0}), flush=True)
    return 0 if wrong == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
