"""accumulate_fixation loop vs one batched generate.

    python tools/accum_loop_bench.py [--fixations 1000]

Loops `accumulate_fixation` over the first F fixations of the C2 stream (the
map stays on the GPU between calls; one scalar max per call), reads the map
once at the end, and compares with one `generate` of the same fixations:
wall times, the ratio, and bitwise equality of the two maps.  One JSON line.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fixations", type=int, default=1000)
    a = ap.parse_args()
    import paper_2601_07571_b200 as gm
    import workloads as W

    scene = W.room_scene()
    k = 10_000.0
    table = W.room_fixations(a.fixations, seed=1, scene=scene)
    fx = [gm.Fixation(r[0], r[1], r[2:5], r[5:9], tuple(r[9:15]), r[15:18]) for r in table]
    cfg = gm.GenerationConfig(k=k)
    sampled = gm.build_sampled_meshes(scene, k)
    gm.generate(scene, sampled, fx, cfg)  # plan upload + batch buffers sized for this batch, warm-up
    t0 = time.perf_counter()
    full = gm.generate(scene, sampled, fx, cfg)
    t_gen = time.perf_counter() - t0
    dm = gm.DensityMap.zeros(sampled)
    gm.accumulate_fixation(dm, scene, sampled, fx[0], cfg)  # warm
    dm.values  # settle the warm-up map (its queued fixation runs, it is read back)
    dm = gm.DensityMap.zeros(sampled)
    t0 = time.perf_counter()
    for f in fx:
        gm.accumulate_fixation(dm, scene, sampled, f, cfg)
    vals = {oid: v.copy() for oid, v in dm.values.items()}  # the one read-back
    t_loop = time.perf_counter() - t0
    same = all(np.array_equal(vals[o], full.values[o]) for o in full.values) and dm.global_max == full.global_max
    print(json.dumps({"fixations": a.fixations, "samples": int(sum(len(v) for v in vals.values())),
                      "generate_ms": t_gen * 1e3, "accumulate_fixation_loop_ms": t_loop * 1e3,
                      "ratio": t_loop / t_gen, "per_call_ms": t_loop * 1e3 / a.fixations, "bitwise_equal": same}))


if __name__ == "__main__":
    main()
