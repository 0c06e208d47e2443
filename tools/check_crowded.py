"""Count the k_texels tiles routed to the crowded pass for a scene/fixations (diagnostic)."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_07571_b200 as gm  # noqa: E402
import workloads as W  # noqa: E402
from paper_2601_07571_b200 import _native  # noqa: E402

base = W.icosphere(3, 1.0)
scene = gm.Scene(tuple(gm.SceneObject(f"s{i}", gm.Mesh(base.vertices * (0.5 + 0.08 * i), base.faces))
                       for i in range(16)))
fx = W.orbit_fixations(6, 7, 2.6, 3.2, jitter=0.2)
for filt in (False, True):
    cfg = gm.GenerationConfig(k=1500.0, filtering_enabled=filt)
    sm = gm.build_sampled_meshes(scene, cfg.k)
    plan = gm.density.get_plan(scene, sm, cfg)
    plan.accumulate(fx, cfg, flags=_native.GM_FLAG_STATS)
    st = (ctypes.c_uint64 * len(_native.STAT_NAMES))()
    plan._lib.gm_plan_stats(plan._h, st)
    d = dict(zip(_native.STAT_NAMES, [int(x) for x in st]))
    print("filtering", filt, "tiles", d["tx_tiles"], "crowded", d["tx_crowded"])
