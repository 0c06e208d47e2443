"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Every array stored here is an output of the reference package itself
(/root/reference/pkg/src/gazemap), so tests that compare the oracle or the
CUDA product against these files are pinned to the reference, not to a
restatement.  The GPU box has no /root/reference; it only reads the .npz.
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GAZEMAP_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

import gazemap as gm  # noqa: E402
from gazemap import kernels, raster  # noqa: E402
from gazemap.geometry import sample_positions_local  # noqa: E402
from scenes import (  # noqa: E402
    challenging_scene,
    icosphere_mesh,
    look_at_quat,
    make_fixation,
    sphere_in_box_scene,
    two_quads_scene,
)

OUT = Path(__file__).resolve().parent
FRUSTUM = (-0.1, 0.1, 0.1, -0.1, 0.1, 100.0)


def fixation_rows(fixations):
    rows = []
    for f in fixations:
        rows.append([f.start_time, f.duration, *f.camera_position, *f.camera_rotation, *f.frustum, *f.gaze_dir])
    return np.array(rows, dtype=np.float64).reshape(-1, 18)


def scene_arrays(scene, prefix, d):
    d[prefix + "ids"] = np.array(scene.object_ids)
    for i, o in enumerate(scene.objects):
        d[f"{prefix}v{i}"] = o.mesh.vertices
        d[f"{prefix}f{i}"] = o.mesh.faces
        d[f"{prefix}t{i}"] = np.concatenate([o.transform.translation, o.transform.rotation, o.transform.scale])


def tilted_gaze(rng, max_tilt):
    down = np.array([0.0, 0.0, -1.0])
    a = rng.uniform(0.0, 2.0 * math.pi)
    axis = np.array([math.cos(a), math.sin(a), 0.0])
    ang = rng.uniform(0.0, max_tilt)
    c, s = math.cos(ang), math.sin(ang)
    return down * c + np.cross(axis, down) * s + axis * (axis @ down) * (1.0 - c)


def c1_fixations(seed=0, n=200):
    """cameras at radius U(2.5,4) looking at the origin."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        pos = d * rng.uniform(2.5, 4.0)
        q = look_at_quat(pos, [0.0, 0.0, 0.0]) if abs(d[1]) < 0.999 else np.array([0.0, 0.0, 0.0, 1.0])
        out.append(gm.Fixation(0.25 * i, rng.uniform(0.1, 0.6), pos, q, FRUSTUM, tilted_gaze(rng, 0.15)))
    return out


def main():
    d = {}
    # ---- stage 1: layout + positions (rotated, scaled transform) --------
    scene = challenging_scene()
    scene_arrays(scene, "lay_", d)
    for k in (1000.0, 6000.0):
        sm = gm.build_sampled_meshes(scene, k)
        for i, o in enumerate(scene.objects):
            s = sm[o.object_id]
            tag = f"lay_k{int(k)}_{i}_"
            d[tag + "res"] = s.resolutions
            d[tag + "off"] = s.offsets
            d[tag + "total"] = np.array(s.total_samples)
            d[tag + "world"] = o.transform.apply(sample_positions_local(o.mesh, s))

    # ---- per-fixation setup (crop frustum, view, near'/far') ------------
    rng = np.random.default_rng(11)
    cone = gm.GazeCone.from_theta(math.radians(1.0))
    fixes, recs = [], []
    for i in range(300):
        pos = rng.uniform(-3, 3, 3)
        tgt = rng.uniform(-3, 3, 3)
        g = tilted_gaze(rng, 1.5705 if i % 3 == 0 else 0.4)
        if g[2] >= -1e-6:
            continue
        fx = make_fixation(pos, target=tgt, gaze_dir=g, duration=rng.uniform(0.1, 0.6))
        view = fx.view_matrix()
        try:
            proj = gm.build_crop_frustum(fx, cone).projection_matrix
            cropped = 1.0
        except gm.GazeOutsideFrustumError:
            proj = fx.projection_matrix()
            cropped = 0.0
        _, _, _, _, n, f = gm.gaze.frustum_from_matrix(proj)
        recs.append([*view[:3, :3].ravel(), *view[:3, 3], proj[0, 0], proj[1, 1], proj[0, 2], proj[1, 2],
                     n, f, cropped, fx.duration / (cone.sigma * gm.gaze.SQRT_TWO_PI)])
        fixes.append(fx)
    d["setup_fix"] = fixation_rows(fixes)
    d["setup_out"] = np.array(recs)
    d["setup_theta"] = np.array(math.radians(1.0))

    # ---- raster: reference depth buffers --------------------------------
    scenes = {"sib": sphere_in_box_scene(), "chal": challenging_scene()}
    rfix = [make_fixation([1.8, 1.4, 2.2], target=[0.0, 0.0, 0.0]),
            make_fixation([-1.5, 2.5, 3.5], target=[0.2, 0.0, 0.0])]
    ri = 0
    for sname, sc in scenes.items():
        scene_arrays(sc, f"ras_{sname}_", d)
        for fx in rfix:
            for crop in (False, True):
                view = fx.view_matrix()
                proj = gm.build_crop_frustum(fx, cone).projection_matrix if crop else fx.projection_matrix()
                for res in (97, 160):
                    buf = gm.rasterize_depth(sc, view, proj, (res, res))
                    d[f"ras{ri}_scene"] = np.array(sname)
                    d[f"ras{ri}_fix"] = fixation_rows([fx])[0]
                    d[f"ras{ri}_crop"] = np.array(crop)
                    d[f"ras{ri}_depth"] = buf.depth
                    ri += 1
    d["ras_count"] = np.array(ri)

    # ---- filter: the reference's own NDC-filtered index set -------------
    # kernels.accumulate with depth == 0, eps_abs = 1e300, gaze = -z and a
    # huge sigma adds exactly 1.0 to every sample that passes the NDC crop
    # filter (kernels.py:302-319) and to no other sample.
    sc = sphere_in_box_scene()
    sm = gm.build_sampled_meshes(sc, 20000.0)
    scene_arrays(sc, "fil_", d)
    world = np.concatenate([o.transform.apply(sample_positions_local(o.mesh, sm[o.object_id])) for o in sc.objects])
    ffix = c1_fixations(seed=3, n=12)
    for j, fx in enumerate(ffix):
        view = fx.view_matrix()
        try:
            proj = gm.build_crop_frustum(fx, cone).projection_matrix
        except gm.GazeOutsideFrustumError:
            proj = fx.projection_matrix()
        _, _, _, _, n, f = gm.gaze.frustum_from_matrix(proj)
        vals = np.zeros(len(world))
        kernels.accumulate(np.ascontiguousarray(world), np.ascontiguousarray(view[:3, :3]),
                           np.ascontiguousarray(view[:3, 3]), np.array([0.0, 0.0, -1.0]), 1e100, 1.0,
                           proj[0, 0], proj[1, 1], proj[0, 2], proj[1, 2], np.zeros((2, 2)), 1e300, 0.0,
                           n, f, vals)
        d[f"fil{j}_idx"] = np.nonzero(vals == 1.0)[0]
        assert np.all((vals == 0.0) | (vals == 1.0))
    d["fil_fix"] = fixation_rows(ffix)
    d["fil_k"] = np.array(20000.0)

    # ---- generate: end-to-end density maps ------------------------------
    cases = {
        "c1": (gm.Scene((gm.SceneObject("icosphere", icosphere_mesh(3, 1.0)),)), c1_fixations(0, 200), 1000.0, {}),
        "sib_off": (sphere_in_box_scene(), c1_fixations(5, 6), 2500.0, {"filtering_enabled": False}),
        "chal_on": (challenging_scene(), c1_fixations(6, 8), 4000.0, {"zbuffer_resolution": 300}),
        "quads_incl": (two_quads_scene(), [make_fixation([0.0, 0.0, 0.0]), make_fixation([0.3, 0.2, 0.5])],
                       300.0, {"object_include_list": {"back"}}),
    }
    for name, (sc, fx, k, kw) in cases.items():
        cfg = gm.GenerationConfig(k=k, **kw)
        sm = gm.build_sampled_meshes(sc, k)
        dm = gm.generate(sc, sm, fx, cfg)
        scene_arrays(sc, f"gen_{name}_", d)
        d[f"gen_{name}_fix"] = fixation_rows(fx)
        d[f"gen_{name}_k"] = np.array(k)
        d[f"gen_{name}_filt"] = np.array(cfg.filtering_enabled)
        d[f"gen_{name}_res"] = np.array(cfg.zbuffer_resolution)
        d[f"gen_{name}_incl"] = np.array(sorted(cfg.object_include_list) if cfg.object_include_list else [])
        d[f"gen_{name}_gmax"] = np.array(dm.global_max)
        for i, oid in enumerate(sc.object_ids):
            d[f"gen_{name}_val{i}"] = dm.values[oid]
    d["gen_cases"] = np.array(list(cases))
    np.savez_compressed(OUT / "golden.npz", **d)
    print("wrote", OUT / "golden.npz", sum(v.nbytes for v in d.values()), "bytes raw")


if __name__ == "__main__":
    main()
