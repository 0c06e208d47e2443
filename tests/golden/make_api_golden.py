"""Golden outputs of the reference's crop-frustum, raster and render API
(SURVEY.md 8a rows a9, a11, a12, a14 and 8f-2), produced by the REFERENCE.

    python tests/golden/make_api_golden.py   -> tests/golden/api.npz

* a9: ellipse_intersection / crop_bounds / build_crop_frustum for 60 gaze
  directions (central, tilted, grazing -- both GazeOutsideFrustumError
  messages) and three cone angles.
* a11/a12/a14: on the rotated-object scene, a general camera (non-square
  96 x 64 buffer): cull_mask keep set, rasterize_depth, kernels.rasterize
  with attributes (depth, tri_id, bary), is_visible of 200 points,
  depth_to_image.
* 8f-2: render_heatmap images (default ramp; a 3-stop ramp with gamma 1, 2
  and 0.7) of a normalized map on that scene at 120 x 90 and 64 x 64.
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GAZEMAP_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

import gazemap as R  # noqa: E402
from gazemap import kernels, raster  # noqa: E402

import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "api.npz"


def gazes(rng, n):
    out = [np.array([0.0, 0.0, -1.0]), np.array([0.0, 0.3, -1.0]), np.array([0.9, 0.0, -0.2]),
           np.array([1.0, 0.0, -0.05]), np.array([0.0, 1.0, 0.0]), np.array([0.2, -0.1, -1.0])]
    while len(out) < n:
        g = rng.normal(size=3)
        g[2] = -abs(g[2]) * rng.uniform(0.05, 3.0)
        out.append(g / np.linalg.norm(g))
    return out


def ref_scene():
    objs = []
    for o in W.rotated_object_scene().objects:
        t = o.transform
        objs.append(R.SceneObject(o.object_id, R.Mesh(o.mesh.vertices, o.mesh.faces),
                                  R.Transform(t.translation, t.rotation, t.scale)))
    return R.Scene(tuple(objs))


def main():
    rng = np.random.default_rng(7)
    d = {}
    # ---- a9
    gs = gazes(rng, 60)
    d["a9_gaze"] = np.array(gs)
    for ti, theta in enumerate((math.radians(1.0), math.radians(5.0), 0.3)):
        cone = R.GazeCone.from_theta(theta)
        ell = np.full((len(gs), 18), np.nan)
        bounds = np.full((len(gs), 4), np.nan)
        err = np.zeros(len(gs), np.int64)
        for i, g in enumerate(gs):
            try:
                e = R.ellipse_intersection(g, 0.1, cone)
            except R.GazeOutsideFrustumError as ex:
                err[i] = 1 if "reach" in str(ex) else 2
                continue
            ell[i] = np.concatenate([e.center_E, [e.major_a, e.minor_b, e.inclination_alpha], e.A0, e.A1, e.B0, e.B1])
            bounds[i] = R.crop_bounds(e)
        d[f"a9_theta{ti}"] = np.float64(theta)
        d[f"a9_ell{ti}"] = ell
        d[f"a9_bounds{ti}"] = bounds
        d[f"a9_err{ti}"] = err
    # ---- raster
    scene = ref_scene()
    cam = np.array([0.3, 1.4, 3.2])
    q = W.look_at_quat(cam, [0.0, 0.2, 0.0])
    fr = (-0.12, 0.1, 0.07, -0.06, 0.1, 50.0)
    fx = R.Fixation(0.0, 1.0, cam, q, fr, [0.0, 0.0, -1.0])
    view = fx.view_matrix()
    proj = fx.projection_matrix()
    d["r_view"], d["r_proj"] = view, proj
    planes = raster.frustum_planes(proj @ view)
    tris = raster.scene_world_triangles(scene)
    d["r_keep"] = kernels.cull_mask(tris, np.ascontiguousarray(planes))
    buf = raster.rasterize_depth(scene, view, proj, (96, 64))
    d["r_depth"] = buf.depth
    d["r_image"] = raster.depth_to_image(buf)
    W_, H_ = 96, 64
    depth = np.full((H_, W_), np.inf)
    tri_id = np.full((H_, W_), -1, np.int32)
    bary = np.zeros((H_, W_, 3))
    kernels.rasterize(np.ascontiguousarray(tris), np.ascontiguousarray(view[:3, :3]), np.ascontiguousarray(view[:3, 3]),
                      proj[0, 0], proj[1, 1], proj[0, 2], proj[1, 2], W_, H_, 0.1, 50.0, depth, tri_id, bary, True)
    d["r_adepth"], d["r_atri"], d["r_abary"] = depth, tri_id, bary
    pts = tris[rng.integers(0, len(tris), 200)].mean(axis=1) + rng.normal(0, 0.01, (200, 3))
    d["r_pts"] = pts
    d["r_vis"] = np.array([raster.is_visible(buf, p) for p in pts])
    # ---- raster with attributes on nested shells (deep tiles: the sorted crowded pass)
    base = R.Mesh(W.icosphere(3, 1.0).vertices, W.icosphere(3, 1.0).faces)
    shells = R.Scene(tuple(R.SceneObject(f"s{i}", R.Mesh(base.vertices * (0.5 + 0.08 * i), base.faces))
                           for i in range(16)))
    scam = np.array([0.4, 0.3, 3.0])
    sq = W.look_at_quat(scam, [0.0, 0.0, 0.0])
    sfx = R.Fixation(0.0, 1.0, scam, sq, (-0.1, 0.1, 0.1, -0.1, 0.1, 50.0), [0.0, 0.0, -1.0])
    sview, sproj = sfx.view_matrix(), sfx.projection_matrix()
    stris = raster.scene_world_triangles(shells)
    sd = np.full((128, 160), np.inf)
    sid = np.full((128, 160), -1, np.int32)
    sb = np.zeros((128, 160, 3))
    kernels.rasterize(np.ascontiguousarray(stris), np.ascontiguousarray(sview[:3, :3]),
                      np.ascontiguousarray(sview[:3, 3]), sproj[0, 0], sproj[1, 1], sproj[0, 2], sproj[1, 2],
                      160, 128, 0.1, 50.0, sd, sid, sb, True)
    d["s_view"], d["s_proj"], d["s_depth"], d["s_tri"], d["s_bary"] = sview, sproj, sd, sid, sb
    # ---- render
    sm = R.build_sampled_meshes(scene, 3000.0)
    vals = {}
    for i, oid in enumerate(scene.object_ids):
        n = sm[oid].total_samples
        v = rng.uniform(0.0, 1.0, n) ** 3
        v[rng.uniform(size=n) < 0.2] = 0.0
        vals[oid] = v
    m = max(v.max() for v in vals.values())
    dm = R.DensityMap({k: v / m for k, v in vals.items()}, global_max=1.0, normalized=True)
    for i, oid in enumerate(scene.object_ids):
        d[f"h_val{i}"] = dm.values[oid]
    ramp = R.ColorMap(((0.0, (0.0, 0.0, 0.2)), (0.4, (0.9, 0.3, 0.0)), (1.0, (1.0, 1.0, 0.8))))
    d["h_ramp"] = np.array([[s[0], *s[1]] for s in ramp.stops])
    d["h_img_default"] = R.render_heatmap(scene, dm, sm, cam, q, fr, resolution=(120, 90))
    for tag, g in (("g1", 1.0), ("g2", 2.0), ("g07", 0.7)):
        d[f"h_img_{tag}"] = R.render_heatmap(scene, dm, sm, cam, q, fr, colormap=ramp.with_gamma(g),
                                             resolution=(64, 64))
    np.savez_compressed(OUT, **d)
    print(f"wrote {OUT}; a9 errors {[int((d[f'a9_err{t}'] > 0).sum()) for t in range(3)]}, "
          f"covered {(tri_id >= 0).mean():.2f}, visible {d['r_vis'].mean():.2f}")


if __name__ == "__main__":
    main()
