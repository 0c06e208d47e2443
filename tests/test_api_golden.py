"""Crop-frustum, raster and render API against the reference's own outputs
(tests/golden/api.npz, from tests/golden/make_api_golden.py).  The crop
frustum (a9) is host C++ and runs on CPU; raster/render run on the GPU."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_2601_07571_b200 as gm
import workloads as W
from paper_2601_07571_b200 import raster

G = dict(np.load(Path(__file__).resolve().parent / "golden" / "api.npz"))


def _bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("ti", [0, 1, 2])
def test_ellipse_and_bounds_bitwise(ti):
    cone = gm.GazeCone.from_theta(float(G[f"a9_theta{ti}"]))
    for i, g in enumerate(G["a9_gaze"]):
        err = int(G[f"a9_err{ti}"][i])
        if err:
            msg = "reach the near clip plane" if err == 1 else "does not cut the near plane"
            with pytest.raises(gm.GazeOutsideFrustumError, match=msg):
                gm.ellipse_intersection(g, 0.1, cone)
            continue
        e = gm.ellipse_intersection(g, 0.1, cone)
        np.testing.assert_array_equal(_bits(e.packed()), _bits(G[f"a9_ell{ti}"][i]))
        np.testing.assert_array_equal(_bits(gm.crop_bounds(e)), _bits(G[f"a9_bounds{ti}"][i]))


def test_build_crop_frustum_matches_setup_table():
    """build_crop_frustum's projection is the one the generation setup uses."""
    fx = W.orbit_fixations(20, 3, 2.0, 3.0)
    cone = gm.GazeCone.from_theta(gm.DEFAULT_THETA)
    setup = gm.fixation_setup(fx)
    for row, s in zip(fx, setup):
        f = gm.Fixation(row[0], row[1], row[2:5], row[5:9], tuple(row[9:15]), row[15:18])
        cf = gm.build_crop_frustum(f, cone)
        p = cf.projection_matrix
        assert (p[0, 0], p[1, 1], p[0, 2], p[1, 2]) == (s[16], s[17], s[18], s[19])
        assert cf.near == row[13] and cf.far == row[14]


def _scene():
    return W.rotated_object_scene()


@pytest.mark.gpu
def test_cull_and_rasterize_depth():
    scene = _scene()
    view, proj = G["r_view"], G["r_proj"]
    tris = raster.scene_world_triangles(scene)
    keep = raster._cull_mask(tris, raster.frustum_planes(proj @ view))
    np.testing.assert_array_equal(keep, G["r_keep"])
    buf = gm.rasterize_depth(scene, view, proj, (96, 64))
    np.testing.assert_array_equal(_bits(buf.depth), _bits(G["r_depth"]))
    np.testing.assert_array_equal(gm.depth_to_image(buf), G["r_image"])
    vis = np.array([gm.is_visible(buf, p) for p in G["r_pts"]])
    np.testing.assert_array_equal(vis, G["r_vis"])


@pytest.mark.gpu
def test_rasterize_with_attributes():
    scene = _scene()
    view, proj = G["r_view"], G["r_proj"]
    tris = raster.scene_world_triangles(scene)
    depth, tri_id, bary = raster.rasterize_with_attributes(tris, view, proj[0, 0], proj[1, 1], proj[0, 2], proj[1, 2],
                                                           (96, 64), 0.1, 50.0)
    np.testing.assert_array_equal(_bits(depth), _bits(G["r_adepth"]))
    np.testing.assert_array_equal(tri_id, G["r_atri"])
    np.testing.assert_array_equal(_bits(bary), _bits(G["r_abary"]))


def _render_setup():
    scene = _scene()
    sm = gm.build_sampled_meshes(scene, 3000.0)
    vals = {oid: G[f"h_val{i}"] for i, oid in enumerate(scene.object_ids)}
    dm = gm.DensityMap(vals, global_max=1.0, normalized=True)
    cam = np.array([0.3, 1.4, 3.2])
    q = W.look_at_quat(cam, [0.0, 0.2, 0.0])
    fr = (-0.12, 0.1, 0.07, -0.06, 0.1, 50.0)
    ramp = gm.ColorMap(tuple((float(r[0]), (float(r[1]), float(r[2]), float(r[3]))) for r in G["h_ramp"]))
    return scene, sm, dm, cam, q, fr, ramp


@pytest.mark.gpu
def test_render_heatmap_bytes(tmp_path):
    scene, sm, dm, cam, q, fr, ramp = _render_setup()
    img = gm.render_heatmap(scene, dm, sm, cam, q, fr, resolution=(120, 90), output_path=tmp_path / "h.png")
    np.testing.assert_array_equal(img, G["h_img_default"])
    from PIL import Image

    np.testing.assert_array_equal(np.asarray(Image.open(tmp_path / "h.png")), img)
    for tag, g in (("g1", 1.0), ("g2", 2.0)):
        img = gm.render_heatmap(scene, dm, sm, cam, q, fr, colormap=ramp.with_gamma(g), resolution=(64, 64))
        np.testing.assert_array_equal(img, G[f"h_img_{tag}"])


@pytest.mark.gpu
def test_render_heatmap_general_gamma_within_one_level():
    """gamma 0.7 goes through CUDA pow (<= 2 ulp vs glibc): channels may move
    by one level at a rounding boundary, nothing else."""
    scene, sm, dm, cam, q, fr, ramp = _render_setup()
    img = gm.render_heatmap(scene, dm, sm, cam, q, fr, colormap=ramp.with_gamma(0.7), resolution=(64, 64))
    diff = np.abs(img.astype(int) - G["h_img_g07"].astype(int))
    assert diff.max() <= 1
    assert (diff > 0).mean() < 1e-3


@pytest.mark.gpu
def test_render_rejects_unnormalized():
    scene, sm, dm, cam, q, fr, _ = _render_setup()
    with pytest.raises(gm.ConfigError):
        gm.render_heatmap(scene, gm.DensityMap(dm.values, 1.0, False), sm, cam, q, fr)


def test_host_depth_match_vs_oracle():
    """is_visible's depth test (C++ host, gm_depth_match) against the oracle's
    restatement of kernels.depth_match on random buffers with holes and edges."""
    from oracle import oracle as O
    from paper_2601_07571_b200 import _native

    rng = np.random.default_rng(5)
    lib = _native.load()
    for H, W in ((8, 8), (1, 7), (5, 1), (1, 1), (16, 9)):
        depth = rng.uniform(1.0, 1.01, (H, W))
        depth[rng.uniform(size=(H, W)) < 0.15] = np.inf
        depth[rng.uniform(size=(H, W)) < 0.15] += 0.5
        depth = np.ascontiguousarray(depth)
        for _ in range(300):
            fx, fy = rng.uniform(-1.0, W + 1.0), rng.uniform(-1.0, H + 1.0)
            d = float(rng.choice([1.0, 1.005, 1.3, 1.5, 2.0]))
            eps = float(rng.choice([1e-3, 5e-3, 0.2]))
            got = bool(lib.gm_depth_match(_native.dptr(depth), H, W, fx, fy, d, eps))
            assert got == O.depth_match(depth, fx, fy, d, eps), (H, W, fx, fy, d, eps)


@pytest.mark.gpu
def test_rasterize_with_attributes_deep_tiles():
    """16 nested shells seen whole: every tile is deep (bboxes cover it > 10x) and
    goes through the sorted crowded pass; depth, winner and barycentrics must
    still be the reference's bits."""
    base = W.icosphere(3, 1.0)
    shells = gm.Scene(tuple(gm.SceneObject(f"s{i}", gm.Mesh(base.vertices * (0.5 + 0.08 * i), base.faces))
                            for i in range(16)))
    view, proj = G["s_view"], G["s_proj"]
    tris = raster.scene_world_triangles(shells)
    depth, tri_id, bary = raster.rasterize_with_attributes(tris, view, proj[0, 0], proj[1, 1], proj[0, 2], proj[1, 2],
                                                           (160, 128), 0.1, 50.0)
    np.testing.assert_array_equal(_bits(depth), _bits(G["s_depth"]))
    np.testing.assert_array_equal(tri_id, G["s_tri"])
    np.testing.assert_array_equal(_bits(bary), _bits(G["s_bary"]))
