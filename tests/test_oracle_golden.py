"""Pin the CPU oracle (oracle/gm_oracle.c) to the reference's own outputs
(tests/golden/golden.npz, produced by tests/golden/make_golden.py running
/root/reference).  Everything here is bitwise: the oracle restates the
reference's floating-point operation order exactly."""

import numpy as np
import pytest

from oracle import oracle as O


def _layouts(g, prefix, k):
    scene = g.scene(prefix)
    return scene, O.build_layouts(scene, k)


@pytest.mark.parametrize("k", [1000, 6000])
def test_layout_and_world_positions_bitwise(golden, k):
    scene, lay = _layouts(golden, "lay_", float(k))
    world = O.world_samples(scene, lay)
    for i, obj in enumerate(scene.objects):
        res, cnt, off, total = lay[obj.object_id]
        tag = f"lay_k{k}_{i}_"
        np.testing.assert_array_equal(res, golden[tag + "res"])
        np.testing.assert_array_equal(off, golden[tag + "off"])
        assert total == int(golden[tag + "total"])
        np.testing.assert_array_equal(world[obj.object_id], golden[tag + "world"])


def test_fixation_setup_bitwise(golden):
    fx = golden["setup_fix"]
    ref = golden["setup_out"]
    theta = float(golden["setup_theta"])
    for row, want in zip(fx, ref):
        s = O.fixation_setup(row, theta, True)
        got = np.array([*s[O.FS_ROT:O.FS_ROT + 9], *s[O.FS_TRANS:O.FS_TRANS + 3], s[O.FS_P00], s[O.FS_P11],
                        s[O.FS_P02], s[O.FS_P12], s[O.FS_NEAR], s[O.FS_FAR], s[O.FS_CROPPED], s[O.FS_AMP]])
        np.testing.assert_array_equal(got, want)
    # both branches (crop and GazeOutsideFrustumError fallback) are covered
    assert 0 < ref[:, 18].sum() < len(ref)


def test_rasterize_bitwise(golden):
    import math

    for i in range(int(golden["ras_count"])):
        scene = golden.scene(f"ras_{golden[f'ras{i}_scene']}_")
        row = golden[f"ras{i}_fix"]
        crop = bool(golden[f"ras{i}_crop"])
        want = golden[f"ras{i}_depth"]
        s = O.fixation_setup(row, math.radians(1.0), crop)
        assert bool(s[O.FS_CROPPED]) == crop
        tris = O.scene_world_triangles(scene)
        planes = O.frustum_planes(s[O.FS_PROJ:O.FS_PROJ + 16].reshape(4, 4), s[O.FS_VIEW:O.FS_VIEW + 16].reshape(4, 4))
        tris = tris[O.cull_mask(tris, planes)]
        got = O.rasterize(tris, s[O.FS_ROT:O.FS_ROT + 9], s[O.FS_TRANS:O.FS_TRANS + 3], s[O.FS_P00], s[O.FS_P11],
                          s[O.FS_P02], s[O.FS_P12], want.shape[1], want.shape[0], s[O.FS_NEAR], s[O.FS_FAR])
        np.testing.assert_array_equal(got, want)


def test_filter_candidates_bitwise(golden):
    import math

    scene = golden.scene("fil_")
    lay = O.build_layouts(scene, float(golden["fil_k"]))
    world = O.world_samples(scene, lay)
    pos = np.concatenate([world[o.object_id] for o in scene.objects])
    for j, row in enumerate(golden["fil_fix"]):
        s = O.fixation_setup(row, math.radians(1.0), True)
        np.testing.assert_array_equal(O.candidates(pos, s), golden[f"fil{j}_idx"])


@pytest.mark.parametrize("case", ["c1", "sib_off", "chal_on", "quads_incl"])
def test_generate_bitwise(golden, case):
    p = f"gen_{case}_"
    scene = golden.scene(p)
    fx = golden[p + "fix"]
    incl = [str(x) for x in golden[p + "incl"]] or None

    vals, gmax = O.generate(scene, O.rows_as_fixations(fx), k=float(golden[p + "k"]),
                            zbuffer_resolution=int(golden[p + "res"]),
                            filtering_enabled=bool(golden[p + "filt"]),
                            object_include_list=set(incl) if incl else None)
    assert gmax == float(golden[p + "gmax"])
    for i, obj in enumerate(scene.objects):
        np.testing.assert_array_equal(vals[obj.object_id], golden[f"{p}val{i}"])
    assert (gmax > 0) == any(np.count_nonzero(vals[o.object_id]) for o in scene.objects)
