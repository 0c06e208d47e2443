"""The reference's own density / estimator test cases (pkg/tests/test_density.py,
test_raster.py, test_acceptance.py criteria 6, 8, 9), run through this
package's drop-in API on the GPU."""

import math

import numpy as np
import pytest

import paper_2601_07571_b200 as gm
import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ON_AXIS_WEIGHT = 1.0 / (math.tan(0.05) * math.sqrt(2.0 * math.pi))


def fix(position, target=None, gaze=(0.0, 0.0, -1.0), duration=1.0, start=0.0):
    q = W.look_at_quat(position, target) if target is not None else np.array([0.0, 0.0, 0.0, 1.0])
    return gm.Fixation(start, duration, np.asarray(position, float), q, W.FRUSTUM, np.asarray(gaze, float))


def run(scene, fixations, **kw):
    cfg = gm.GenerationConfig(**kw)
    sampled = gm.build_sampled_meshes(scene, cfg.k)
    return gm.generate(scene, sampled, fixations, cfg), sampled, cfg


def quad_scene(half=1.0, z=-2.0):
    return gm.Scene((gm.SceneObject("q", W.quad(half, z)),))


def two_quads():
    return gm.Scene((gm.SceneObject("front", W.quad(5.0, -2.0)), gm.SceneObject("back", W.quad(5.0, -4.0))))


def sphere_in_box():
    return gm.Scene((gm.SceneObject("box", W.box(1.0)), gm.SceneObject("sphere", W.icosphere(2, 0.5))))


def test_gaze_away_from_object_all_zero():
    scene = gm.Scene((gm.SceneObject("q", W.quad(0.2, -2.0), gm.Transform([3.0, 0, 0], [0, 0, 0, 1], [1, 1, 1])),))
    dm, _, _ = run(scene, [fix([0.0, 0.0, 0.0])], k=1000.0)
    assert dm.global_max == 0.0 and np.all(dm.values["q"] == 0.0)


def test_object_behind_viewpoint_all_zero():
    dm, _, _ = run(quad_scene(z=2.0), [fix([0.0, 0.0, 0.0])], k=1000.0)
    assert np.all(dm.values["q"] == 0.0)


def test_on_axis_sample_weight():
    v = np.array([[0.0, 0.0, -2.0], [0.3, 0.0, -2.0], [0.0, 0.3, -2.0]])
    scene = gm.Scene((gm.SceneObject("t", gm.Mesh(v, [[0, 1, 2]])),))
    dm, _, _ = run(scene, [fix([0.0, 0.0, 0.0])], k=100.0, theta=0.05)
    assert dm.global_max == pytest.approx(ON_AXIS_WEIGHT, rel=1e-12)
    assert dm.global_max == pytest.approx(7.97219546, abs=1e-6)


def test_matches_direct_weights_when_unoccluded():
    scene = quad_scene()
    f = fix([0.0, 0.0, 0.0])
    dm, sampled, cfg = run(scene, [f], k=2000.0)
    pts = gm.sample_positions_local(scene.objects[0].mesh, sampled["q"])
    cam = pts @ f.view_matrix()[:3, :3].T + f.view_matrix()[:3, 3]
    expected = np.array([gm.gaussian_weight(c, f.gaze_dir, f.duration, cfg.cone()) for c in cam])
    np.testing.assert_allclose(dm.values["q"], expected, rtol=1e-12, atol=0.0)


def test_two_identical_fixations_double_exactly():
    scene = quad_scene()
    f = fix([0.0, 0.0, 0.0])
    one, _, _ = run(scene, [f], k=1000.0)
    two, _, _ = run(scene, [f, f], k=1000.0)
    np.testing.assert_array_equal(two.values["q"], 2.0 * one.values["q"])
    assert two.global_max == 2.0 * one.global_max


def test_duration_scales_linearly():
    a, _, _ = run(quad_scene(), [fix([0.0, 0.0, 0.0], duration=1.0)], k=1000.0)
    b, _, _ = run(quad_scene(), [fix([0.0, 0.0, 0.0], duration=2.5)], k=1000.0)
    np.testing.assert_allclose(b.values["q"], 2.5 * a.values["q"], rtol=1e-12)


def test_zero_fixations():
    dm, _, _ = run(two_quads(), [], k=1000.0)
    assert dm.global_max == 0.0 and dm.total_samples > 0
    assert all(np.all(v == 0.0) for v in dm.values.values())


def test_occluded_back_quad_zero():
    dm, _, _ = run(two_quads(), [fix([0.0, 0.0, 0.0])], k=1000.0)
    assert np.all(dm.values["back"] == 0.0)
    assert dm.values["front"].max() > 0.0


def test_global_max_tracks_values():
    dm, _, _ = run(sphere_in_box(), [fix([0.0, 0.0, 3.0], target=[0.0, 0.0, 0.0])], k=5000.0)
    assert dm.global_max == max(v.max() for v in dm.values.values()) > 0.0


def test_object_include_list():
    dm, _, _ = run(two_quads(), [fix([0.0, 0.0, 0.0])], k=1000.0, object_include_list={"back"})
    assert np.all(dm.values["front"] == 0.0)
    dm2, _, _ = run(two_quads(), [fix([0.3, 0.2, 0.5])], k=1000.0, object_include_list={"front"})
    assert np.all(dm2.values["back"] == 0.0) and dm2.values["front"].max() > 0


def test_partition_additivity():
    scene = sphere_in_box()
    fx = [fix([0.0, 0.0, 3.0], target=[0, 0, 0], start=float(i)) for i in range(3)] + \
         [fix([2.0, 1.0, 2.0], target=[0.1, 0, 0], start=float(i + 3)) for i in range(3)]
    full, _, _ = run(scene, fx, k=5000.0)
    first, _, _ = run(scene, fx[:3], k=5000.0)
    second, _, _ = run(scene, fx[3:], k=5000.0)
    for oid in full.values:
        np.testing.assert_allclose(full.values[oid], first.values[oid] + second.values[oid], rtol=1e-9, atol=1e-12)


def test_timings_and_progress():
    scene = quad_scene()
    cfg = gm.GenerationConfig(k=1000.0)
    sampled = gm.build_sampled_meshes(scene, cfg.k)
    timers = gm.Timings()
    seen = []
    f = fix([0.0, 0.0, 0.0])
    gm.generate(scene, sampled, [f, f], cfg, timers=timers, progress=lambda i, n: seen.append((i, n)))
    assert seen == [(1, 2), (2, 2)]
    for phase in ("cull", "rasterize", "accumulate"):
        assert timers.phases[phase] >= 0.0
    assert timers.phases["rasterize"] > 0.0


def test_filtered_matches_unfiltered():
    scene = sphere_in_box()
    f = fix([2.0, 1.5, 2.5], target=[0.0, 0.0, 0.0])
    on, _, _ = run(scene, [f], k=5000.0, filtering_enabled=True)
    off, _, _ = run(scene, [f], k=5000.0, filtering_enabled=False)
    for oid in on.values:
        np.testing.assert_allclose(on.values[oid], off.values[oid], rtol=1e-6, atol=1e-12)


def test_grazing_cone_falls_back_to_unfiltered_bitwise():
    g = np.array([1.0, 0.0, -0.01])
    f = fix([0.0, 0.0, 0.0], gaze=g / np.linalg.norm(g))
    on, _, _ = run(quad_scene(), [f], k=1000.0, filtering_enabled=True)
    off, _, _ = run(quad_scene(), [f], k=1000.0, filtering_enabled=False)
    for oid in on.values:
        np.testing.assert_array_equal(on.values[oid], off.values[oid])


def test_filtering_equivalence_criterion_6():
    """Acceptance criterion 6 (test_acceptance.py:289-323): >= 99.9% of samples
    agree within 1e-6 and every disagreement is a visibility flip."""
    scene = sphere_in_box()
    fx = [fix([0.0, 0.0, 3.0], target=[0, 0, 0]), fix([1.8, 1.4, 2.2], target=[0, 0, 0]),
          fix([-2.0, 0.5, 2.0], target=[0.2, 0, 0])]
    on, _, _ = run(scene, fx, k=20000.0, filtering_enabled=True)
    off, _, _ = run(scene, fx, k=20000.0, filtering_enabled=False)
    scale = max(off.global_max, 1e-300)
    agree = total = unexplained = 0
    for oid in on.values:
        a, b = on.values[oid], off.values[oid]
        match = np.abs(a - b) / scale <= 1e-6
        agree += int(match.sum())
        total += len(a)
        bad = np.nonzero(~match)[0]
        unexplained += int(np.sum((a[bad] == 0.0) == (b[bad] == 0.0)))
    assert agree / total >= 0.999 and unexplained == 0


def test_deterministic_across_runs_and_batch_sizes():
    scene = sphere_in_box()
    fx = W.orbit_fixations(64, 9, 2.0, 4.0, jitter=0.3)
    cfg = gm.GenerationConfig(k=10000.0)
    sampled = gm.build_sampled_meshes(scene, cfg.k)
    ref = gm.generate(scene, sampled, fx, cfg)
    for b in (0, 1, 7, 64):
        again = gm.generate(scene, sampled, fx, cfg, batch=b)
        assert again.global_max == ref.global_max
        for oid in ref.values:
            np.testing.assert_array_equal(again.values[oid], ref.values[oid])


def test_accumulate_fixation_in_place():
    scene = sphere_in_box()
    cfg = gm.GenerationConfig(k=5000.0)
    sampled = gm.build_sampled_meshes(scene, cfg.k)
    fx = [fix([0.0, 0.0, 3.0], target=[0, 0, 0]), fix([2.0, 1.0, 2.0], target=[0.1, 0, 0])]
    dm = gm.DensityMap.zeros(sampled)
    for f in fx:
        out = gm.accumulate_fixation(dm, scene, sampled, f, cfg)
        assert out is dm
    full = gm.generate(scene, sampled, fx, cfg)
    for oid in dm.values:
        np.testing.assert_array_equal(dm.values[oid], full.values[oid])
    assert dm.global_max == full.global_max


def test_accumulate_fixation_loop_stays_on_device():
    """A loop of accumulate_fixation keeps the map on the GPU (no full-map
    copies per call) and still matches generate bit for bit; reading
    .values mid-loop, editing the arrays, interleaving generate() on the same
    plan and a second map on the same plan all behave like the reference."""
    scene, k, table = W.c1()
    cfg = gm.GenerationConfig(k=k)
    sampled = gm.build_sampled_meshes(scene, k)
    fx = [gm.Fixation(r[0], r[1], r[2:5], r[5:9], tuple(r[9:15]), r[15:18]) for r in table[:24]]
    dm = gm.DensityMap.zeros(sampled)
    held = dm.values["icosphere"]  # the array object must keep receiving the values
    for f in fx[:12]:
        gm.accumulate_fixation(dm, scene, sampled, f, cfg)
    half = gm.generate(scene, sampled, fx[:12], cfg)  # reuses the plan: dm is read back first
    np.testing.assert_array_equal(held, half.values["icosphere"])
    assert dm.global_max == half.global_max
    for f in fx[12:18]:
        gm.accumulate_fixation(dm, scene, sampled, f, cfg)
    v = dm.values["icosphere"]  # readback, and the caller may now edit the arrays
    assert v is held
    np.testing.assert_array_equal(v, gm.generate(scene, sampled, fx[:18], cfg).values["icosphere"])
    other = gm.DensityMap.zeros(sampled)
    gm.accumulate_fixation(other, scene, sampled, fx[0], cfg)  # takes the plan over
    for f in fx[18:]:
        gm.accumulate_fixation(dm, scene, sampled, f, cfg)
    full = gm.generate(scene, sampled, fx, cfg)
    np.testing.assert_array_equal(dm.values["icosphere"], full.values["icosphere"])
    assert dm.global_max == full.global_max
    np.testing.assert_array_equal(other.values["icosphere"],
                                  gm.generate(scene, sampled, fx[:1], cfg).values["icosphere"])
    # an edit of the host arrays after reading them is honoured by the next call
    dm.values["icosphere"][:] = 0.0
    gm.accumulate_fixation(dm, scene, sampled, fx[0], cfg)
    np.testing.assert_array_equal(dm.values["icosphere"],
                                  gm.generate(scene, sampled, fx[:1], cfg).values["icosphere"])


def test_normalize_and_estimator():
    scene = sphere_in_box()
    dm, _, _ = run(scene, [fix([0.0, 0.0, 3.0], target=[0, 0, 0])], k=5000.0)
    out = gm.normalize(dm)
    assert out.normalized and out.global_max == 1.0
    assert max(v.max() for v in out.values.values()) == 1.0
    assert all(v.min() >= 0.0 for v in out.values.values())
    twice = gm.normalize(out)
    for oid in out.values:
        np.testing.assert_array_equal(out.values[oid], twice.values[oid])
    for oid in dm.values:  # GPU normalize == numpy division
        np.testing.assert_array_equal(out.values[oid], dm.values[oid] / dm.global_max)
    est = gm.FixationDensityMapper(scene=scene, k=5000.0)
    X = [fix([0.0, 0.0, 3.0], target=[0, 0, 0])]
    est.fit(X)
    vec = est.transform(X)
    assert vec.shape == (est.n_samples_out_,)
    np.testing.assert_array_equal(vec, np.concatenate([est.density_map_.values[o] for o in scene.object_ids]))
    with pytest.raises(ValueError):
        gm.FixationDensityMapper().fit(X)


def test_reference_dataclasses_accepted():
    """Duck typing: objects shaped like the reference's dataclasses."""

    class Obj:
        def __init__(self, oid, mesh):
            self.object_id, self.mesh, self.transform = oid, mesh, gm.Transform.identity()

    class Sc:
        def __init__(self, objs):
            self.objects = tuple(objs)

        @property
        def object_ids(self):
            return [o.object_id for o in self.objects]

    scene = Sc([Obj("front", W.quad(5.0, -2.0)), Obj("back", W.quad(5.0, -4.0))])
    cfg = gm.GenerationConfig(k=1000.0)
    sampled = gm.build_sampled_meshes(scene, cfg.k)
    rows = O.rows_as_fixations(W.orbit_fixations(3, 1, 2.0, 3.0))
    dm = gm.generate(scene, sampled, rows, cfg)
    vals, gmax = O.generate(scene, rows, k=cfg.k)
    for oid in vals:
        np.testing.assert_allclose(dm.values[oid], vals[oid], rtol=1e-12, atol=0)


def test_integration_md_ctypes_stub_runs():
    """The ctypes stub INTEGRATION.md section 2 tells a reference maintainer to
    add (gazemap/_b200.py replacing density.generate) is executed as written,
    against the built library, and gives the package's own result."""
    import re
    from pathlib import Path

    from paper_2601_07571_b200 import _native

    text = (Path(__file__).resolve().parents[1] / "INTEGRATION.md").read_text()
    block = re.findall(r"```python\n(# gazemap/_b200\.py.*?)```", text, re.S)[0]
    block = block.replace("/path/to/_gazemap_b200.so", str(_native.SO_PATH))
    ns = {"DensityMap": gm.DensityMap, "InvalidFrustumError": gm.InvalidFrustumError}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    scene, k, table = W.c1()
    fx = [gm.Fixation(r[0], r[1], r[2:5], r[5:9], tuple(r[9:15]), r[15:18]) for r in table[:64]]
    cfg = gm.GenerationConfig(k=k)
    sampled = gm.build_sampled_meshes(scene, k)
    got = ns["generate"](scene, sampled, fx, cfg)
    want = gm.generate(scene, sampled, fx, cfg)
    assert got.global_max == want.global_max > 0
    for oid in want.values:
        np.testing.assert_array_equal(got.values[oid], want.values[oid])


def test_accumulate_fixation_zero_map_replaced_values():
    """A DensityMap.zeros whose values dict is replaced (or read and edited)
    before the first call must be uploaded, not cleared on the device."""
    scene, k, table = W.c1()
    cfg = gm.GenerationConfig(k=k)
    sampled = gm.build_sampled_meshes(scene, k)
    fx = [gm.Fixation(r[0], r[1], r[2:5], r[5:9], tuple(r[9:15]), r[15:18]) for r in table[:6]]
    base = gm.generate(scene, sampled, fx[:3], cfg)
    dm = gm.DensityMap.zeros(sampled)
    dm.values = {o: v.copy() for o, v in base.values.items()}
    dm.global_max = base.global_max
    for f in fx[3:]:
        gm.accumulate_fixation(dm, scene, sampled, f, cfg)
    full = gm.generate(scene, sampled, fx, cfg)
    np.testing.assert_allclose(dm.values["icosphere"], full.values["icosphere"], rtol=1e-12, atol=0.0)
    assert dm.global_max == pytest.approx(full.global_max, rel=1e-12)
