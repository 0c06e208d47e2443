"""Full-size checks on the bench workload (C2 room: 98,080 triangles,
2,189,280 samples): bit-exact layout / positions / filter sets and oracle
parity on a fixation prefix, plus size-independent properties over
thousands of fixations (determinism, additivity across partitions,
filtered ~ unfiltered)."""

import hashlib

import numpy as np
import pytest

import paper_2601_07571_b200 as gm
import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def room():
    scene, k, fx = W.c2(4096)
    sampled = gm.build_sampled_meshes(scene, k)
    cfg = gm.GenerationConfig(k=k)
    plan = gm.get_plan(scene, sampled, cfg) if hasattr(gm, "get_plan") else None
    from paper_2601_07571_b200.density import get_plan

    plan = get_plan(scene, sampled, cfg)
    return scene, k, fx, sampled, cfg, plan


def test_room_layout_and_positions_bitwise(room):
    scene, k, fx, sampled, cfg, plan = room
    lay = O.build_layouts(scene, k)
    assert sum(v[3] for v in lay.values()) == 2_189_280
    for oid, (res, cnt, off, total) in lay.items():
        np.testing.assert_array_equal(sampled[oid].resolutions, res)
        np.testing.assert_array_equal(sampled[oid].offsets, off)
        assert sampled[oid].total_samples == total
    world = O.world_samples(scene, lay)
    np.testing.assert_array_equal(plan.positions(), np.concatenate([world[o.object_id] for o in scene.objects]))


def test_room_candidate_sets_bitwise(room):
    scene, k, fx, sampled, cfg, plan = room
    pos = plan.positions()
    for filtering in (True, False):
        c = gm.GenerationConfig(k=k, filtering_enabled=filtering)
        got = plan.candidates(fx[:8], c)
        for row, idx in zip(fx[:8], got):
            want = O.candidates(pos, O.fixation_setup(row, c.theta, filtering))
            np.testing.assert_array_equal(idx, want)
            assert len(want) > 0


@pytest.mark.parametrize("filtering", [True, False])
def test_room_values_vs_oracle_prefix(room, filtering):
    scene, k, fx, sampled, cfg, plan = room
    n = 24
    c = gm.GenerationConfig(k=k, filtering_enabled=filtering)
    dm = gm.generate(scene, sampled, fx[:n], c)
    vals, gmax = O.generate(scene, O.rows_as_fixations(fx[:n]), k=k, filtering_enabled=filtering, threads=8,
                            layouts=O.build_layouts(scene, k))
    assert dm.global_max == pytest.approx(gmax, rel=1e-12)
    nz = 0
    for oid in vals:
        np.testing.assert_array_equal(dm.values[oid] != 0, vals[oid] != 0)
        np.testing.assert_allclose(dm.values[oid], vals[oid], rtol=1e-12, atol=0.0)
        nz += int((vals[oid] != 0).sum())
    assert nz > 1000


def _digest(dm):
    h = hashlib.sha256()
    for oid in sorted(dm.values):
        h.update(np.ascontiguousarray(dm.values[oid]).tobytes())
    return h.hexdigest()


def test_room_determinism_and_additivity(room):
    scene, k, fx, sampled, cfg, plan = room
    full = gm.generate(scene, sampled, fx, cfg)
    again = gm.generate(scene, sampled, fx, cfg, batch=333)
    assert _digest(full) == _digest(again)  # checksum determinism (cli bench, gm/cli.py:180-186)
    a = gm.generate(scene, sampled, fx[:1500], cfg)
    b = gm.generate(scene, sampled, fx[1500:], cfg)
    for oid in full.values:
        np.testing.assert_allclose(full.values[oid], a.values[oid] + b.values[oid], rtol=1e-9, atol=1e-12)
    assert full.global_max > 0


def test_room_one_vs_two_streams_bitwise(room):
    """The two-stream batch pipeline keeps every sample's accumulation in log
    order: identical bits to one stream, for several batch sizes."""
    from paper_2601_07571_b200 import _native

    scene, k, fx, sampled, cfg, plan = room
    outs = []
    for flags, batch in ((_native.GM_FLAG_ONE_STREAM, 0), (_native.GM_FLAG_TWO_STREAMS, 0),
                         (_native.GM_FLAG_TWO_STREAMS, 257), (_native.GM_FLAG_ONE_STREAM, 257)):
        plan.accumulate(fx, cfg, reset=True, batch=batch, flags=flags)
        outs.append(plan.read())
    for o in outs[1:]:
        np.testing.assert_array_equal(o.view(np.uint64), outs[0].view(np.uint64))


def test_room_filtered_vs_unfiltered(room):
    """Per fixation, filtering changes nothing but the z-buffer footprint: a
    sample's weight is identical in both paths (same Gaussian, bitwise) unless
    its visibility flips (zero in exactly one path) -- acceptance criterion 6's
    invariant (test_acceptance.py:289-323), checked fixation by fixation."""
    scene, k, fx, sampled, cfg, plan = room
    flips = same = 0
    for row in fx[:12]:
        on = gm.generate(scene, sampled, row[None, :], gm.GenerationConfig(k=k, filtering_enabled=True))
        off = gm.generate(scene, sampled, row[None, :], gm.GenerationConfig(k=k, filtering_enabled=False))
        for oid in on.values:
            x, y = on.values[oid], off.values[oid]
            diff = x != y
            assert np.all((x[diff] == 0.0) | (y[diff] == 0.0))  # every disagreement is a visibility flip
            flips += int(diff.sum())
            same += int(((x == y) & (x != 0)).sum())
    assert same > 0 and flips < 0.2 * same


def test_shells_occlusion_vs_oracle():
    """C5-style nested shells (occlusion-dominated), reduced size."""
    base = W.icosphere(4, 1.0)
    scene = gm.Scene(tuple(gm.SceneObject(f"s{i}", gm.Mesh(base.vertices * (0.5 + 0.25 * i), base.faces))
                           for i in range(6)))
    fx = W.orbit_fixations(16, 4, 3.0, 4.5, jitter=0.3)
    for filtering in (True, False):
        cfg = gm.GenerationConfig(k=4000.0, filtering_enabled=filtering)
        sampled = gm.build_sampled_meshes(scene, cfg.k)
        dm = gm.generate(scene, sampled, fx, cfg)
        vals, gmax = O.generate(scene, O.rows_as_fixations(fx), k=cfg.k, filtering_enabled=filtering, threads=8)
        assert dm.global_max == pytest.approx(gmax, rel=1e-12)
        for oid in vals:
            np.testing.assert_array_equal(dm.values[oid] != 0, vals[oid] != 0)
            np.testing.assert_allclose(dm.values[oid], vals[oid], rtol=1e-12, atol=0.0)
        inner = sum(int((vals[f"s{i}"] != 0).sum()) for i in range(5))
        assert inner == 0  # only the outermost shell is visible


def test_deep_shells_crowded_pass_vs_oracle():
    """16 nested icosphere(3) shells, full frustum: the texel tiles are deep
    (triangle bboxes cover them > 10x), so the z-buffer texels come from the
    sorted crowded pass of k_texels."""
    base = W.icosphere(3, 1.0)
    scene = gm.Scene(tuple(gm.SceneObject(f"s{i}", gm.Mesh(base.vertices * (0.5 + 0.08 * i), base.faces))
                           for i in range(16)))
    fx = W.orbit_fixations(6, 7, 2.6, 3.2, jitter=0.2)
    cfg = gm.GenerationConfig(k=1500.0, filtering_enabled=False)
    sampled = gm.build_sampled_meshes(scene, cfg.k)
    dm = gm.generate(scene, sampled, fx, cfg)
    vals, gmax = O.generate(scene, O.rows_as_fixations(fx), k=cfg.k, filtering_enabled=False, threads=8)
    assert dm.global_max == pytest.approx(gmax, rel=1e-12)
    for oid in vals:
        np.testing.assert_array_equal(dm.values[oid] != 0, vals[oid] != 0)
        np.testing.assert_allclose(dm.values[oid], vals[oid], rtol=1e-12, atol=0.0)


def test_room_staged_readback_roundtrip(room):
    """gm_plan_read streams maps > 8 MiB through two pinned stages (17.5 MB
    here: three chunks, ragged tail): a write -> read round trip returns the
    same bits, and the normalized read equals raw / max bit-for-bit (k_normalize
    divides, like the reference's values / global_max)."""
    scene, k, fx, sampled, cfg, plan = room
    assert plan.n_samples * 8 > 2 * (8 << 20)
    rng = np.random.default_rng(7)
    vals = rng.random(plan.n_samples) * 1e3
    plan.write(vals)
    back = plan.read()
    np.testing.assert_array_equal(back.view(np.uint64), vals.view(np.uint64))
    gmax = float(vals.max())
    np.testing.assert_array_equal(plan.read(normalized_by=gmax).view(np.uint64), (vals / gmax).view(np.uint64))
