"""Dynamic scenes: per-fixation pose overrides on the GPU
path against the reference's own generate() (tests/golden/dynamic.npz, from
tests/golden/make_dynamic_golden.py): identical contributing-sample sets and
values to 1e-12 relative, global max, filtering on and off."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_2601_07571_b200 as gm

pytestmark = pytest.mark.gpu
RTOL = 1e-12
G = dict(np.load(Path(__file__).resolve().parent / "golden" / "dynamic.npz"))


def _scene():
    ids = [str(x) for x in G["ids"]]
    objs = []
    for i, oid in enumerate(ids):
        t = G[f"t{i}"]
        objs.append(gm.SceneObject(oid, gm.Mesh(G[f"v{i}"], G[f"f{i}"]), gm.Transform(t[0:3], t[3:7], t[7:10])))
    return gm.Scene(tuple(objs)), ids


def _fixations(ids):
    out = []
    for f, row in enumerate(G["fix"]):
        ov = {}
        for ff, oi, v in zip(G["spec_f"], G["spec_o"], G["spec_v"]):
            if ff == f:
                ov[ids[oi] if oi >= 0 else "not_in_scene"] = gm.Transform(v[0:3], v[3:7], v[7:10])
        out.append(gm.Fixation(row[0], row[1], row[2:5], row[5:9], tuple(row[9:15]), row[15:18], overrides=ov))
    return out


@pytest.mark.parametrize("filtering", [True, False])
@pytest.mark.parametrize("batch", [0, 3])
def test_dynamic_vs_reference(filtering, batch):
    scene, ids = _scene()
    fx = _fixations(ids)
    tag = "on" if filtering else "off"
    cfg = gm.GenerationConfig(k=float(G["k"]), filtering_enabled=filtering)
    sm = gm.build_sampled_meshes(scene, cfg.k)
    dm = gm.generate(scene, sm, fx, cfg, batch=batch)
    assert dm.global_max == pytest.approx(float(G[f"gmax_{tag}"]), rel=RTOL)
    for i, oid in enumerate(ids):
        want = G[f"val_{tag}{i}"]
        got = dm.values[oid]
        assert np.array_equal(got != 0, want != 0), oid
        np.testing.assert_allclose(got, want, rtol=RTOL, atol=0)


def test_dynamic_accumulate_fixation_and_plan_restored():
    """accumulate_fixation honours one fixation's overrides, and the cached
    plan is back at the base poses afterwards (a static generate after a
    dynamic one equals a fresh static generate)."""
    scene, ids = _scene()
    fx = _fixations(ids)
    cfg = gm.GenerationConfig(k=float(G["k"]))
    sm = gm.build_sampled_meshes(scene, cfg.k)
    static = [gm.Fixation(f.start_time, f.duration, f.camera_position, f.camera_rotation, f.frustum, f.gaze_dir)
              for f in fx]
    want_static = gm.generate(scene, sm, static, cfg)
    dyn = gm.generate(scene, sm, fx, cfg)
    again = gm.generate(scene, sm, static, cfg)
    for oid in ids:
        np.testing.assert_array_equal(again.values[oid], want_static.values[oid])
    dm = gm.DensityMap({oid: np.zeros(sm[oid].total_samples) for oid in ids}, 0.0, False)
    for f in fx:
        gm.accumulate_fixation(dm, scene, sm, f, cfg)
    for oid in ids:
        np.testing.assert_allclose(dm.values[oid], dyn.values[oid], rtol=RTOL, atol=0)


def test_dynamic_log_roundtrip(tmp_path):
    """The same dynamic session written as a fixation log (pose-override groups,
    gaze.py:130-188 schema), parsed by the C++ ingestion, generated on the GPU."""
    scene, ids = _scene()
    lines = ["# dynamic session"]
    for f, row in enumerate(G["fix"]):
        toks = [repr(float(v)) for v in row]
        for ff, oi, v in zip(G["spec_f"], G["spec_o"], G["spec_v"]):
            if ff == f:
                toks.append(ids[oi] if oi >= 0 else "not_in_scene")
                toks.extend(repr(float(x)) for x in v)
        lines.append(" ".join(toks))
    p = tmp_path / "dyn.log"
    p.write_text("\n".join(lines) + "\n")
    fx = gm.parse_fixation_log(p)
    assert len(fx) == len(G["fix"]) and sum(bool(f.overrides) for f in fx) == len(set(G["spec_f"].tolist()))
    cfg = gm.GenerationConfig(k=float(G["k"]))
    sm = gm.build_sampled_meshes(scene, cfg.k)
    dm = gm.generate(scene, sm, fx, cfg)
    for i, oid in enumerate(ids):
        np.testing.assert_allclose(dm.values[oid], G[f"val_on{i}"], rtol=RTOL, atol=0)
