"""Host-side logic of the drop-in API (CPU only): validation, data model,
scalar helpers and their reference KATs (pkg/tests/test_geometry.py,
test_gaze.py, test_density.py)."""

import math

import numpy as np
import pytest

import paper_2601_07571_b200 as gm


class TestConfigValidation:
    def test_defaults_valid(self):
        gm.GenerationConfig().validate()

    @pytest.mark.parametrize("kw", [{"k": 0.0}, {"k": -1.0}, {"theta": 0.0}, {"theta": math.pi / 2},
                                    {"zbuffer_resolution": 0}, {"epsilon_abs": -1e-3}, {"epsilon_rel": -1e-3},
                                    {"time_window": (5.0, 1.0)}])
    def test_rejects(self, kw):
        with pytest.raises(gm.ConfigError):
            gm.GenerationConfig(**kw).validate()

    def test_cone(self):
        c = gm.GenerationConfig(theta=0.05).cone()
        assert c.sigma == math.tan(0.05) and c.phi == math.atan(4.0 * c.sigma)


class TestDataModel:
    def test_transform_validation(self):
        with pytest.raises(ValueError):
            gm.Transform([0, 0], [0, 0, 0, 1], [1, 1, 1])
        with pytest.raises(ValueError):
            gm.Transform([0, 0, 0], [0, 0, 0, 2], [1, 1, 1])
        t = gm.Transform([1, 2, 3], [0, 0, 0, 1], [1, 1, 1])
        np.testing.assert_array_equal(t.apply(np.zeros((1, 3))), [[1, 2, 3]])

    def test_mesh_face_range(self):
        with pytest.raises(ValueError):
            gm.Mesh(np.zeros((3, 3)), [[0, 1, 3]])

    def test_scene_unique_ids(self):
        m = gm.Mesh(np.eye(3), [[0, 1, 2]])
        with pytest.raises(ValueError):
            gm.Scene((gm.SceneObject("a", m), gm.SceneObject("a", m)))
        s = gm.Scene((gm.SceneObject("a", m),))
        assert s.object_ids == ["a"] and s.object("a").mesh is m
        with pytest.raises(KeyError):
            s.object("b")

    def test_fixation_validation_and_row(self):
        fr = (-0.1, 0.1, 0.1, -0.1, 0.1, 100.0)
        f = gm.Fixation(1.0, 0.5, [1, 2, 3], [0, 0, 0, 1], fr, [0.0, 0.0, -2.0])
        np.testing.assert_array_equal(f.gaze_dir, [0, 0, -1])
        row = f.row()
        assert row.shape == (18,) and row[1] == 0.5 and tuple(row[9:15]) == fr
        np.testing.assert_array_equal(gm.fixation_table([f])[0], row)
        for bad in (dict(duration=0.0), dict(gaze_dir=[0, 0, 1.0]), dict(gaze_dir=[0, 0, 0.0]),
                    dict(frustum=(0.1, -0.1, 0.1, -0.1, 0.1, 100)), dict(frustum=(-0.1, 0.1, 0.1, -0.1, 0, 100))):
            kw = dict(start_time=0.0, duration=1.0, camera_position=[0, 0, 0], camera_rotation=[0, 0, 0, 1],
                      frustum=fr, gaze_dir=[0, 0, -1.0])
            kw.update(bad)
            with pytest.raises(ValueError):
                gm.Fixation(**kw)

    def test_fixation_table_passthrough(self):
        t = np.zeros((3, 18))
        assert gm.fixation_table(t) is not None and gm.fixation_table(t).shape == (3, 18)
        with pytest.raises(ValueError):
            gm.fixation_table(np.zeros((3, 17)))

    def test_density_map(self):
        sm = {"a": gm.SampledMesh("a", np.ones(1, np.int64), np.full(1, 3, np.int64), np.zeros(1, np.int64), 3, 1.0)}
        d = gm.DensityMap.zeros(sm)
        assert d.total_samples == 3 and d.global_max == 0.0 and not d.normalized
        c = d.copy()
        c.values["a"][0] = 1.0
        assert d.values["a"][0] == 0.0

    def test_timings(self):
        t = gm.Timings()
        t.add("cull", 0.5)
        t.add("cull", 0.25)
        t.add("x", 1.0)
        assert t.phases["cull"] == 0.75 and t.phases["x"] == 1.0


class TestScalarHelpers:
    def test_triangle_area(self):
        assert gm.triangle_area((0, 0, 0), (1, 0, 0), (0, 1, 0)) == pytest.approx(0.5)
        assert gm.triangle_area((0, 0, 0), (2, 0, 0), (1, 0, 0)) == 0.0
        assert gm.triangle_area((0, 0, 0), (1, 0, 0), (0.5, 0.866025, 0)) == pytest.approx(0.433013, abs=1e-6)

    def test_adaptive_resolution_kats(self):
        assert gm.adaptive_resolution(0.5, 6) == 1
        assert gm.adaptive_resolution(0.0, 40000) == 1
        assert gm.adaptive_resolution(0.01, 10000) == 13
        assert gm.sample_count(13) / 0.01 >= 10000
        with pytest.raises(gm.ConfigError):
            gm.adaptive_resolution(1.0, 0)

    @pytest.mark.parametrize("idx,expected", [(0, (0, 0)), (3, (2, 0)), (5, (2, 2))])
    def test_rowcol_kats(self, idx, expected):
        assert gm.sample_index_to_rowcol(idx) == expected

    def test_rowcol_roundtrip(self):
        idx = 0
        for row in range(101):
            for col in range(row + 1):
                assert gm.sample_index_to_rowcol(idx) == (row, col)
                idx += 1
        with pytest.raises(IndexError):
            gm.sample_index_to_rowcol(-1)

    def test_barycentric(self):
        assert gm.rowcol_to_barycentric(0, 0, 2) == (0.0, 0.0, 1.0)
        assert gm.rowcol_to_barycentric(2, 2, 2) == (1.0, 0.0, 0.0)
        assert gm.rowcol_to_barycentric(2, 0, 2) == (0.0, 1.0, 0.0)
        assert gm.rowcol_to_barycentric(1, 0, 2) == pytest.approx((0.0, 0.5, 0.5))
        with pytest.raises(IndexError):
            gm.rowcol_to_barycentric(3, 0, 2)

    def test_gaussian_weight(self):
        cone = gm.GazeCone.from_theta(0.05)
        g = np.array([0.0, 0.0, -1.0])
        on = gm.gaussian_weight([0.0, 0.0, -3.0], g, 1.0, cone)
        assert on == pytest.approx(1.0 / (cone.sigma * math.sqrt(2 * math.pi)), rel=1e-12)
        one = gm.gaussian_weight([3.0 * cone.sigma, 0.0, -3.0], g, 1.0, cone)
        assert one == pytest.approx(on * math.exp(-0.5), rel=1e-12)
        assert gm.gaussian_weight([1.0, 0.0, -1.0], g, 1.0, cone) == 0.0
        assert gm.gaussian_weight([0.0, 0.0, 1.0], g, 1.0, cone) == 0.0

    def test_perspective_roundtrip(self):
        P = gm.perspective_matrix(-0.2, 0.1, -0.05, 0.15, 0.1, 100.0)
        l, r, b, t, n, f = gm.frustum_from_matrix(P)
        for got, want in zip((l, r, b, t, n, f), (-0.2, 0.1, -0.05, 0.15, 0.1, 100.0)):
            assert got == pytest.approx(want, rel=1e-9)
        with pytest.raises(gm.InvalidFrustumError):
            gm.perspective_matrix(0.1, -0.1, -0.1, 0.1, 0.1, 100)
        with pytest.raises(gm.InvalidFrustumError):
            gm.perspective_matrix(-0.1, 0.1, -0.1, 0.1, 0.0, 100)


def test_estimator_params_roundtrip():
    est = gm.FixationDensityMapper(k=1234.0)
    assert est.get_params()["k"] == 1234.0
    est.set_params(k=5678.0)
    assert est.k == 5678.0
    with pytest.raises(ValueError):
        est.fit([])


def test_error_hierarchy():
    for e in (gm.ConfigError, gm.ParseError, gm.GazeOutsideFrustumError, gm.InvalidFrustumError,
              gm.LayoutMismatchError):
        assert issubclass(e, gm.GazemapError)
    pe = gm.ParseError("bad", path="x.txt", line=3)
    assert str(pe) == "x.txt: line 3: bad" and pe.line == 3
