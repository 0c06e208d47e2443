"""Export / persistence wire formats against the reference's
own bytes (tests/golden/export.npz, from tests/golden/make_export_golden.py).

CPU tests drive the C++ record formatter with positions from the C oracle
(bit-exact restatement of sample_positions_local / Transform.apply); the GPU
test runs the public write_export end to end (positions from k_positions)."""

from __future__ import annotations

import zlib
from pathlib import Path

import numpy as np
import pytest

import paper_2601_07571_b200 as gm
import workloads as W
from oracle import oracle as O
from paper_2601_07571_b200 import io_export

G = dict(np.load(Path(__file__).resolve().parent / "golden" / "export.npz"))
CSV = zlib.decompress(G["csv"].tobytes())
CSV_SUB = zlib.decompress(G["csv_sub"].tobytes())
MAP = zlib.decompress(G["map"].tobytes())


def _setup():
    scene = W.rotated_object_scene()
    ids = [str(x) for x in G["ids"]]
    values = {oid: G[f"val{i}"] for i, oid in enumerate(ids)}
    return scene, ids, gm.DensityMap(values, global_max=12.5, normalized=False)


def _layout(obj, k):
    tri = obj.mesh.vertices[obj.mesh.faces].reshape(-1, 9)
    res, cnt, off, total = O.layout(tri, k)
    sm = gm.SampledMesh(obj.object_id, res, cnt, off, int(total), k)
    local = O.positions_local(tri, res, cnt, off, total)
    t = obj.transform
    world = O.transform_apply(local, t.translation, t.rotation, t.scale)
    return sm, local, world


def test_formatter_matches_reference_bytes():
    scene, ids, dm = _setup()
    k = float(G["k"])
    out = [b"# world positions use each object's static base pose\n", (io_export.EXPORT_HEADER + "\n").encode()]
    for oid in sorted(ids):
        sm, local, world = _layout(scene.object(oid), k)
        out.append(io_export._format_records(oid, sm, local, world, dm.values[oid]))
    assert b"".join(out) == CSV


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_formatter_thread_count_invariant(threads):
    scene, ids, dm = _setup()
    sm, local, world = _layout(scene.object("cube"), float(G["k"]))
    a = io_export._format_records("cube", sm, local, world, dm.values["cube"], threads=1)
    b = io_export._format_records("cube", sm, local, world, dm.values["cube"], threads=threads)
    assert a == b


def test_save_map_bytes_and_roundtrip(tmp_path):
    _, ids, dm = _setup()
    p = tmp_path / "m.gzm"
    gm.save_map(dm, p, "abc123", float(G["k"]))
    assert p.read_bytes() == MAP
    back, header = gm.load_map(p, expect_layout_hash="abc123")
    assert header["magic"] == "GAZEMAP1" and back.global_max == 12.5 and not back.normalized
    for oid in ids:
        np.testing.assert_array_equal(back.values[oid].view(np.uint64), dm.values[oid].view(np.uint64))
    with pytest.raises(gm.LayoutMismatchError):
        gm.load_map(p, expect_layout_hash="other")
    bad = tmp_path / "bad.gzm"
    bad.write_bytes(MAP[:-8])
    with pytest.raises(gm.ParseError, match="truncated"):
        gm.load_map(bad)


@pytest.mark.gpu
def test_write_export_gpu_matches_reference(tmp_path):
    scene, ids, dm = _setup()
    sm = gm.build_sampled_meshes(scene, float(G["k"]))
    p = tmp_path / "e.csv"
    n = gm.write_export(dm, scene, sm, p)
    assert n == int(G["count"])
    assert p.read_bytes() == CSV
    n2 = gm.write_export(dm, scene, sm, tmp_path / "s.csv", objects=["plane", "cube"])
    assert (tmp_path / "s.csv").read_bytes() == CSV_SUB
    assert n2 == sum(sm[o].total_samples for o in ("plane", "cube"))
