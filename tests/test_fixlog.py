"""Fixation-log ingestion against the reference's own
parse_fixation_log outcomes (tests/golden/fixlog_cases.json, written by
tests/golden/make_fixlog_golden.py): parsed values bit-for-bit, same rows
and order, same exception type and message.  Host C++ only: runs on CPU."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2601_07571_b200 as gm
from paper_2601_07571_b200 import fixlog

CASES = json.loads((Path(__file__).resolve().parent / "golden" / "fixlog_cases.json").read_text())


def _rows(fx):
    out = []
    for f in fx:
        vals = [f.start_time, f.duration, *f.camera_position, *f.camera_rotation, *f.frustum, *f.gaze_dir]
        ov = {k: [float(x).hex() for x in (*t.translation, *t.rotation, *t.scale)] for k, t in f.overrides.items()}
        out.append({"v": [float(x).hex() for x in vals], "ov": ov})
    return out


@pytest.mark.parametrize("case", CASES, ids=[f"{c['name']}-{c['window']}" for c in CASES])
def test_matches_reference(case, tmp_path):
    p = tmp_path / f"{case['name']}.log"
    p.write_bytes(case["text"].encode("utf-8"))
    window = tuple(case["window"]) if case["window"] else None
    exp = case["expect"]
    if "error" in exp:
        with pytest.raises(Exception) as ei:
            gm.parse_fixation_log(p, window)
        assert type(ei.value).__name__ == exp["error"]
        assert str(ei.value).replace(str(p), "{path}") == exp["message"]
        with pytest.raises(type(ei.value)):
            gm.parse_fixation_table(p, window)
    else:
        fx = gm.parse_fixation_log(p, window)
        assert _rows(fx) == exp["rows"]
        table = gm.parse_fixation_table(p, window)
        assert table.shape == (len(exp["rows"]), 18)
        want = np.array([[float.fromhex(x) for x in r["v"]] for r in exp["rows"]]).reshape(-1, 18)
        np.testing.assert_array_equal(table.view(np.uint64), want.view(np.uint64))
        if not exp["rows"]:
            assert fx == []


def test_table_is_the_generate_input(tmp_path):
    case = next(c for c in CASES if c["name"] == "room_stream" and c["window"] is None)
    p = tmp_path / "room.log"
    p.write_bytes(case["text"].encode())
    fx = gm.parse_fixation_log(p)
    assert isinstance(fx, list) and isinstance(fx, gm.FixationLog)
    assert gm.fixation_table(fx) is fx.table
    np.testing.assert_array_equal(fx.table, np.array([f.row() for f in fx]))


def test_multithreaded_chunks_line_numbers(tmp_path):
    """> 1 MiB logs are split across threads at line boundaries: rows, order
    and the line number of a late error must not depend on the split."""
    import workloads as W

    fx = W.room_fixations(12000, seed=9)
    lines = []
    for i, r in enumerate(fx):
        lines.append(" ".join(repr(float(v)) for v in r))
        if i % 500 == 0:
            lines.append("# c")
    p = tmp_path / "big.log"
    p.write_bytes(("\r\n".join(lines) + "\r\n").encode())
    assert p.stat().st_size > (1 << 20)
    t1 = fixlog.parse_fixation_table(p, threads=1)
    t8 = fixlog.parse_fixation_table(p, threads=8)
    np.testing.assert_array_equal(t1.view(np.uint64), t8.view(np.uint64))
    assert len(t1) == 12000
    bad = list(lines)
    bad[10000] = bad[10000].replace(" ", " q", 1)
    p.write_bytes(("\n".join(bad) + "\n").encode())
    for th in (1, 3, 8):
        with pytest.raises(gm.ParseError, match="line 10001: bad numeric field"):
            fixlog.parse_fixation_table(p, threads=th)


def _log_text(n):
    lines = ["# start dur px py pz qx qy qz qw l r t b n f gx gy gz"]
    for i in range(n):
        lines.append(f"{0.25 * i} {0.1 + 0.01 * i} {0.1 * i} 1.5 2.0 0 0 0 1 -0.1 0.1 0.1 -0.1 0.1 100 "
                     f"{0.01 * i} 0.02 -1")
    return "\n".join(lines) + "\n"


def test_in_place_edits_invalidate_cached_table(tmp_path):
    # FixationLog caches the parsed (F, 18) table; list edits must not leave it stale
    p = tmp_path / "f.log"
    p.write_text(_log_text(6))
    log = gm.parse_fixation_log(p)
    rows = [f.row() for f in log]
    np.testing.assert_array_equal(gm.fixation_table(log), np.array(rows))
    log.reverse()
    np.testing.assert_array_equal(gm.fixation_table(log), np.array(rows[::-1]))
    log[0] = log[1]
    np.testing.assert_array_equal(gm.fixation_table(log)[0], rows[::-1][1])
    for edit in (lambda L: L.sort(key=lambda f: f.duration), lambda L: L.append(L[0]), lambda L: L.pop(),
                 lambda L: L.insert(2, L[3]), lambda L: L.__delitem__(0), lambda L: L.extend(L[:2])):
        fresh = gm.parse_fixation_log(p)
        edit(fresh)
        np.testing.assert_array_equal(gm.fixation_table(fresh), np.array([f.row() for f in fresh]))
    again = gm.parse_fixation_log(p)
    again += again[:1]
    assert isinstance(again, fixlog.FixationLog) and len(again) == 7
    np.testing.assert_array_equal(gm.fixation_table(again), np.array([f.row() for f in again]))


def test_overrides_placed_into_parsed_log_are_seen(tmp_path):
    from paper_2601_07571_b200.density import _override_list

    p = tmp_path / "f.log"
    p.write_text(_log_text(3))
    log = gm.parse_fixation_log(p)
    assert _override_list(log) is None
    f0 = log[0]
    moved = gm.Fixation(f0.start_time, f0.duration, f0.camera_position, f0.camera_rotation, f0.frustum, f0.gaze_dir,
                        overrides={"a": gm.Transform([1.0, 0.0, 0.0], [0, 0, 0, 1], [1, 1, 1])})
    log[0] = moved
    ovs = _override_list(log)
    assert ovs is not None and ovs[0] is moved.overrides
