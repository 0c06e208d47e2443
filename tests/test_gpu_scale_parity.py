"""Values parity at benchmark scale: windows of the real bench streams
(bench.workload: C2 on/off, C3 k=30k and k=100k, the C4 session stream, full
C5), each generated on its own through the drop-in API and compared with the
CPU oracle (oracle/gm_oracle.c, pinned bit-exact to the reference by
tests/test_oracle_golden.py) on the same inputs.

Bar (BASELINE north star): values within 1e-5 relative / 1e-7 absolute, the
contributing sample set exact.  Held here: contributing sets identical,
values within rtol 1e-12 (the only non-bit-exact operation on the path is CUDA
exp() vs glibc exp(), <= 1 ulp per contribution), global max within 1e-12.

Reference: density.py:203-227 (generate), kernels.py:219-340 (accumulate,
depth_match).  Windows come from the start, the middle and the end of each
stream; every window is a separate generate() call (not a prefix run).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2601_07571_b200 as gm
import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu

THREADS = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
_CACHE: dict = {}


def _room():
    if "room" not in _CACHE:
        _CACHE["room"] = W.room_scene()
    return _CACHE["room"]


def _stream(name):
    """The bench's fixation streams (bench.workload, rank 0)."""
    if name not in _CACHE:
        scene = _room()
        if name == "c2":
            _CACHE[name] = W.room_fixations(100_000, seed=1, scene=scene)
        elif name == "c3":
            _CACHE[name] = W.room_fixations(10_000, seed=1, scene=scene)
        elif name == "c5":
            _CACHE[name] = W.orbit_fixations(50_000, 4, 4.5, 6.0, jitter=0.3)
    return _CACHE[name]


def _layout(scene, k, key):
    key = ("layout", key)
    if key not in _CACHE:
        _CACHE[key] = (gm.build_sampled_meshes(scene, k), O.build_layouts(scene, k))
    return _CACHE[key]


def _check(scene, k, table, filtering, key):
    sampled, lay = _layout(scene, k, key)
    cfg = gm.GenerationConfig(k=k, filtering_enabled=filtering)
    dm = gm.generate(scene, sampled, table, cfg)
    want, gmax = O.generate(scene, O.rows_as_fixations(table), k=k, filtering_enabled=filtering, threads=THREADS,
                            layouts=lay)
    assert gmax > 0
    assert dm.global_max == pytest.approx(gmax, rel=1e-12, abs=0)
    contributing = 0
    for oid, v in want.items():
        got = dm.values[oid]
        np.testing.assert_array_equal(got != 0, v != 0, err_msg=f"contributing set of {oid}")
        np.testing.assert_allclose(got, v, rtol=1e-12, atol=0.0, err_msg=oid)
        contributing += int((v != 0).sum())
    return contributing


C2_WINDOWS = [(0, 500), (50_000, 50_500), (99_500, 100_000)]


@pytest.mark.parametrize("filtering", [True, False], ids=["filtered", "unfiltered"])
@pytest.mark.parametrize("window", C2_WINDOWS, ids=["start", "middle", "end"])
def test_c2_stream_windows(window, filtering):
    a, b = window
    n = _check(_room(), 10_000.0, _stream("c2")[a:b], filtering, "c2")
    assert n > 10_000


C3_WINDOWS = [(0, 500), (5_000, 5_500), (9_500, 10_000)]


@pytest.mark.parametrize("k", [30_000.0, 100_000.0], ids=["k30k", "k100k"])
@pytest.mark.parametrize("window", C3_WINDOWS, ids=["start", "middle", "end"])
def test_c3_density_sweep_windows(window, k):
    a, b = window
    n = _check(_room(), k, _stream("c3")[a:b], True, f"c3-{k}")
    assert n > 10_000


# C4: 50 users x 20k; windows = start of user 0, the user 24 -> 25 boundary
# (fixations 499,900 .. 500,100 of the 1M stream), the end of user 49
C4_WINDOWS = [(0, 1, 0, 200), (24, 2, 19_900, 20_100), (49, 1, 19_800, 20_000)]


@pytest.mark.parametrize("first,users,a,b", C4_WINDOWS, ids=["start", "user-boundary", "end"])
def test_c4_session_windows(first, users, a, b):
    table = W.session_fixations(users=users, first_user=first, scene=_room())[a:b]
    n = _check(_room(), 10_000.0, table, True, "c2")
    assert n > 5_000


@pytest.mark.parametrize("window", [(0, 200), (49_800, 50_000)], ids=["start", "end"])
def test_c5_nested_shells_windows(window):
    """Full C5: 12 icosphere(6) shells, 983,040 occluders, 15.5 M samples."""
    if "shells" not in _CACHE:
        _CACHE["shells"] = W.shells_scene()
    scene = _CACHE["shells"]
    a, b = window
    n = _check(scene, 20_000.0, _stream("c5")[a:b], True, "c5")
    assert n > 10_000
    dm_inner = gm.generate(scene, _layout(scene, 20_000.0, "c5")[0], _stream("c5")[a:a + 8],
                           gm.GenerationConfig(k=20_000.0))
    assert all(not np.any(dm_inner.values[f"shell{i}"]) for i in range(11))  # only the outer shell is seen


def test_c4_session_stream_is_sharded_by_user():
    """The C4 generator yields user u's stream independently of the others
    (bench shards the 1M stream by contiguous ranges; tests take windows)."""
    full = W.session_fixations(users=3, per_user=500, scene=_room())
    part = W.session_fixations(users=1, per_user=500, scene=_room(), first_user=1)
    np.testing.assert_array_equal(full[500:1000], part)


# ------------------------------------------------------------ self-check build

def _check_build_run(*args):
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    so = root / "paper_2601_07571_b200" / "_gazemap_b200_check.so"
    assert so.exists(), "GM_CHECK variant missing: run __graft_entry__.build()"
    env = dict(os.environ, GAZEMAP_B200_SO=str(so))
    r = subprocess.run([sys.executable, str(root / "tools" / "check_run.py"), *args], env=env,
                       capture_output=True, text=True, timeout=900)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert line, r.stdout + r.stderr
    return json.loads(line[-1])


@pytest.mark.parametrize("args", [("--config", "c2", "--fixations", "2048"),
                                  ("--config", "c2", "--fixations", "1024", "--start", "60000", "--unfiltered"),
                                  ("--config", "c5", "--fixations", "256"),
                                  ("--config", "c3k100", "--fixations", "512", "--start", "4000")],
                         ids=["c2", "c2-unfiltered", "c5", "c3k100"])
def test_check_build_finds_no_violation(args):
    """The GM_CHECK build re-does every float32-bound and conservative-cull
    decision in exact float64 on the device (texel bounds and winners, level-1
    / level-3 candidate culls, the 3x3 texel marks, every depth test and the
    tile-max occlusion shortcut) and counts disagreements: all must be 0."""
    res = _check_build_run(*args)
    c = res["counters"]
    assert c["tx_texels"] > 0 and c["cand_pairs"] > 0 and c["depth_tests"] > 0
    assert res["violations"] == 0, res


def test_segment_overflow_resume_is_bitwise():
    """Screen-triangle segments that overflow mid-pass: the host grows them
    and resumes from the failed batch (run_batches); the map is bit-identical
    to a run that never overflowed, and the retry is reported."""
    from paper_2601_07571_b200 import _native
    from paper_2601_07571_b200.density import ScenePlan

    scene = _room()
    k = 10_000.0
    sampled, _ = _layout(scene, k, "c2")
    table = _stream("c2")[20_000:20_768]
    cfg = gm.GenerationConfig(k=k)
    ids = [o.object_id for o in scene.objects]
    ref = ScenePlan(scene, sampled, ids)
    ref.accumulate(table, cfg, reset=True, batch=128)
    want = ref.read()
    assert ref.last_timings.retries == 0
    plan = ScenePlan(scene, sampled, ids)
    _native.check(plan._lib.gm_plan_set_segment_capacity(plan._h, 48))
    plan.accumulate(table, cfg, reset=True, batch=128)
    assert plan.last_timings.retries >= 1
    np.testing.assert_array_equal(plan.read().view(np.uint64), want.view(np.uint64))


def test_production_build_reports_no_check_counters():
    import ctypes

    from paper_2601_07571_b200 import _native, density

    scene = _room()
    sampled, _ = _layout(scene, 10_000.0, "c2")
    plan = density.get_plan(scene, sampled, gm.GenerationConfig(k=10_000.0), 0)
    out = (ctypes.c_uint64 * len(_native.CHECK_NAMES))()
    flag = ctypes.c_int(-1)
    _native.check(plan._lib.gm_plan_check(plan._h, out, 0, ctypes.byref(flag)))
    if os.environ.get("GAZEMAP_B200_SO", "").endswith("_check.so"):
        assert flag.value == 1
    else:
        assert flag.value == 0 and not any(out)
