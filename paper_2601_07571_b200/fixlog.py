"""Fixation-log ingestion: drop-in for the reference's
`parse_fixation_log` (gazemap/gaze.py:130-188).

The line parser runs in C++ (csrc/gm_fixlog.cpp, multi-threaded over
line-aligned chunks) and returns the whole (F, 18) fixation table at once --
the layout the C-ABI's generation entry points take -- with each row's
Fixation validation verdict and its pose-override groups.  This module
applies the time window and raises the reference's ParseError for the first
failing line in file order; the message of a line the C++ scanner rejected is
produced by re-running the reference's per-line logic on that one line
(`_parse_line`), so the error text is the reference's own.  Files with
non-ASCII bytes (Unicode whitespace and digits have Python-specific meaning)
are parsed by `_parse_line` throughout.

`parse_fixation_log` returns a `FixationLog`: a list of Fixation objects (as
the reference returns) that also carries `.table`, so `generate` skips the
per-object conversion.  `parse_fixation_table` returns only the table.
"""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np

from . import _native
from .errors import ParseError
from .gaze import FIX_COLUMNS, Fixation
from .geometry import Transform

__all__ = ["FixationLog", "parse_fixation_log", "parse_fixation_table"]

_K_NON_ASCII = 5
_VALIDATION_MESSAGES = {
    1: "gaze_dir must be a nonzero vector",
    2: "duration must be > 0",
    3: "frustum needs 0 < near < far",
    4: "frustum needs left < right and bottom < top",
    5: "gaze_dir must point into the viewed half-space (z < 0)",
}
_SPLIT = re.compile(r"[,\s]+")


class FixationLog(list):
    """list[Fixation] in log order plus `.table` ((F, 18) float64, gaze
    normalised) and `.line` (1-based source line of each fixation)."""

    table: np.ndarray
    line: np.ndarray

    @property
    def has_overrides(self) -> bool:
        return any(f.overrides for f in self)

    def _stale(self) -> None:
        # the cached table / line numbers / override count describe the list as
        # parsed; any in-place edit makes consumers rebuild from the Fixation objects
        for name in ("table", "line", "n_override_groups"):
            self.__dict__.pop(name, None)


def _invalidating(name: str):
    base = getattr(list, name)

    def method(self, *args, **kwargs):
        self._stale()
        return base(self, *args, **kwargs)

    method.__name__ = name
    method.__doc__ = base.__doc__
    return method


for _name in ("__setitem__", "__delitem__", "__iadd__", "__imul__", "append", "extend", "insert", "pop", "remove",
              "clear", "sort", "reverse"):
    setattr(FixationLog, _name, _invalidating(_name))
del _name


def _parse_line(raw: str, path, ln: int):
    """One line of the reference loop (gaze.py:148-185): None for blank and
    header lines, else (18 floats, overrides dict); raises ParseError (or the
    reference's IndexError for a separators-only line)."""
    line = raw.split("#", 1)[0].strip()
    if not line:
        return None
    tokens = [t for t in _SPLIT.split(line) if t]
    try:
        float(tokens[0])
    except ValueError:
        return None
    if len(tokens) < 18:
        raise ParseError(f"expected at least 18 fields, got {len(tokens)}", path, ln)
    try:
        vals = [float(t) for t in tokens[:18]]
    except ValueError as e:
        raise ParseError(f"bad numeric field: {e}", path, ln)
    overrides = {}
    rest = tokens[18:]
    if len(rest) % 11 != 0:
        raise ParseError("pose override groups must be (object_id + 10 floats)", path, ln)
    for g in range(0, len(rest), 11):
        oid = rest[g]
        try:
            nums = [float(t) for t in rest[g + 1:g + 11]]
            overrides[oid] = Transform(np.array(nums[0:3]), np.array(nums[3:7]), np.array(nums[7:10]))
        except ValueError as e:
            raise ParseError(f"bad pose override for {oid!r}: {e}", path, ln)
    return vals, overrides


def _fixation(vals, overrides) -> Fixation:
    return Fixation(start_time=vals[0], duration=vals[1], camera_position=np.array(vals[2:5]),
                    camera_rotation=np.array(vals[5:9]), frustum=tuple(vals[9:15]),
                    gaze_dir=np.array(vals[15:18]), overrides=overrides)


def _parse_python(path, time_window) -> FixationLog:
    """The reference algorithm line by line (non-ASCII files)."""
    t0, t1 = (None, None) if time_window is None else time_window
    out, lines = [], []
    with open(path, "r") as fh:
        for ln, raw in enumerate(fh, start=1):
            r = _parse_line(raw, path, ln)
            if r is None:
                continue
            vals, overrides = r
            start = vals[0]
            if t0 is not None and not (t0 <= start < t1):
                continue
            try:
                out.append(_fixation(vals, overrides))
            except ValueError as e:
                raise ParseError(str(e), path, ln)
            lines.append(ln)
    log = FixationLog(out)
    log.table = np.array([f.row() for f in out], dtype=np.float64).reshape(-1, FIX_COLUMNS)
    log.line = np.asarray(lines, dtype=np.int64)
    return log


def _scan(data: bytes, threads: int = 0):
    lib = _native.load()
    h = ctypes.c_void_p()
    buf = ctypes.c_char_p(data)
    _native.check(lib.gm_fixlog_parse(buf, len(data), int(threads), ctypes.byref(h)), "gm_fixlog_parse")
    try:
        info = np.zeros(7, np.int64)
        lib.gm_fixlog_error(h, _native.iptr(info))
        R = int(lib.gm_fixlog_rows(h))
        G = int(lib.gm_fixlog_groups(h))
        table = np.empty((R, FIX_COLUMNS))
        line = np.empty(R, np.int64)
        code = np.empty(R, np.int32)
        gstart = np.empty(R + 1, np.int64)
        goid = np.empty((max(G, 1), 2), np.int64)
        gvals = np.empty((max(G, 1), 10))
        lib.gm_fixlog_copy(h, _native.dptr(table), _native.iptr(line), code.ctypes.data_as(ctypes.c_void_p),
                           _native.iptr(gstart), _native.iptr(goid), _native.dptr(gvals))
    finally:
        lib.gm_fixlog_free(h)
    return info, table, line, code, gstart, goid[:G], gvals[:G]


def _read(path, time_window, threads):
    path = Path(path)
    data = path.read_bytes()
    info, table, line, code, gstart, goid, gvals = _scan(data, threads)
    if int(info[0]) == _K_NON_ASCII:
        return None, path
    R = len(table)
    err_line = int(info[1]) if info[0] else None
    # time window (gaze.py:171-173), applied after the override groups are built
    if time_window is None:
        inwin = np.ones(R, bool)
    else:
        t0, t1 = time_window
        start = table[:, 0]
        inwin = (t0 <= start) & (start < t1)
    bad_v = np.nonzero(inwin & (code != 0))[0]
    v_row = int(bad_v[0]) if len(bad_v) else None
    # pose overrides (gaze.py:160-170): Transform validation in file order,
    # before the row's window check and Fixation validation
    ngroups = np.diff(gstart)
    overrides = [None] * R
    limit = R if v_row is None else v_row + 1
    for r in np.nonzero(ngroups[:limit])[0]:
        d = {}
        for g in range(int(gstart[r]), int(gstart[r + 1])):
            oid = data[goid[g, 0]:goid[g, 0] + goid[g, 1]].decode("ascii")
            nums = gvals[g]
            try:
                d[oid] = Transform(np.array(nums[0:3]), np.array(nums[3:7]), np.array(nums[7:10]))
            except ValueError as e:
                raise ParseError(f"bad pose override for {oid!r}: {e}", path, int(line[r]))
        overrides[r] = d
    if v_row is not None:
        raise ParseError(_VALIDATION_MESSAGES[int(code[v_row])], path, int(line[v_row]))
    if err_line is not None:
        raw = data[info[5]:info[5] + info[6]].decode("ascii")
        _parse_line(raw, path, err_line)  # raises the reference's exact error
        raise ParseError("unparsable line", path, err_line)  # not reached
    keep = np.nonzero(inwin)[0]
    return (np.ascontiguousarray(table[keep]), line[keep], [overrides[r] for r in keep]), path


def parse_fixation_table(path, time_window=None, threads: int = 0) -> np.ndarray:
    """(F, 18) float64 fixation table of a log (gaze normalised), same rows,
    order and errors as parse_fixation_log."""
    res, p = _read(path, time_window, threads)
    if res is None:
        return _parse_python(p, time_window).table
    return res[0]


def parse_fixation_log(path, time_window=None, threads: int = 0) -> FixationLog:
    """Parse a fixation log, keeping start_time in [t0, t1) (reference
    gaze.py:130-188: same line schema, header/comment handling, pose-override
    groups, ParseError messages and line numbers)."""
    res, p = _read(path, time_window, threads)
    if res is None:
        return _parse_python(p, time_window)
    table, line, overrides = res
    log = FixationLog()
    if len(table):
        t = table.tolist()
        new = Fixation.__new__
        for r, ov in zip(t, overrides):
            f = new(Fixation)
            # the row already passed Fixation.__post_init__ (C++ verdict 0) and
            # its gaze is normalised: set the fields without re-validating
            f.__dict__.update(start_time=r[0], duration=r[1], camera_position=np.array(r[2:5]),
                              camera_rotation=np.array(r[5:9]), frustum=tuple(r[9:15]),
                              gaze_dir=np.array(r[15:18]), overrides=ov if ov is not None else {})
            log.append(f)
    log.table = table
    log.line = line
    log.n_override_groups = sum(len(o) for o in overrides if o)
    return log
