"""Golden cases for fixation-log ingestion, produced by the
REFERENCE's parse_fixation_log (gazemap/gaze.py:130-188).

    python tests/golden/make_fixlog_golden.py

Writes tests/golden/fixlog_cases.json: per case the exact file bytes (latin-1
string), the time window, and the reference's outcome -- either the parsed
fixations (every float as float.hex, overrides included) or the exception
type and message (path replaced by "{path}").  tests/test_fixlog.py replays
them against paper_2601_07571_b200.parse_fixation_log without the reference.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GAZEMAP_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import gazemap as gm  # noqa: E402

import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "fixlog_cases.json"
GOOD = "0.5 0.25 0 1.6 0 0 0 0 1 -0.1 0.1 0.1 -0.1 0.1 100 0.01 0.02 -1"


def cases():
    c = {
        "few_fields": GOOD + "\n1 2 3\n",
        "bad_number": GOOD + "\n" + GOOD.replace("0.25", "0.2x5", 1) + "\n",
        "bad_number_quote": GOOD + "\n" + GOOD.replace("0.25", "0.2'5", 1) + "\n",
        "group_count": GOOD + " cube 1 2\n",
        "bad_override_number": GOOD + " cube 1 2 3 0 0 0 1 1 1 x\n",
        "bad_quaternion": GOOD + " cube 1 2 3 0 0 0 2 1 1 1\n",
        "bad_quaternion_before_bad_number": GOOD + " cube 1 2 3 0 0 0 2 1 1 1\n" + GOOD.replace("0.25", "zz") + "\n",
        "overrides_two_groups": GOOD + " cube 1 2 3 0 0 0 1 1 1 1 sphere 0 0 0 0 0.6 0 0.8 2 2 2\n" + GOOD + "\n",
        "duration": GOOD.replace("0.25", "-1", 1) + "\n",
        "invalid_outside_window": GOOD.replace("0.5 0.25", "50 -1", 1) + "\n" + GOOD + "\n",
        "zero_gaze": GOOD.replace("0.01 0.02 -1", "0 0 0") + "\n",
        "gaze_backwards": GOOD.replace("0.01 0.02 -1", "0 0 1") + "\n",
        "near_far": GOOD.replace("0.1 100", "0.1 0.05") + "\n",
        "bounds": GOOD.replace("-0.1 0.1 0.1 -0.1", "0.1 -0.1 0.1 -0.1") + "\n",
        "separators_only": GOOD + "\n,,,\n",
        "underscore": GOOD.replace("0.25", "0.2_5", 1) + "\n",
        "double_underscore": GOOD.replace("0.25", "0.2__5", 1) + "\n",
        "inf_nan": GOOD.replace("0.5 ", "inf ", 1).replace("0 1.6", "nan 1.6") + "\n",
        "hex_float": GOOD.replace("0.25", "0x1p-2", 1) + "\n",
        "exponents": GOOD.replace("0.25", "2.5e-1", 1).replace("100", "1E+2") + "\n",
        "bare_dots": GOOD.replace("0.25", ".25", 1).replace(" 1 -0.1", " 1. -0.1") + "\n",
        "header_mid_file": GOOD + "\nabc def\n" + GOOD + "\n",
        "control_whitespace": GOOD.replace(" ", "\x0b", 3) + "\x0c\n" + "\x1c" + GOOD + "\n",
        "non_ascii": GOOD + "\n " + GOOD + "\n",
        "nul_byte": GOOD.replace("0.25", "0.25\x00", 1) + "\n",
        "signs": GOOD.replace("0.25", "+0.25", 1).replace("1.6", "-1.6") + "\n",
        "nan_start": GOOD.replace("0.5 ", "nan ", 1) + "\n",
        "sign_only": GOOD.replace("0.25", "-", 1) + "\n",
        "dangling_exponent": GOOD.replace("0.25", "1e", 1) + "\n",
        "infinity": GOOD.replace("0.25", "-Infinity", 1) + "\n",
        "comments_blank": "# c\n   \n" + GOOD + "  # tail\n",
        "crlf_and_cr": GOOD + "\r\n" + GOOD + "\r" + GOOD + "\r\n",
        "commas": GOOD.replace(" ", ",") + "\n" + GOOD.replace(" ", " , ") + "\n",
        "empty": "",
    }
    # a realistic room stream: repr floats, mixed separators and line endings, headers, overrides
    fx = W.room_fixations(300, seed=5)
    lines = ["# session 1", "start dur px py pz qx qy qz qw l r t b n f gx gy gz"]
    for i, r in enumerate(fx):
        ln = (", " if i % 3 == 0 else " \t").join(repr(float(v)) for v in r)
        if i % 11 == 0:
            ln += "  # note"
        if i % 13 == 0:
            ln += " cube 1 2 3 0 0 0 1 1 1 1"
        lines.append(ln)
    c["room_stream"] = "\r\n".join(lines[:100]) + "\n" + "\r".join(lines[100:200]) + "\r" + "\n".join(lines[200:]) + "\n"
    return c


def outcome(path, window):
    try:
        fx = gm.parse_fixation_log(path, window)
    except Exception as e:  # noqa: BLE001 - the reference's exact exception is the fixture
        return {"error": type(e).__name__, "message": str(e).replace(str(path), "{path}")}
    rows = []
    for f in fx:
        vals = [f.start_time, f.duration, *f.camera_position, *f.camera_rotation, *f.frustum, *f.gaze_dir]
        ov = {k: [float(x).hex() for x in (*t.translation, *t.rotation, *t.scale)] for k, t in f.overrides.items()}
        rows.append({"v": [float(x).hex() for x in vals], "ov": ov})
    return {"rows": rows}


def main():
    out = []
    with tempfile.TemporaryDirectory() as td:
        for name, text in cases().items():
            p = Path(td) / f"{name}.log"
            p.write_bytes(text.encode("utf-8"))
            for window in (None, [0.0, 10.0], [0.0, 0.0]):
                out.append({"name": name, "text": text, "window": window,
                            "expect": outcome(p, tuple(window) if window else None)})
    OUT.write_text(json.dumps(out, indent=0, ensure_ascii=True))
    print(f"wrote {len(out)} cases to {OUT}")


if __name__ == "__main__":
    main()
