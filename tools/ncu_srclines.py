"""Per-source-line hot spots of an ncu report (warp-stall samples and
instructions executed), from `ncu -i X --page source --csv --print-source cuda,sass`.

    python tools/ncu_srclines.py report.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys


def lines(rep, kern=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res, fn, path, hdr = [], None, None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1]
            continue
        if r[0] == "Function Name":
            fn = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0]:
            continue
        if kern and kern not in (fn or ""):
            continue
        d = dict(zip(hdr, r))
        try:
            samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            inst = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        res.append((fn, path.split("/")[-1], int(r[0]), r[1].strip(), samp, inst))
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    L = lines(rep, kern)
    ts = sum(x[4] for x in L) or 1
    ti = sum(x[5] for x in L) or 1
    print(f"total samples {ts}, instructions {ti}")
    for fn, f, ln, src, s, i in sorted(L, key=lambda x: -x[4])[:top]:
        print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% inst  {f}:{ln}  {src[:90]}")
