"""Per-source-line hot spots of one kernel in an ncu report (cuda,sass view).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep k_texels [top]
"""

import csv
import io
import subprocess
import sys


def main(path, kernel, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, agg = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r) if h not in ("Source",)}
            continue
        if hdr is None or len(r) < 8 or r[2] != "-":
            continue
        try:
            inst = int(r[hdr["Instructions Executed"]])
            samp = int(r[hdr["Warp Stall Sampling (All Samples)"]])
        except (ValueError, KeyError):
            continue
        agg.append((samp, inst, f"{fname}:{r[0]}", r[1][:90]))
    ts = sum(a[0] for a in agg) or 1
    ti = sum(a[1] for a in agg) or 1
    print(f"total samples {ts}  total warp-instr {ti}")
    for samp, inst, loc, src in sorted(agg, reverse=True)[:top]:
        print(f"{100 * samp / ts:5.1f}% samp {100 * inst / ti:5.1f}% inst  {loc:22s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
