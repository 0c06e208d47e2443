"""Per-kernel totals of an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file X`).

    python tools/launch_summary.py gpurun_out/launches_r2.csv "title" > profiles/r2_launches.md
"""

import collections
import csv
import sys


def main(path, title):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}
    acc = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        acc[name][0] += 1
        acc[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    skip = ("k_peak_fma",)  # bench.py's roofline denominators, not part of the step
    items = [(k, v) for k, v in acc.items() if not k.startswith(skip)]
    tot = sum(v[1] for _, v in items)
    print(f"# {title}\n")
    print(f"Source: `{path}` (ncu --metrics gpu__time_duration.sum --clock-control none: serialised, cold-cache "
          "launch times; shares, not absolute step times).  bench.py's FMA peak-measurement kernels excluded.\n")
    print("| kernel | launches | total ms | share | us per launch |")
    print("|---|---|---|---|---|")
    for k, (n, t) in sorted(items, key=lambda x: -x[1][1]):
        if t / tot < 0.001:
            continue
        print(f"| `{k[:70]}` | {n} | {t / 1e6:.2f} | {100 * t / tot:.1f}% | {t / n / 1e3:.1f} |")
    print(f"\nTotal {tot / 1e6:.2f} ms over {sum(v[0] for _, v in items)} launches.")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "ncu launch list")
