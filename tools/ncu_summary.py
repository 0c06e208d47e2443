"""Summarise ncu outputs into markdown for profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/r1_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/r1_full.md
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Grid Size", "Block Size", "Waves Per SM"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__inst_executed.sum", "gpu__time_duration.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(t for _, t in agg.values()) or 1.0
    print(f"| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")


def _ncu_csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(path):
    rows = _ncu_csv([path, "--page", "details"])
    hdr = rows[0]
    I = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) < 15:
            continue
        key = (r[I["ID"]], r[I["Kernel Name"]].split("(")[0])
        per.setdefault(key, {})[r[I["Metric Name"]]] = (r[I["Metric Value"]], r[I["Metric Unit"]])
    raw = _ncu_csv([path, "--page", "raw"])
    rawv = {}
    if raw:
        rh = raw[0]
        for r in raw[2:]:
            if len(r) != len(rh):
                continue
            d = dict(zip(rh, r))
            rawv[(d.get("ID"), d.get("Kernel Name", "").split("(")[0])] = d
    for (kid, name), m in per.items():
        print(f"### launch {kid}: `{name}`\n")
        print("| metric | value |\n|---|---|")
        for k in KEYS:
            if k in m:
                print(f"| {k} | {m[k][0]} {m[k][1]} |")
        d = rawv.get((kid, name), {})
        for k in RAW:
            if k in d:
                print(f"| {k} | {d[k]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
