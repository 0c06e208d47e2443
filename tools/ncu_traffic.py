"""DRAM traffic per launch of each kernel in an ncu --set full report, for
bench.py's roofline.traffic.

    python tools/ncu_traffic.py gpurun_out/prof_r1.ncu-rep 1024 > profiles/r1_ncu_traffic.json

(1024 = fixations per batch, i.e. per launch, in the profiled run)
"""

import collections
import csv
import io
import json
import subprocess
import sys


def main(path, batch):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                          "sm__inst_executed.avg.per_cycle_active,sm__inst_issued.avg.pct_of_peak_sustained_active,"
                          "smsp__inst_executed.sum,lts__t_sector_hit_rate.pct"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1.0, "us": 1e-3, "ns": 1e-6}
    acc = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "")  # template arguments kept: k_texels<0, 0, 0>
        rd = float(r[hdr.index("dram__bytes_read.sum")]) * scale[units[hdr.index("dram__bytes_read.sum")]]
        wr = float(r[hdr.index("dram__bytes_write.sum")]) * scale[units[hdr.index("dram__bytes_write.sum")]]
        t = float(r[hdr.index("gpu__time_duration.sum")]) * scale[units[hdr.index("gpu__time_duration.sum")]]
        a = acc[name]
        a[0] += 1
        a[1] += rd + wr
        a[2] += t
        a[3] += float(r[hdr.index("sm__inst_executed.avg.per_cycle_active")])
        a[4] += float(r[hdr.index("sm__inst_issued.avg.pct_of_peak_sustained_active")])
        if "smsp__inst_executed.sum" in hdr:
            j = hdr.index("smsp__inst_executed.sum")
            a[5] += float(r[j].replace(",", "")) * {"inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}.get(units[j], 1)
        if "lts__t_sector_hit_rate.pct" in hdr:
            a[6] += float(r[hdr.index("lts__t_sector_hit_rate.pct")])
    res = {k: {"launches": n, "dram_bytes_per_launch": b / n, "ms_per_launch_cold": t / n,
               "ipc": ipc / n, "issue_pct_of_peak": iss / n, "inst_executed_per_launch": inst / n,
               "l2_hit_rate_pct": l2 / n, "fixations_per_launch": batch}
           for k, (n, b, t, ipc, iss, inst, l2) in acc.items()}
    print(json.dumps({"source": path, "how": "ncu --set full --clock-control none (serialised, cold cache)",
                      "kernels": res}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1024)
