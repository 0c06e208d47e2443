"""Recompute every `frac` of a bench.py JSON line from its own counters and the
committed ncu JSON, and print the arithmetic as markdown.

    python tools/roofline_report.py profiles/r2_bench.jsonl [profiles/r2_ncu_traffic.json] > profiles/r2_roofline.md
"""

import json
import sys


def main(bench_path, ncu_path="profiles/r2_ncu_traffic.json"):
    line = next(json.loads(ln) for ln in open(bench_path) if ln.startswith("{") and '"impl"' not in ln)
    ncu = json.load(open(ncu_path))["kernels"]
    r, st, pk = line["roofline"], line["roofline"]["work"], line["peaks"]
    ss = line["phases_single_stream_ms"]
    batches = line["phases_ms"]["batches"]
    t_tex = ss["texels"] / 1e3
    out = [f"# Roofline arithmetic of the C2 bench line (`{bench_path}`, first line)", ""]
    out.append(f"Inputs: k_texels time (both passes, single-stream pass, CUDA events) {ss['texels']:.2f} ms over "
               f"{batches} batches; measured peaks FP64 {pk['fp64']:.2f} / FP32 {pk['fp32']:.2f} TFLOP/s "
               f"(gm_peak_flops), HBM {pk['hbm_gbs']} GB/s (MEASURED_PEAKS.json); work counters from the "
               "instrumented pass (`roofline.work`); per-launch DRAM bytes and warp instructions from "
               f"`{ncu_path}`.")
    out.append("")
    a = 16.0 * st["bbox_px"] / t_tex / 1e12
    out.append(f"* **headline (`roofline`)**, SURVEY 8d raster definition: 16 FP64 flops x bbox_px "
               f"{st['bbox_px']:.4g} / {t_tex:.4f} s = {a:.2f} TFLOP/s; / {pk['fp64']:.2f} = **{a / pk['fp64']:.3f}** "
               f"(line: {r['frac']:.3f}).")
    b = 32.0 * st["texels"] / t_tex / 1e12
    out.append(f"* `views.marked_texels`: 32 x texels {st['texels']:.4g} / {t_tex:.4f} s = {b:.3f} TFLOP/s; "
               f"/ {pk['fp64']:.2f} = {b / pk['fp64']:.4f}.")
    k1 = next(v for k, v in ncu.items() if k.startswith("k_texels<0, 0, 0"))
    k2 = next((v for k, v in ncu.items() if k.startswith("k_texels_crowded<0, 0, 0")), None)
    launch_ms = ss["texels"] / batches
    bytes_ = k1["dram_bytes_per_launch"] + (k2["dram_bytes_per_launch"] if k2 else 0.0)
    gbs = bytes_ / (launch_ms / 1e3) / 1e9
    out.append(f"* `views.hbm`: DRAM bytes of both launches {bytes_:.4g} B / {launch_ms:.4f} ms per batch = "
               f"{gbs:.0f} GB/s; / {pk['hbm_gbs']} = {gbs / pk['hbm_gbs']:.3f}.")
    inst = k1["inst_executed_per_launch"] + (k2["inst_executed_per_launch"] if k2 else 0.0)
    clk = line["clocks"]["sm_max_mhz"] or 1965.0
    rate = inst / (launch_ms / 1e3)
    peak = 4.0 * 148 * clk * 1e6
    out.append(f"* `views.issue`: warp instructions of both launches {inst:.4g} / {launch_ms:.4f} ms = "
               f"{rate / 1e9:.0f} G/s; / (4 x 148 x {clk:.0f} MHz = {peak / 1e9:.0f} G/s) = {rate / peak:.3f}.")
    s8 = line["roofline_step_fp32"]
    n = line["config"]["samples"]
    f = line["config"]["fixations_per_gpu"]
    step = line["ms_per_step"] / 1e3
    flops = 26.0 * n * f + 43.0 * st["ndc_candidates"]
    out.append(f"* `roofline_step_fp32` (SURVEY 8d step figure): (26 x {n} x {f} + 43 x {st['ndc_candidates']:.4g}) "
               f"/ {step:.4f} s = {flops / step / 1e12:.2f} TFLOP/s; / {pk['fp32']:.2f} = {flops / step / 1e12 / pk['fp32']:.3f} "
               f"(line: {s8['frac']:.3f}).")
    out.append("")
    out.append("The headline and the step figure are *effective* rates: the work is the reference algorithm's, "
               "most of which the culls and the marked-texel design never execute. `issue` is what bounds the "
               "kernel as built: instruction issue / latency on irregular float32 selection work, with HBM at "
               "the fraction `hbm` shows.")
    print("\n".join(out))


if __name__ == "__main__":
    main(*sys.argv[1:])
