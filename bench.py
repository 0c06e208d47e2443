"""Benchmark: surface fixation density-map generation on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one full density-map generation (all fixations of the workload)
over the resident scene.  Workload (BASELINE.json configs[1]):
C2 room, 98,080 triangles / 20 objects, k = 10,000 samples/m^2 (N = 2.19 M
samples), 100,000 fixations, 4-sigma filtering on, 512^2 z-buffer.  Under
torchrun (N > 1) every rank generates its own 100,000-fixation shard of an
N x 100,000 stream (weak scaling) and the partial maps are combined with one
NCCL sum all-reduce, followed by the global max.

metric: sample-fixation pairs per second (N_samples * F / t), the same
numerator for CPU and GPU, filtered or not.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sample-fixation pairs/s (density-map generation)"
UNIT = "pairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2",
                    choices=["c1", "c2", "c2off", "c3k1", "c3k3", "c3k10", "c3k30", "c3k100", "c4", "c5"])
    ap.add_argument("--fixations", type=int, default=0, help="override fixations per rank")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-fixations", type=int, default=0)
    ap.add_argument("--no-stats", action="store_true", help="skip the instrumented roofline pass (profiling runs)")
    ap.add_argument("--collective", choices=["auto", "p2p", "nccl"], default="auto",
                    help="N > 1: fused peer reduce kernel (p2p; auto falls back to NCCL if peers cannot be mapped)")
    return ap.parse_args()


def shard_of(name: str, fx: np.ndarray, rank: int, world: int):
    """(this rank's fixations, total fixations of the job, scaling mode)."""
    if name == "c4":
        from paper_2601_07571_b200.sharding import shard_range

        a, b = shard_range(len(fx), rank, world)
        return np.ascontiguousarray(fx[a:b]), len(fx), "strong"
    return fx, len(fx) * world, "weak"


def workload(name: str, n_fix: int, rank: int):
    import workloads as W

    filtering = True
    if name == "c1":
        scene, k, fx = W.c1()
    elif name in ("c2", "c2off"):
        scene = W.room_scene()
        k = 10_000.0
        fx = W.room_fixations(n_fix or 100_000, seed=1 + 1000 * rank, scene=scene)
        filtering = name == "c2"
    elif name.startswith("c3k"):
        scene = W.room_scene()
        k = 1000.0 * int(name[3:])
        fx = W.room_fixations(n_fix or 10_000, seed=1 + 1000 * rank, scene=scene)
    elif name == "c4":
        # strong scaling: one 50 x 20k session stream, each rank its contiguous shard
        # (sharded by the caller, see shard_of)
        scene = W.room_scene()
        k = 10_000.0
        fx = W.session_fixations(scene=scene)
        if n_fix:
            fx = fx[:n_fix]
    elif name == "c5":
        scene = W.shells_scene()
        k = 20_000.0
        fx = W.orbit_fixations(n_fix or 50_000, 4 + 1000 * rank, 4.5, 6.0, jitter=0.3)
    else:
        raise ValueError(name)
    if n_fix:
        fx = fx[:n_fix]
    desc = {"c1": "C1 icosphere(3), k=1e3, 200 fixations",
            "c2": "C2 room 98,080 tris/20 objects, k=1e4, 100k fixations, filtering on",
            "c2off": "C2 room 98,080 tris/20 objects, k=1e4, 100k fixations, filtering off",
            "c4": "C4 room, 50 users x 20k fixations (1M), k=1e4, filtering on",
            "c5": "C5 12 nested icosphere(6) shells 983,040 tris, k=2e4, 50k fixations"}.get(
                name, f"C3 room sample-density sweep, k={name[3:]}e3, 10k fixations")
    return scene, k, np.ascontiguousarray(fx), filtering, desc


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_port_pairs_per_s(scene, k, fx, filtering, n_fix, threads):
    """The oracle port (oracle/gm_oracle.c: the reference algorithm restated in
    C, numba's prange -> OpenMP over samples) on a bounded fixation prefix."""
    from oracle import oracle as O

    lay = O.build_layouts(scene, k)
    N = sum(v[3] for v in lay.values())
    rows = O.rows_as_fixations(fx[:n_fix])
    O.generate(scene, rows[:2], k=k, filtering_enabled=filtering, threads=threads, layouts=lay)  # warm
    t0 = time.perf_counter()
    O.generate(scene, rows, k=k, filtering_enabled=filtering, threads=threads, layouts=lay)
    dt = time.perf_counter() - t0
    return N * len(rows) / dt, dt, N


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    if rank != 0:
        return
    scene, k, fx, filtering, desc = workload(args.config, args.fixations, 0)
    threads = host_threads()
    per_step = args.cpu_fixations or (300 if args.config != "c1" else 200)
    from oracle import oracle as O

    lay = O.build_layouts(scene, k)
    N = sum(v[3] for v in lay.values())
    rows = O.rows_as_fixations(fx)
    for i in range(args.warmup):
        O.generate(scene, rows[:max(2, per_step // 10)], k=k, filtering_enabled=filtering, threads=threads, layouts=lay)
    times = []
    for s in range(args.steps):
        sl = rows[(s * per_step) % len(rows):][:per_step]
        t0 = time.perf_counter()
        O.generate(scene, sl, k=k, filtering_enabled=filtering, threads=threads, layouts=lay)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    v = N * per_step / t
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "samples": int(N), "fixations_per_step": per_step,
                   "note": "CPU port of the reference algorithm (oracle/gm_oracle.c), bounded prefix per step"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{per_step} fixations of the workload per step, {N} samples"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_ours(args, rank, world):
    import paper_2601_07571_b200 as gm
    from paper_2601_07571_b200 import _native

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        # GM_BENCH_DEVICE_MOD / GM_BENCH_BACKEND let a 1-GPU box exercise the multi-rank
        # path (ranks sharing a device over gloo); the product run is NCCL, one GPU per rank
        ndev = int(os.environ.get("GM_BENCH_DEVICE_MOD", "0")) or torch.cuda.device_count()
        local = int(os.environ.get("LOCAL_RANK", rank)) % max(ndev, 1)
        torch.cuda.set_device(local)
        dist.init_process_group(os.environ.get("GM_BENCH_BACKEND", "nccl"))
    device = local if world > 1 else 0

    scene, k, fx_all, filtering, desc = workload(args.config, args.fixations, rank)
    fx, total_F, scaling = shard_of(args.config, fx_all, rank, world)
    cfg = gm.GenerationConfig(k=k, filtering_enabled=filtering)
    sampled = gm.build_sampled_meshes(scene, k, device=device)
    plan = gm.ScenePlan(scene, sampled, scene.object_ids, device=device)
    lib = _native.load()
    N = plan.n_samples
    F = len(fx)
    ccfg = _native.GmConfig(cfg.theta, cfg.epsilon_abs, cfg.epsilon_rel, cfg.zbuffer_resolution,
                            int(filtering), args.batch, 0)
    bad = np.zeros(1, np.int64)
    _native.check(lib.gm_plan_prepare(plan._h, _native.dptr(fx), F, ctypes.byref(ccfg), _native.iptr(bad)))

    coll_used = None
    if world > 1:
        from paper_2601_07571_b200.sharding import reduce_peers

    def one_step(timed_stats=None):
        tm = _native.GmTimings()
        ms = ctypes.c_float(0.0)
        _native.check(lib.gm_plan_run(plan._h, 1, 0, ctypes.byref(tm), ctypes.byref(ms)), "gm_plan_run")
        extra = 0.0
        if world > 1:
            # the ranks' partial maps -> the sum on every rank + global max (device ms of
            # this rank's fused peer-reduce kernel, or of NCCL's all-reduce)
            nonlocal coll_used
            gmax, coll_used, extra = reduce_peers(plan, None, args.collective)
        else:
            gmax = plan.global_max()
        return ms.value + extra, tm, gmax

    for _ in range(args.warmup):
        one_step()
    times, tms = [], []
    with ClockSampler(device) as clk:
        for _ in range(args.steps):
            _native.check(lib.gm_plan_flush_l2(plan._h, 512 << 20))
            plan.sync()
            if world > 1:
                dist.barrier()
            t, tm, gmax = one_step()
            times.append(t)
            tms.append(tm)
    step_ms = float(np.mean(times))
    if world > 1:
        import torch

        tt = torch.tensor([step_ms], device=f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms = float(tt.item())
    value = N * total_F / (step_ms / 1e3)
    tm = tms[-1]
    # per step: k_set_i64, then per batch k_tri_setup, k_level1, k_fix32, k_mark, k_coarse, k_texels,
    # k_texels<crowded>, k_samples (+ 4 CUB radix-sort kernels ordering the super-chunks); then k_max
    launches = int(tm.batches) * 8 + 2
    library_launches = int(tm.batches) * 4

    # ---- e2e through the public API (host table in, host values out) -----
    # Every step: fixation table (host) -> host setup -> H2D -> kernels -> D2H of
    # the values.  N > 1: sharding.generate_sharded over the concatenated
    # N x F stream (each rank's contiguous shard is its own F fixations) with
    # the NCCL all-reduce inside the timed region.
    e2e = None
    if not args.no_e2e:
        if world > 1:
            from paper_2601_07571_b200.sharding import generate_sharded

            full = fx_all if scaling == "strong" else np.concatenate(
                [workload(args.config, args.fixations, r)[2] for r in range(world)])

            def e2e_call():
                return generate_sharded(scene, sampled, full, cfg, device=device, collective=args.collective)
        else:
            def e2e_call():
                return gm.generate(scene, sampled, fx, cfg, device=device)
        e2e_call()  # plan upload + warm
        e_times = []
        for _ in range(max(1, min(args.steps, 3))):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            e2e_call()
            e_times.append(time.perf_counter() - t0)
        e_t = float(np.mean(e_times))
        if world > 1:
            import torch

            tt = torch.tensor([e_t], device=f"cuda:{device}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_t = float(tt.item())
        e2e = {"value": N * total_F / e_t, "unit": UNIT, "h2d_bytes_per_step": int(F * (208 + 80)),
               "d2h_bytes_per_step": int(N * 8), "ms_per_step": e_t * 1e3,
               "path": "paper_2601_07571_b200.generate (fixation table in host memory -> values dict)"
               if world == 1 else "paper_2601_07571_b200.sharding.generate_sharded (partial maps + peer reduce)",
               "timing": "host wall clock around the API call"}

    # ---- algorithmic work of this step (one instrumented, untimed pass) ----
    stats = (ctypes.c_uint64 * len(_native.STAT_NAMES))()
    tm_s = _native.GmTimings()
    ms_s = ctypes.c_float(0.0)
    if not args.no_stats:
        _native.check(lib.gm_plan_run(plan._h, 1, _native.GM_FLAG_STATS, ctypes.byref(tm_s), ctypes.byref(ms_s)))
        _native.check(lib.gm_plan_stats(plan._h, stats))
    st = dict(zip(_native.STAT_NAMES, [int(x) for x in stats]))
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(peaks_path.read_text()) if peaks_path.exists() else {}
    clk_ghz = peaks.get("sm_max_mhz", 1965.0) / 1e3
    # FP64 SIMT peak (nominal, no measured FP64 figure exists): 148 SM x 64 FP64 lanes x 2 (FMA) x max clock
    fp64_peak = 148 * 64 * 2 * clk_ghz / 1e3
    # algorithmic FP64 flops per unit, counted from the reference source (kernels.py):
    #   exact sample evaluation (camera transform :305-307 + NDC projection :314-315) 26
    #   cone test (:330-337) 14, depth test (:323-327 + bilinear :231-261) 24
    #   marked texel: the writer's exact pixel test -- 3 edge functions (:107-109, 23) + l, inv_w,
    #   1/inv_w (:119-125, 9) -- whether k_texels evaluates it in float64 or proves it with float32 bounds
    fl = {"k_samples<mark>": 26 * st["exact_evals"] + 14 * st["ndc_candidates"],
          "k_texels": 32 * st["texels"],
          "k_samples<accumulate>": 26 * st["exact_evals"] + 14 * st["ndc_candidates"] + 24 * st["cone_candidates"]}
    # per-kernel device time for the roofline: the timed steps overlap batches on several streams, so
    # their per-phase events include concurrent work; one more untimed pass on a single stream gives
    # each kernel's own time (CUDA events on the stream it runs on)
    tm1 = _native.GmTimings()
    ms1 = ctypes.c_float(0.0)
    if not args.no_stats:
        _native.check(lib.gm_plan_run(plan._h, 1, _native.GM_FLAG_ONE_STREAM, ctypes.byref(tm1), ctypes.byref(ms1)))
    else:
        tm1 = tm
    times = {"k_samples<mark>": tm1.mark_ms, "k_texels": tm1.texel_ms, "k_samples<accumulate>": tm1.accumulate_ms,
             "k_tri_setup": tm1.cull_ms}
    dom = max(times, key=times.get)
    dom_flops = fl.get(dom, 0)
    ach = dom_flops / (times[dom] / 1e3) / 1e12 if times[dom] else None
    # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    # (profiles/r1_ncu_traffic.json, written by tools/ncu_traffic.py), per launch like `achieved`
    traffic, hbm, issue = None, None, None
    tpath = ROOT / "profiles" / "r1_ncu_traffic.json"
    kname = {"k_samples<mark>": "k_mark", "k_samples<accumulate>": "k_samples<0>",
             "k_texels": "k_texels<0, 0, 0, 0>"}.get(dom, dom)
    if tpath.exists():
        tk = json.loads(tpath.read_text())["kernels"].get(kname)
        if tk and int(tm.batches):
            traffic = tk["dram_bytes_per_launch"]
            launch_ms = times[dom] / int(tm.batches)
            gbs = traffic / (launch_ms / 1e3) / 1e9
            hbm_peak = peaks.get("hbm_gbs", 7700.0)
            hbm = {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                   "launch_ms": launch_ms, "fixations_per_launch": tk["fixations_per_launch"]}
            if "ipc" in tk:  # the bound that does apply: instruction issue (4 warp-instr/cycle/SM)
                issue = {"ipc": tk["ipc"], "peak_ipc": 4.0, "frac": tk["ipc"] / 4.0,
                         "issue_slots_busy": tk["issue_pct_of_peak"] / 100.0, "source": "ncu --set full"}
    roof = {"bound": "fp64", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": (ach / fp64_peak) if ach else None, "traffic": traffic, "hbm": hbm, "issue": issue,
            "kernel": dom,
            "kernel_ms_per_step": times[dom], "kernel_share": times[dom] / max(ms1.value, 1e-9) if ms1.value else None,
            "timing": "kernel times from one untimed single-stream pass (CUDA events); share of that pass",
            "algorithmic_flops_per_step": dom_flops,
            "peak_kind": "nominal FP64 FMA peak at max SM clock (MEASURED_PEAKS.json has no FP64 figure)",
            "work": st}
    # SURVEY.md 8d's step roofline: algorithmic FLOPs of the reference's per-pair work -- 26 per nominal
    # sample-fixation pair (camera transform + NDC projection, kernels.py:305-315) + 43 per NDC candidate
    # (depth test + Gaussian, :323-340) -- over the whole step, against the FP32 SIMT peak (nominal:
    # 148 SM x 128 lanes x 2 x max clock; the path computes in FP64 for parity, the FP32 peak is the
    # survey's yardstick).  Culling means most nominal pairs are never evaluated, so this can exceed 1.
    fp32_peak = 148 * 128 * 2 * clk_ghz / 1e3
    step_flops = 26.0 * N * F + 43.0 * st.get("ndc_candidates", 0)
    step_tf = step_flops / (step_ms / 1e3) / 1e12 if st.get("ndc_candidates") else None
    roof_step = {"bound": "fp32", "achieved": step_tf, "peak": fp32_peak, "unit": "TFLOP/s",
                 "frac": step_tf / fp32_peak if step_tf else None, "algorithmic_flops_per_step": step_flops,
                 "definition": "SURVEY.md 8d: (26 N F + 43 sum C_ndc) / t / P_FP32 (per rank)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            n_cpu = args.cpu_fixations or (200 if args.config == "c1" else 1000)
            v, dt, _ = cpu_port_pairs_per_s(scene, k, fx, filtering, n_cpu, host_threads())
            cpu = {"value": v, "unit": UNIT, "cores": host_threads(), "kind": "port",
                   "sample": f"first {n_cpu} fixations of the workload ({dt:.1f} s), oracle/gm_oracle.c with OpenMP"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": host_threads(), "kind": "port", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "samples": int(N), "triangles": int(plan._lib.gm_plan_num_triangles(plan._h)),
                       "fixations_per_gpu": int(F), "fixations_total": int(total_F),
                       "zbuffer": cfg.zbuffer_resolution, "filtering": filtering,
                       "parallelism": (f"fixation-sharded x{world}, " + ("fused peer reduce (CUDA IPC over NVLink)"
                                       if coll_used == "p2p" else "NCCL sum all-reduce")) if world > 1 else "single GPU",
                       "l2": "flushed (512 MiB write) before every timed step",
                       "timing": "CUDA events on the plan stream around each full generation (+ all-reduce)"},
            "e2e": e2e, "roofline": roof, "roofline_step_fp32": roof_step, "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": launches,
            "library_launches": library_launches,
            "phases_ms": {"cull": tm.cull_ms, "mark": tm.mark_ms, "texels": tm.texel_ms,
                          "accumulate": tm.accumulate_ms, "batches": tm.batches, "retries": tm.retries,
                          "screen_tris": tm.screen_tris,
                          "note": "per-batch event spans summed; batches overlap on 3 streams, so phases overlap"},
            "phases_single_stream_ms": {"total": ms1.value, "cull": tm1.cull_ms, "mark": tm1.mark_ms,
                                        "texels": tm1.texel_ms, "accumulate": tm1.accumulate_ms},
            "global_max": gmax,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if args.gpus == 1 else 1))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
