"""Benchmark: surface fixation density-map generation on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one full density-map generation (all fixations of the workload)
over the resident scene.  Workload (BASELINE.json configs[1]):
C2 room, 98,080 triangles / 20 objects, k = 10,000 samples/m^2 (N = 2.19 M
samples), 100,000 fixations, 4-sigma filtering on, 512^2 z-buffer.

Multi-GPU: `--gpus N` runs one process per GPU.  Without WORLD_SIZE in the
environment bench.py launches the N ranks itself (torch.distributed.run,
127.0.0.1); under an external torchrun it is one of them.  The default C2
line is weak-scaled (every rank generates its own 100,000-fixation shard of an
N x 100,000 stream); `--config c4` is the strong-scaled session stream
(50 users x 20k = 1M fixations, contiguous shards).  The ranks' partial maps
are combined by the package's fused peer-reduce kernel (CUDA IPC over
NVLink), NCCL all-reduce as fallback, then the global max.

metric: sample-fixation pairs per second (N_samples * F / t), the same
numerator for CPU and GPU, filtered or not.

--impl reference: the unmodified reference package (numba, staged under
baseline/_ref by pip) on the box's host cores, on a bounded fixation prefix
per step; without baseline/_ref the C port of the reference algorithm
(oracle/gm_oracle.c) stands in, and the line says so.
"""

from __future__ import annotations

import argparse
import ctypes
import gc
import json
import os
import socket
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
REF_DIR = ROOT / "baseline" / "_ref"
CONFIGS = ["c1", "c2", "c2off", "c3k1", "c3k3", "c3k10", "c3k30", "c3k100", "c4", "c5"]
# fixations per timed step of the CPU reference arm (bounded samples, ~10 s each on 16 cores)
REF_PER_STEP = {"c1": 200, "c2": 300, "c2off": 100, "c4": 300, "c5": 16, "c3k1": 400, "c3k3": 300,
                "c3k10": 300, "c3k30": 150, "c3k100": 60}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2", choices=CONFIGS)
    ap.add_argument("--fixations", type=int, default=0, help="override fixations per rank")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cold", action="store_true", help="skip the cold map-generation-time measurement")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-fixations", type=int, default=0)
    ap.add_argument("--ref-kind", choices=["auto", "stock", "port"], default="auto",
                    help="--impl reference: the numba reference (stock) or the C port")
    ap.add_argument("--no-stats", action="store_true", help="skip the instrumented roofline pass (profiling runs)")
    ap.add_argument("--collective", choices=["auto", "p2p", "nccl"], default="auto",
                    help="N > 1: fused peer reduce kernel (p2p; auto falls back to NCCL if peers cannot be mapped)")
    return ap.parse_args()


# ------------------------------------------------------------- workloads

def shard_of(name: str, fx: np.ndarray, rank: int, world: int):
    """(this rank's fixations, total fixations of the job, scaling mode)."""
    if name == "c4":
        from paper_2601_07571_b200.sharding import shard_range

        a, b = shard_range(len(fx), rank, world)
        return np.ascontiguousarray(fx[a:b]), len(fx), "strong"
    return fx, len(fx) * world, "weak"


DESC = {"c1": "C1 icosphere(3), k=1e3, 200 fixations",
        "c2": "C2 room 98,080 tris/20 objects, k=1e4, 100k fixations, filtering on",
        "c2off": "C2 room 98,080 tris/20 objects, k=1e4, 100k fixations, filtering off",
        "c4": "C4 room, 50 users x 20k fixations (1M), k=1e4, filtering on, strong-scaled",
        "c5": "C5 12 nested icosphere(6) shells 983,040 tris, k=2e4, 50k fixations"}


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
        scene = W.room_scene()
        k = 10_000.0
        fx = W.session_fixations(scene=scene)  # every rank builds the same 1M stream, shard_of cuts it
    elif name == "c5":
        scene = W.shells_scene()
        k = 20_000.0
        fx = W.orbit_fixations(n_fix or 50_000, 4 + 1000 * rank, 4.5, 6.0, jitter=0.3)
    else:
        raise ValueError(name)
    if n_fix:
        fx = fx[:n_fix]
    desc = DESC.get(name, f"C3 room sample-density sweep, k={name[3:]}e3, 10k fixations")
    return scene, k, np.ascontiguousarray(fx), filtering, desc


# ------------------------------------------------------------- helpers

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


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


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


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """`--gpus N` without an external launcher: start the N ranks (one per
    GPU) through torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


# ------------------------------------------------------------- reference arm

def _stock_reference():
    """The unmodified reference package installed under baseline/_ref (or None)."""
    if not (REF_DIR / "gazemap" / "__init__.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gm_bench_numba_cache")
    os.environ.setdefault("NUMBA_NUM_THREADS", str(max(8, host_threads())))
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import gazemap

    return gazemap


def _to_reference(R, scene, rows):
    objs = tuple(R.SceneObject(o.object_id, R.Mesh(np.asarray(o.mesh.vertices, np.float64),
                                                   np.asarray(o.mesh.faces, np.int64)),
                               R.Transform(np.asarray(o.transform.translation, np.float64),
                                           np.asarray(o.transform.rotation, np.float64),
                                           np.asarray(o.transform.scale, np.float64)))
                 for o in scene.objects)
    fx = [R.Fixation(float(r[0]), float(r[1]), r[2:5].copy(), r[5:9].copy(), tuple(float(x) for x in r[9:15]),
                     r[15:18].copy()) for r in rows]
    return R.Scene(objs), fx


def run_reference(args, rank, world):
    if rank != 0:
        return
    scene, k, fx, filtering, desc = workload(args.config, args.fixations, 0)
    threads = host_threads()
    per_step = args.cpu_fixations or REF_PER_STEP.get(args.config, 200)
    R = _stock_reference() if args.ref_kind != "port" else None
    if args.ref_kind == "stock" and R is None:
        raise SystemExit("baseline/_ref has no reference install")
    times = []
    if R is not None:
        import numba

        rscene, rfx = _to_reference(R, scene, fx)
        cfg = R.GenerationConfig(k=k, filtering_enabled=filtering)
        t0 = time.perf_counter()
        sampled = R.build_sampled_meshes(rscene, k)
        t_sample = time.perf_counter() - t0
        N = sum(int(sm.total_samples) for sm in sampled.values())
        for i in range(args.warmup):  # JIT compile (first) + warm caches on a short slice
            R.generate(rscene, sampled, rfx[:2], cfg, workers=threads)
        for s in range(args.steps):
            a = (s * per_step) % max(1, len(rfx) - per_step + 1)
            t0 = time.perf_counter()
            R.generate(rscene, sampled, rfx[a:a + per_step], cfg, workers=threads)
            times.append(time.perf_counter() - t0)
        kind = "reference"
        how = (f"unmodified reference package (baseline/_ref, numba {numba.__version__}, "
               f"{numba.get_num_threads()} threads, layer {numba.threading_layer()}), "
               f"gazemap.generate(workers={threads}); build_sampled_meshes {t_sample * 1e3:.0f} ms (not in the step)")
    else:
        from oracle import oracle as O

        lay = O.build_layouts(scene, k)
        N = sum(v[3] for v in lay.values())
        rows = O.rows_as_fixations(fx)
        for i in range(args.warmup):
            O.generate(scene, rows[:2], k=k, filtering_enabled=filtering, threads=threads, layouts=lay)
        for s in range(args.steps):
            a = (s * per_step) % max(1, len(rows) - per_step + 1)
            t0 = time.perf_counter()
            O.generate(scene, rows[a:a + per_step], k=k, filtering_enabled=filtering, threads=threads, layouts=lay)
            times.append(time.perf_counter() - t0)
        kind = "port"
        how = "C port of the reference algorithm (oracle/gm_oracle.c, OpenMP); baseline/_ref not installed"
    t = sum(times) / len(times)
    v = N * per_step / t
    sample = f"{per_step} consecutive fixations of the workload per step (N = {N} samples), {how}"
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == "c4" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "samples": int(N), "fixations_per_step": per_step,
                   "ms_per_fixation": t * 1e3 / per_step, "extrapolated_full_map_s": t / per_step * len(fx),
                   "note": "bounded prefix per step; the per-fixation loop (density.py:223-226) is sequential, "
                           "so its cost scales linearly with the fixation count"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------- our arm

def _peaks(lib, device, peaks):
    """Measured FP64 / FP32 FMA peaks (gm_peak_flops) with the driver's HBM figure."""
    from paper_2601_07571_b200 import _native

    out = {}
    for name, fp64 in (("fp64", 1), ("fp32", 0)):
        v = np.zeros(1)
        rc = lib.gm_peak_flops(device, fp64, _native.dptr(v))
        out[name] = float(v[0]) if rc == 0 and v[0] > 0 else None
    clk = peaks.get("sm_max_mhz", 1965.0) / 1e3
    out["fp64_nominal"] = 148 * 64 * 2 * clk / 1e3
    out["fp32_nominal"] = 148 * 128 * 2 * clk / 1e3
    out["hbm_gbs"] = peaks.get("hbm_gbs")
    out["how"] = ("FMA loops in the extension (gm_peak_flops: 8 independent chains/thread, 148x8 CTAs of 256, "
                  "best of 3 after warm-up, CUDA events), measured in this run; HBM from MEASURED_PEAKS.json")
    return out


def _ncu_kernels():
    for name in ("r2_ncu_traffic.json", "r1_ncu_traffic.json"):
        p = ROOT / "profiles" / name
        if p.exists():
            d = json.loads(p.read_text())
            return d.get("kernels", {}), f"profiles/{name}"
    return {}, None


def _roofline(st, tm1, ms1, batches, pk, clk_mhz):
    """Roofline views of the dominant kernel (k_texels, both launches of a
    batch) and SURVEY 8d's whole-step figure.  Times are per-batch averages
    from the untimed single-stream pass (CUDA events on the stream the kernels
    run on); counts from the instrumented pass of the same workload."""
    times = {"k_samples<mark>": tm1.mark_ms, "k_texels": tm1.texel_ms, "k_samples<accumulate>": tm1.accumulate_ms,
             "k_tri_setup": tm1.cull_ms}
    dom = max(times, key=times.get)
    t_s = times["k_texels"] / 1e3
    launch_ms = times["k_texels"] / max(batches, 1)
    fp64 = pk["fp64"] or pk["fp64_nominal"]
    # SURVEY 8d raster definition: the reference rasterizer's FP64 pixel tests -- every pixel of
    # every culled-in triangle's clamped bbox: px+0.5 and three 5-flop edge functions = 16 flops
    # (kernels.py:104-111); counted per batch by k_coarse (bbox_px)
    raster_flops = 16.0 * st.get("bbox_px", 0)
    raster_tf = raster_flops / t_s / 1e12 if t_s and raster_flops else None
    # this design's exact work: one exact pixel test of the writer per marked texel -- 3 edge
    # functions (15) + l_i, inv_w, 1/inv_w (9) + cx, cy, bbox-local shift (8) = 32 FP64 flops
    texel_flops = 32.0 * st.get("texels", 0)
    texel_tf = texel_flops / t_s / 1e12 if t_s and texel_flops else None
    kern, src = _ncu_kernels()
    def pick(*prefixes):  # the production instantiation of each pass (template arguments vary by round)
        for pre in prefixes:
            for name, v in kern.items():
                if name.startswith(pre):
                    return v
        return None

    k1 = pick("k_texels<0, 0, 0", "k_texels<0, 0, 0, 0>")
    k2 = pick("k_texels_crowded<0, 0, 0", "k_texels<0, 0, 1, 0>")
    traffic = hbm = issue = None
    if k1:
        traffic = k1["dram_bytes_per_launch"] + (k2["dram_bytes_per_launch"] if k2 else 0.0)
        gbs = traffic / (launch_ms / 1e3) / 1e9 if launch_ms else None
        hbm = {"achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
               "frac": gbs / pk["hbm_gbs"] if gbs and pk["hbm_gbs"] else None,
               "bytes_per_batch": traffic, "launch_ms": launch_ms,
               "definition": "DRAM bytes of both k_texels launches of one batch (ncu) / their live time"}
        if "inst_executed_per_launch" in k1:
            inst = k1["inst_executed_per_launch"] + (k2.get("inst_executed_per_launch", 0.0) if k2 else 0.0)
            rate = inst / (launch_ms / 1e3) if launch_ms else None
            peak = 4.0 * 148 * clk_mhz * 1e6
            issue = {"achieved": rate / 1e9 if rate else None, "peak": peak / 1e9, "unit": "Gwarp-inst/s",
                     "frac": rate / peak if rate else None, "inst_per_batch": inst,
                     "definition": "warp instructions of both launches (ncu smsp__inst_executed.sum) / live time "
                                   "vs 4 issue slots x 148 SMs x max SM clock"}
    roof = {"bound": "fp64", "achieved": raster_tf, "peak": fp64, "unit": "TFLOP/s",
            "frac": raster_tf / fp64 if raster_tf else None, "traffic": traffic,
            "kernel": "k_texels (first pass + crowded pass, per batch)", "dominant_phase": dom,
            "kernel_ms_per_step": times["k_texels"], "kernel_share": times["k_texels"] / ms1 if ms1 else None,
            "definition": "SURVEY 8d raster work: 16 FP64 flops per reference pixel test (bbox pixels of the "
                          "culled-in screen triangles, kernels.py:104-111) / k_texels time; an effective rate -- "
                          "k_texels evaluates only the texels the depth tests read, so it can exceed 1",
            "peak_kind": "measured FP64 FMA peak (gm_peak_flops)" if pk["fp64"] else "nominal FP64 (no measurement)",
            "views": {"marked_texels": {"achieved": texel_tf, "peak": fp64, "unit": "TFLOP/s",
                                        "frac": texel_tf / fp64 if texel_tf else None,
                                        "definition": "32 FP64 flops per marked texel (the writer's exact pixel "
                                                      "test) / k_texels time"},
                      "hbm": hbm, "issue": issue},
            "ncu_source": src, "work": st}
    return roof


def run_ours(args, rank, world):
    import paper_2601_07571_b200 as gm
    from paper_2601_07571_b200 import _native, density

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
    lib = _native.load()
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(peaks_path.read_text()) if peaks_path.exists() else {}
    pk = _peaks(lib, device, peaks)

    # the job's whole stream for the sharded API calls (each rank generates its contiguous shard).
    # Weak scaling: the job stream is the ranks' streams back to back; generate_sharded on rank r
    # reads only rows [r F, (r + 1) F), so the other ranks' rows are placeholders here (same
    # shape, not read) instead of regenerating every rank's 100k-fixation stream on every rank
    job_fx = None
    if world > 1:
        job_fx = fx_all if scaling == "strong" else np.concatenate([fx_all] * world)

    # ---- map generation time, cold: build_sampled_meshes + generate + normalize on
    # in-memory inputs with a fresh plan (scene upload, sampling, buffer allocation all inside)
    cold = None
    if not args.no_cold and not args.no_e2e:
        cold_ms, stages = [], None
        for rep in range(2):
            density.release_plans()
            gc.collect()
            # settle: the previous plan's cudaFree of ~20 GB must not land in the next allocation
            _native.check(lib.gm_normalize(device, _native.dptr(np.ones(8)), 8, 1.0, _native.dptr(np.empty(8))))
            if world > 1:
                dist.barrier()
            tmr = gm.Timings()
            t0 = time.perf_counter()
            sampled_c = gm.build_sampled_meshes(scene, k, device=device)
            t1 = time.perf_counter()
            if world > 1:
                from paper_2601_07571_b200.sharding import generate_sharded

                dm = generate_sharded(scene, sampled_c, job_fx, cfg, device=device, collective=args.collective,
                                      timers=tmr)
            else:
                dm = gm.generate(scene, sampled_c, fx, cfg, device=device, timers=tmr)
            nm = gm.normalize(dm, timers=tmr, device=device)
            t2 = time.perf_counter()
            cold_ms.append((t2 - t0) * 1e3)
            ph = dict(tmr.phases)
            stages = {"build_sampled_meshes": (t1 - t0) * 1e3,
                      **{k2: v * 1e3 for k2, v in ph.items()}}
            del dm, nm, sampled_c
        cold = {"ms": float(min(cold_ms)), "reps_ms": cold_ms, "pairs_per_s": None, "stages_ms": stages,
                "definition": "wall time of build_sampled_meshes + generate + normalize from in-memory inputs, "
                              "fresh ScenePlan (upload, sampling, buffer allocation included), CUDA initialised; "
                              "stages: device phases are per-batch event spans of overlapped streams"}

    sampled = gm.build_sampled_meshes(scene, k, device=device)
    plan = density.get_plan(scene, sampled, cfg, device)
    N = plan.n_samples
    F = len(fx)
    if cold is not None:
        cold["pairs_per_s"] = N * total_F / (cold["ms"] / 1e3)
    ccfg = _native.GmConfig(cfg.theta, cfg.epsilon_abs, cfg.epsilon_rel, cfg.zbuffer_resolution,
                            int(filtering), args.batch, 0)
    bad = np.zeros(1, np.int64)
    _native.check(lib.gm_plan_prepare(plan._h, _native.dptr(fx), F, ctypes.byref(ccfg), _native.iptr(bad)))

    coll_used, reduce_ms = None, []
    if world > 1:
        from paper_2601_07571_b200.sharding import reduce_peers

    def one_step():
        tm = _native.GmTimings()
        ms = ctypes.c_float(0.0)
        _native.check(lib.gm_plan_run(plan._h, 1, 0, ctypes.byref(tm), ctypes.byref(ms)), "gm_plan_run")
        extra = 0.0
        if world > 1:
            # the ranks' partial maps -> the sum on every rank + global max (device ms of
            # this rank's fused peer-reduce kernel, or of NCCL's all-reduce)
            nonlocal coll_used
            gmax, coll_used, extra = reduce_peers(plan, None, args.collective)
            reduce_ms.append(extra)
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
    # (N > 1: k_reduce_peers instead of k_max)
    launches = int(tm.batches) * 8 + 2
    library_launches = int(tm.batches) * 4

    # ---- e2e through the public API (host table in, host values out), every timed step ----
    # fixation table (host) -> host setup -> H2D of the setup records -> kernels -> D2H of the values.
    # N > 1: sharding.generate_sharded over the job's stream (each rank's contiguous shard) with the
    # peer reduce inside the timed region.
    e2e = None
    if not args.no_e2e:
        if world > 1:
            from paper_2601_07571_b200.sharding import generate_sharded

            def e2e_call(tmr=None):
                return generate_sharded(scene, sampled, job_fx, cfg, device=device, collective=args.collective,
                                        timers=tmr)
        else:
            def e2e_call(tmr=None):
                return gm.generate(scene, sampled, fx, cfg, device=device, timers=tmr)
        e2e_call()  # warm
        e_times, tmr = [], None
        for _ in range(max(1, args.steps)):
            if world > 1:
                dist.barrier()
            tmr = gm.Timings()
            t0 = time.perf_counter()
            e2e_call(tmr)
            e_times.append(time.perf_counter() - t0)
        e_t = float(np.mean(e_times))
        if world > 1:
            import torch

            tt = torch.tensor([e_t], device=f"cuda:{device}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_t = float(tt.item())
        e2e = {"value": N * total_F / e_t, "unit": UNIT, "h2d_bytes_per_step": int(F * (208 + 80)),
               "d2h_bytes_per_step": int(N * 8), "ms_per_step": e_t * 1e3, "samples": len(e_times),
               "stages_ms_last": {k2: v * 1e3 for k2, v in tmr.phases.items()} if tmr else None,
               "path": "paper_2601_07571_b200.generate (fixation table in host memory -> values dict)"
               if world == 1 else "paper_2601_07571_b200.sharding.generate_sharded (partial maps + peer reduce)",
               "timing": "host wall clock around the API call, mean of `steps` warm calls (plan cached); "
                         "stages: host setup / upload / readback wall, device phases as overlapped event spans"}
        if cold is not None:
            e2e["cold"] = cold

    # ---- algorithmic work of this step (one instrumented, untimed pass) ----
    stats = (ctypes.c_uint64 * len(_native.STAT_NAMES))()
    tm_s = _native.GmTimings()
    ms_s = ctypes.c_float(0.0)
    if not args.no_stats:
        _native.check(lib.gm_plan_run(plan._h, 1, _native.GM_FLAG_STATS, ctypes.byref(tm_s), ctypes.byref(ms_s)))
        _native.check(lib.gm_plan_stats(plan._h, stats))
    st = dict(zip(_native.STAT_NAMES, [int(x) for x in stats]))
    # per-kernel device time: the timed steps overlap batches on several streams, so their per-phase
    # events include concurrent work; one more untimed pass on a single stream gives each kernel's own
    # time (CUDA events on the stream it runs on)
    tm1 = _native.GmTimings()
    ms1 = ctypes.c_float(0.0)
    if not args.no_stats:
        _native.check(lib.gm_plan_run(plan._h, 1, _native.GM_FLAG_ONE_STREAM, ctypes.byref(tm1), ctypes.byref(ms1)))
    else:
        tm1 = tm
    clk_mhz = peaks.get("sm_max_mhz", 1965.0)
    roof = _roofline(st, tm1, ms1.value, int(tm1.batches), pk, clk_mhz)
    if e2e is not None and ms1.value > 0:
        # SURVEY 8d per-stage split of the warm end-to-end call: host stages from the call's own wall
        # clocks; the device step (overlapped streams) apportioned by the single-stream phase shares
        last = e2e.get("stages_ms_last") or {}
        dev = step_ms
        share = {k2: v / ms1.value for k2, v in (("cull+project", tm1.cull_ms), ("filter+mark", tm1.mark_ms),
                                                 ("raster (texels)", tm1.texel_ms),
                                                 ("accumulate", tm1.accumulate_ms))}
        e2e["split_ms"] = {"host setup (fixation table -> setup records)": last.get("setup"),
                           **{k2: dev * v for k2, v in share.items()},
                           "other device (sorts, coarse bins, overlap)": dev * (1.0 - sum(share.values())),
                           "global max": last.get("max"), "D2H read-back": last.get("readback"),
                           "end-to-end (measured)": e2e["ms_per_step"]}
        e2e["split_note"] = ("H2D of the setup records (h2d_bytes_per_step) rides inside the device step, "
                             "one 288-byte record per fixation, overlapped with the previous batch")
    # SURVEY 8d's step roofline: algorithmic FLOPs of the reference's per-pair work -- 26 per nominal
    # sample-fixation pair (camera transform + NDC projection, kernels.py:305-315) + 43 per NDC candidate
    # (depth test + Gaussian, :323-340) -- over the whole step, against the measured FP32 FMA peak (the
    # path computes in FP64 for parity; the FP32 peak is the survey's yardstick).  Culling means most
    # nominal pairs are never evaluated: an effective rate.
    fp32_peak = pk["fp32"] or pk["fp32_nominal"]
    step_flops = 26.0 * N * F + 43.0 * st.get("ndc_candidates", 0)
    step_tf = step_flops / (step_ms / 1e3) / 1e12 if st.get("ndc_candidates") else None
    roof_step = {"bound": "fp32", "achieved": step_tf, "peak": fp32_peak, "unit": "TFLOP/s",
                 "frac": step_tf / fp32_peak if step_tf else None, "algorithmic_flops_per_step": step_flops,
                 "definition": "SURVEY.md 8d: (26 N F + 43 sum C_ndc) / t / P_FP32 (per rank, measured FP32 peak)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            n_cpu = args.cpu_fixations or (200 if args.config == "c1" else 1000)
            v, dt, _ = cpu_port_pairs_per_s(scene, k, fx, filtering, n_cpu, host_threads())
            cpu = {"value": v, "unit": UNIT, "cores": host_threads(), "kind": "port",
                   "sample": f"first {n_cpu} fixations of the workload ({dt:.1f} s), oracle/gm_oracle.c with OpenMP"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": host_threads(), "kind": "port", "sample": f"failed: {e}"}

    multi = None
    if world > 1:
        nv = 2.0 * (world - 1) / world * 8.0 * N if coll_used == "p2p" else None
        rms = float(np.mean(reduce_ms)) if reduce_ms else None
        multi = {"collective": coll_used, "reduce_ms_mean": rms,
                 "nvlink_bytes_per_rank": nv,
                 "nvlink_gbs_per_rank": nv / (rms / 1e3) / 1e9 if nv and rms else None,
                 "fixations_per_rank": int(F)}
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
                       "timing": "CUDA events on the plan stream around each full generation (+ reduce), max over ranks"},
            "e2e": e2e, "roofline": roof, "roofline_step_fp32": roof_step, "peaks": pk, "cpu_baseline": cpu,
            "clocks": clk.summary(), "gpu_launches": launches, "library_launches": library_launches,
            "multi_gpu": multi,
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if args.impl == "reference" else 1))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
