"""Fixation-sharded generation across GPUs (one process per GPU).

Fixations are independent and their contributions add (
reference test_density.py:139-155), so rank r accumulates its contiguous
shard of the fixation log into a partial map on its own GPU, one sum
all-reduce combines the partial maps, and the global max is taken on the
reduced buffer (the max of per-rank maxima is not the max of the sum).

The reduce of the GPU path is this package's own kernel (reduce_peers):
every rank maps its peers' accumulators (CUDA IPC over NVLink/NVSwitch), sums
its slice over the ranks in rank order (the same bits on every rank and every
run), stores the sum into every peer's map and takes the slice max, so the
reduce-scatter, all-gather and global max are one pass over HBM with no
staging copy.  torch.distributed is the plumbing (handle exchange, barriers,
a scalar max); NCCL's all-reduce on the zero-copy tensor view of the
accumulator is the fallback when peer mapping fails on some rank
(collective="nccl" forces it), gloo carries the CPU tests.
"""

from __future__ import annotations

import socket
import time

import numpy as np

from .density import DensityMap, GenerationConfig, get_plan
from .gaze import fixation_table

__all__ = ["shard_range", "generate_sharded", "reduce_peers"]


def shard_range(n: int, rank: int, world: int) -> tuple:
    """Contiguous [start, stop) of rank `rank` when n items split over `world`
    ranks as evenly as possible (first n % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class _CudaArray:
    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


def reduce_peers(plan, group=None, collective: str = "auto") -> tuple:
    """Sum the ranks' partial maps in place on every rank; returns (global max,
    collective used, device ms of this rank's reduce).  Collective over `group`:
    every rank must call it after its partial map is complete."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if collective not in ("auto", "p2p", "nccl"):
        raise ValueError(f"unknown collective {collective!r}")
    # every rank must hold the same sample layout: the peer kernel addresses the
    # peers' maps by this rank's slice bounds, NCCL needs equal buffer lengths
    me = (int(plan.n_samples), socket.gethostname())
    peers = [None] * world
    dist.all_gather_object(peers, me, group=group)
    sizes = sorted({n for n, _ in peers})
    if len(sizes) != 1:
        raise ValueError(f"ranks hold different sample layouts (n_samples {sizes}); cannot reduce their maps")
    same_node = len({h for _, h in peers}) == 1
    if collective == "p2p" and not same_node:
        raise RuntimeError("collective='p2p' needs every rank on one node (CUDA IPC peer mapping)")
    use_p2p = collective != "nccl" and same_node
    if use_p2p:
        handles = [None] * world
        dist.all_gather_object(handles, plan.ipc_handle(), group=group)
        ok = True
        try:
            plan.open_peers(rank, world, b"".join(handles))
        except Exception:
            if collective == "p2p":
                raise
            ok = False
        flags = [None] * world
        dist.all_gather_object(flags, ok, group=group)
        use_p2p = all(flags)
    if use_p2p:
        plan.sync()
        dist.barrier(group=group)  # every partial map is complete
        smax, ms = plan.reduce_peers()
        dist.barrier(group=group)  # every slice is stored in every map
        maxima = [None] * world
        dist.all_gather_object(maxima, smax, group=group)
        return max(maxima), "p2p", ms
    dev = torch.cuda.current_device()
    vals = torch.as_tensor(_CudaArray(plan.values_device_ptr(), plan.n_samples), device=f"cuda:{dev}")
    plan.sync()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    dist.all_reduce(vals, op=dist.ReduceOp.SUM, group=group)
    ev1.record()
    torch.cuda.synchronize(dev)
    return plan.global_max(), "nccl", ev0.elapsed_time(ev1)


def generate_sharded(scene, sampled_meshes: dict, fixations, config: GenerationConfig, group=None,
                     device: int | None = None, local_compute=None, collective: str = "auto",
                     timers=None) -> DensityMap:
    """generate() over all ranks of `group` (torch.distributed); every rank
    returns the full reduced, un-normalized map.

    `local_compute(scene, sampled_meshes, table, config) -> flat values` may be
    injected (tests run the CPU oracle here under gloo); by default the shard
    runs on this rank's GPU and the reduce happens in HBM (reduce_peers;
    `collective` "auto" = peer kernel, NCCL if a rank cannot map its peers).
    """
    import torch
    import torch.distributed as dist

    config.validate()
    table = fixation_table(fixations)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    a, b = shard_range(len(table), rank, world)
    shard = table[a:b]
    if local_compute is None:
        dev = torch.cuda.current_device() if device is None else device
        objs = shard if isinstance(fixations, np.ndarray) else list(fixations)[a:b]
        t0 = time.perf_counter()
        plan = get_plan(scene, sampled_meshes, config, dev)
        if timers is not None:
            timers.add("upload", time.perf_counter() - t0)
        plan.accumulate_log(objs, config, reset=True, timers=timers)
        plan.sync()
        t0 = time.perf_counter()
        if world > 1:
            gmax, _, _ = reduce_peers(plan, group, collective)
        else:
            gmax = plan.global_max()
        gmax = gmax if len(table) else 0.0
        t1 = time.perf_counter()
        values = plan.split(plan.read(), sampled_meshes)
        if timers is not None:
            timers.add("reduce_max", t1 - t0)
            timers.add("readback", time.perf_counter() - t1)
        return DensityMap(values, global_max=gmax)
    flat = np.ascontiguousarray(local_compute(scene, sampled_meshes, shard, config), dtype=np.float64)
    t = torch.from_numpy(flat)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    flat = t.numpy()
    gmax = float(flat.max()) if len(table) and len(flat) else 0.0
    included = [o.object_id for o in scene.objects
                if config.object_include_list is None or o.object_id in config.object_include_list]
    values, o = {}, 0
    for oid in [x.object_id for x in scene.objects]:
        if oid not in sampled_meshes:
            continue
        n = int(sampled_meshes[oid].total_samples)
        if oid in included:
            values[oid] = flat[o:o + n].copy()
            o += n
        else:
            values[oid] = np.zeros(n)
    return DensityMap(values, global_max=max(gmax, 0.0))
