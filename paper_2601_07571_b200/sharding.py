"""Fixation-sharded generation across GPUs (one process per GPU).

Fixations are independent and their contributions add (
reference test_density.py:139-155), so rank r accumulates its contiguous
shard of the fixation log into a partial map on its own GPU, one sum
all-reduce combines the partial maps, and the global max is taken on the
reduced buffer (the max of per-rank maxima is not the max of the sum).

Plumbing is torch.distributed: NCCL over NVLink/NVSwitch for CUDA ranks,
gloo for the CPU tests.  The partial map stays in HBM: the plan's device
accumulator is wrapped zero-copy as a torch tensor and reduced in place.
"""

from __future__ import annotations

import numpy as np

from .density import DensityMap, GenerationConfig, get_plan
from .gaze import fixation_table

__all__ = ["shard_range", "generate_sharded"]


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


def _gpu_partial(scene, sampled_meshes, shard, config, device):
    """Accumulate on this rank's GPU (pose overrides honoured); return (torch
    tensor aliasing the plan's device values, plan)."""
    import torch

    plan = get_plan(scene, sampled_meshes, config, device)
    plan.accumulate_log(shard, config, reset=True)
    plan.sync()
    t = torch.as_tensor(_CudaArray(plan.values_device_ptr(), plan.n_samples), device=f"cuda:{device}")
    return t, plan


def generate_sharded(scene, sampled_meshes: dict, fixations, config: GenerationConfig, group=None,
                     device: int | None = None, local_compute=None) -> DensityMap:
    """generate() over all ranks of `group` (torch.distributed); every rank
    returns the full reduced, un-normalized map.

    `local_compute(scene, sampled_meshes, table, config) -> flat values` may be
    injected (tests run the CPU oracle here under gloo); by default the shard
    runs on this rank's GPU and the reduce happens in HBM.
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
        vals, plan = _gpu_partial(scene, sampled_meshes, objs, config, dev)
        if world > 1:
            dist.all_reduce(vals, op=dist.ReduceOp.SUM, group=group)
        torch.cuda.synchronize(dev)
        gmax = plan.global_max() if len(table) else 0.0
        values = plan.split(plan.read(), sampled_meshes)
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
