"""Fused peer reduce of fixation-sharded partial maps (sharding.reduce_peers,
gm_plan_reduce_peers): two ranks share cuda:0 here (CUDA IPC maps a peer
process's accumulator on the same device exactly as it maps a peer GPU's over
NVLink), gloo carries the handle exchange.  The reduced map must be the rank-
order sum of the partial maps bit for bit, identical on both ranks, and equal
to a single-process generate within the reference's partition tolerance
(t/test_density.py:139-155)."""

import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _scene():
    import workloads as W

    return W.rotated_object_scene(), W.orbit_fixations(24, 5, 1.5, 3.5, jitter=0.4)


def _worker(rank, world, port, out_dir):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2601_07571_b200 as gm
    from paper_2601_07571_b200.density import get_plan
    from paper_2601_07571_b200.sharding import generate_sharded, reduce_peers, shard_range

    scene, fx = _scene()
    cfg = gm.GenerationConfig(k=1500.0)
    sampled = gm.build_sampled_meshes(scene, cfg.k)
    a, b = shard_range(len(fx), rank, world)
    plan = get_plan(scene, sampled, cfg, 0)
    plan.accumulate_log(fx[a:b], cfg, reset=True)
    plan.sync()
    partial = plan.read()
    gmax, used, ms = reduce_peers(plan, None, "p2p")
    reduced = plan.read()
    # the API path (collective "auto") on a fresh accumulation
    dm = generate_sharded(scene, sampled, fx, cfg)
    api = np.concatenate([dm.values[o.object_id] for o in scene.objects])
    # the collective fallback (all_reduce on the zero-copy torch view of the accumulator; NCCL in
    # production, gloo here) on a fresh accumulation of the same shard
    plan.accumulate_log(fx[a:b], cfg, reset=True)
    plan.sync()
    gmax_c, used_c, _ = reduce_peers(plan, None, "nccl")
    coll = plan.read()
    # ranks whose plans hold different sample layouts must refuse to reduce
    inc = gm.GenerationConfig(k=1500.0, object_include_list={scene.objects[0].object_id} if rank else None)
    other = get_plan(scene, sampled, inc, 0)
    try:
        reduce_peers(other, None, "auto")
        mismatch = "no error"
    except ValueError as e:
        mismatch = str(e)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), partial=partial, reduced=reduced, gmax=gmax, used=used,
             ms=ms, api=api, api_gmax=dm.global_max, coll=coll, gmax_c=gmax_c, used_c=used_c, mismatch=mismatch)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_peer_reduce_bitwise():
    import torch.multiprocessing as mp

    import paper_2601_07571_b200 as gm

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        r = [dict(np.load(os.path.join(d, f"r{i}.npz"))) for i in range(2)]
    assert str(r[0]["used"]) == "p2p" and str(r[1]["used"]) == "p2p"
    want = r[0]["partial"] + r[1]["partial"]  # rank order, as k_reduce_peers sums
    np.testing.assert_array_equal(r[0]["reduced"], want)
    np.testing.assert_array_equal(r[1]["reduced"], want)
    assert float(r[0]["gmax"]) == float(want.max()) == float(r[1]["gmax"])
    np.testing.assert_array_equal(r[0]["api"], r[1]["api"])
    np.testing.assert_array_equal(r[0]["api"], want)
    for k in range(2):  # collective fallback: a + b of two operands is the same bits in either order
        assert str(r[k]["used_c"]) == "nccl"
        np.testing.assert_array_equal(r[k]["coll"], want)
        assert float(r[k]["gmax_c"]) == float(want.max())
        assert "different sample layouts" in str(r[k]["mismatch"])
    # single-process generate: additivity within the reference's partition tolerance
    scene, fx = _scene()
    cfg = gm.GenerationConfig(k=1500.0)
    sampled = gm.build_sampled_meshes(scene, cfg.k)
    full = gm.generate(scene, sampled, fx, cfg)
    flat = np.concatenate([full.values[o.object_id] for o in scene.objects])
    assert flat.max() > 0
    np.testing.assert_allclose(want, flat, rtol=1e-12, atol=0.0)
    assert float(r[0]["api_gmax"]) == pytest.approx(full.global_max, rel=1e-12)
