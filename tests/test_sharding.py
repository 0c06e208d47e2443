"""Fixation sharding across ranks (world_size 2, gloo, CPU): partition,
sum all-reduce of the partial maps, max after the reduce.  The per-rank
compute is the CPU oracle here (the GPU path is covered by -m gpu tests);
what is under test is the host-side sharding / reduction logic."""

import os
import socket
import tempfile

import numpy as np
import pytest

from paper_2601_07571_b200.sharding import shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 101):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _oracle_compute(scene, sampled, table, config):
    from oracle import oracle as O

    vals, _ = O.generate(scene, O.rows_as_fixations(table), k=config.k, theta=config.theta,
                         zbuffer_resolution=config.zbuffer_resolution, filtering_enabled=config.filtering_enabled,
                         object_include_list=config.object_include_list)
    ids = [o.object_id for o in scene.objects]
    inc = [i for i in ids if config.object_include_list is None or i in config.object_include_list]
    return np.concatenate([vals[i] for i in inc]) if inc else np.zeros(0)


def _worker(rank, world, port, out_dir):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2601_07571_b200 as gm
    import workloads as W
    from oracle import oracle as O
    from paper_2601_07571_b200.sharding import generate_sharded

    scene = W.rotated_object_scene()
    fx = W.orbit_fixations(9, 3, 1.5, 3.5, jitter=0.4)
    cfg = gm.GenerationConfig(k=1500.0)
    lay = O.build_layouts(scene, cfg.k)
    sampled = {oid: gm.SampledMesh(oid, r, c, o, t, cfg.k) for oid, (r, c, o, t) in lay.items()}
    dm = generate_sharded(scene, sampled, fx, cfg, local_compute=_oracle_compute)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), gmax=dm.global_max,
             **{f"v_{k}": v for k, v in dm.values.items()})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_sharded_equals_single():
    import torch.multiprocessing as mp

    import workloads as W
    from oracle import oracle as O

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        r0 = dict(np.load(os.path.join(d, "r0.npz")))
        r1 = dict(np.load(os.path.join(d, "r1.npz")))
    scene = W.rotated_object_scene()
    fx = W.orbit_fixations(9, 3, 1.5, 3.5, jitter=0.4)
    full, gmax = O.generate(scene, O.rows_as_fixations(fx), k=1500.0)
    assert gmax > 0
    for oid, v in full.items():
        np.testing.assert_array_equal(r0[f"v_{oid}"], r1[f"v_{oid}"])  # every rank holds the reduced map
        np.testing.assert_allclose(r0[f"v_{oid}"], v, rtol=1e-12, atol=0.0)  # additivity
    assert float(r0["gmax"]) == pytest.approx(gmax, rel=1e-12)
