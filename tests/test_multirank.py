"""N>1 host logic on CPU (gloo, world_size 2): the weak-scaling walker sharding
of bench.py (rank r walks global ids r*V + v) and its max/sum reductions.  The
per-rank walks run on the oracle; the GPU arm uses the same ids and reductions
with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist

    import bench
    import oracle
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = oracle.Graph.rmat(9, 16, 3).synth_philox("uniform", 1.0, 5.0, seed=4)
    nv = g.nv
    q = np.arange(nv, dtype=np.uint32)
    r = oracle.run(g, oracle.Model("node2vec", a=0.5, b=2.0), q, walk_length=20, seed=5,
                   ratio=1.3, rng="philox", qid_base=rank * nv)
    ws = r.stats["steps"] - r.stats["dead_ends"]
    total = bench.reduce_sum(ws, dist, torch.device("cpu"))
    slowest = bench.reduce_max(float(rank + 1), dist, torch.device("cpu"))
    np.save(os.path.join(out_dir, f"paths{rank}.npy"), r.paths)
    np.save(os.path.join(out_dir, f"meta{rank}.npy"), np.array([ws, total, slowest]))
    dist.barrier()
    dist.destroy_process_group()


def test_weak_scaling_shards_and_reductions(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import oracle
    g = oracle.Graph.rmat(9, 16, 3).synth_philox("uniform", 1.0, 5.0, seed=4)
    nv = g.nv
    # one process walking both ranks' global ids gives the same paths
    q = np.tile(np.arange(nv, dtype=np.uint32), world)
    full = oracle.run(g, oracle.Model("node2vec", a=0.5, b=2.0), q, walk_length=20, seed=5,
                      ratio=1.3, rng="philox")
    parts = [np.load(tmp_path / f"paths{r}.npy") for r in range(world)]
    assert np.array_equal(full.paths, np.concatenate(parts))
    metas = [np.load(tmp_path / f"meta{r}.npy") for r in range(world)]
    assert metas[0][1] == metas[1][1] == metas[0][0] + metas[1][0]
    assert metas[0][1] == full.stats["steps"] - full.stats["dead_ends"]
    assert metas[0][2] == metas[1][2] == float(world)
    # distinct global ids draw distinct streams
    assert not np.array_equal(parts[0], parts[1])
