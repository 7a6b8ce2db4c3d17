"""N>1 host logic on CPU (gloo, world_size 2): bench.py's walker partitions and
its max/sum reductions and end-of-run path gather.

* strong scaling (the default for --gpus N): the global walker ids are
  hash-partitioned over the ranks (paper_2512_00705_b200.shard_of, the host
  twin of bench.shard_ids) and each walker keeps its global id as stream key,
  so the union of the shards is exactly the one-process run;
* weak scaling (--weak): rank r walks global ids r*V + v.

The per-rank walks run on the oracle here (no GPU); tests/test_gpu_multirank.py
runs the same bench path on the CUDA library."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph():
    import oracle
    return oracle.Graph.rmat(9, 16, 3).synth_philox("uniform", 1.0, 5.0, seed=4)


def _init(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _weak_worker(rank, world, port, out_dir):
    import torch

    import bench
    import oracle
    dist = _init(rank, world, port)
    g = _graph()
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
    mp.spawn(_weak_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import oracle
    g = _graph()
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


def _strong_worker(rank, world, port, out_dir):
    import torch

    import bench
    import oracle
    import paper_2512_00705_b200 as dw
    dist = _init(rank, world, port)
    g = _graph()
    nv = g.nv
    cpu = torch.device("cpu")
    ids = bench.shard_ids(torch, 0, nv, world, rank, cpu)
    host = np.nonzero(dw.shard_of(np.arange(nv), world) == rank)[0]
    assert np.array_equal(ids.numpy(), host), "device and host partitions differ"
    r = oracle.run(g, oracle.Model("node2vec", a=0.5, b=2.0), ids.numpy().astype(np.uint32),
                   walk_length=20, seed=5, ratio=1.3, rng="philox",
                   qids=ids.numpy().astype(np.uint64))
    ws = r.stats["steps"] - r.stats["dead_ends"]
    total = bench.reduce_sum(ws, dist, cpu)
    lengths = torch.from_numpy(r.lengths.astype(np.int32))
    paths = torch.from_numpy(r.paths.view(np.int32))
    ga = bench.gather_shards(torch, dist, cpu, (torch.from_numpy(ids.numpy().astype(np.int32)),
                                                ids, 0), lengths, paths, rank, world, nv,
                             keep=True)
    np.save(os.path.join(out_dir, f"ids{rank}.npy"), ids.numpy())
    np.save(os.path.join(out_dir, f"paths{rank}.npy"), r.paths)
    np.save(os.path.join(out_dir, f"meta{rank}.npy"), np.array([ws, total]))
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered_paths.npy"), ga["paths"].numpy().view(np.uint32))
        np.save(os.path.join(out_dir, "gathered_lengths.npy"), ga["lengths"].numpy())
        np.save(os.path.join(out_dir, "gathered_steps.npy"), np.array([ga["walk_steps_check"]]))
    dist.barrier()
    dist.destroy_process_group()


def test_strong_scaling_hash_partition_matches_one_process(tmp_path):
    world = 2
    mp.spawn(_strong_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import oracle
    g = _graph()
    nv = g.nv
    full = oracle.run(g, oracle.Model("node2vec", a=0.5, b=2.0), np.arange(nv, dtype=np.uint32),
                      walk_length=20, seed=5, ratio=1.3, rng="philox")
    ids = [np.load(tmp_path / f"ids{r}.npy") for r in range(world)]
    # a partition: disjoint, covering, and balanced
    allids = np.sort(np.concatenate(ids))
    assert np.array_equal(allids, np.arange(nv))
    assert all(abs(len(i) - nv / world) < 0.05 * nv for i in ids)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"paths{r}.npy"), full.paths[ids[r]])
    metas = [np.load(tmp_path / f"meta{r}.npy") for r in range(world)]
    assert metas[0][1] == metas[1][1] == full.stats["steps"] - full.stats["dead_ends"]
    # the end-of-run gather reassembles the one-process output in query order
    assert np.array_equal(np.load(tmp_path / "gathered_paths.npy"), full.paths)
    assert np.array_equal(np.load(tmp_path / "gathered_lengths.npy"),
                          full.lengths.astype(np.int32))
    assert np.load(tmp_path / "gathered_steps.npy")[0] == metas[0][1]


def test_shard_of_spreads_consecutive_ids():
    import paper_2512_00705_b200 as dw
    for world in (2, 4, 8):
        s = dw.shard_of(np.arange(1 << 16), world)
        counts = np.bincount(s, minlength=world)
        assert counts.min() > 0.95 * (1 << 16) / world
        # no long runs of one rank
        assert np.mean(s[1:] == s[:-1]) < 0.5
