"""bench.py's multi-rank path on the CUDA library (-m gpu).

`bench.py --gpus 2` re-executes itself under torch.distributed.run; here both
ranks share cuda:0 with the gloo backend (--device 0 --backend gloo), the only
way to run two ranks on a one-GPU box.  Each rank builds the graph, walks its
hash-partitioned shard of the global walker ids through dw_run_device (the
timed path) and dw_run_compact (the e2e path) and gathers the shards to rank
0; the union of the shards must equal the one-rank run of the same command."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

ARGS = ["--scale", "12", "--steps", "1", "--warmup", "0", "--no-cpu-baseline",
        "--e2e-steps", "1", "--ratio", "1.3", "--walk-length", "40"]


def _bench(extra, tmp):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + ARGS + extra,
                         capture_output=True, text=True, env=env, cwd=tmp, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def _load(d, world):
    parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    ids = np.concatenate([p["qids"] for p in parts])
    order = np.argsort(ids)
    lengths = np.concatenate([p["lengths"] for p in parts])[order]
    paths = np.concatenate([p["paths"] for p in parts])[order]
    return ids[order], lengths, paths, parts


def test_two_ranks_strong_scaling_equals_one_rank(tmp_path):
    one = _bench(["--dump", str(tmp_path / "one")], tmp_path)
    two = _bench(["--gpus", "2", "--device", "0", "--backend", "gloo", "--gather",
                  "--dump", str(tmp_path / "two")], tmp_path)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["scaling"] == "strong"
    nv = 1 << 12
    assert one["walkers_per_step"] == two["walkers_per_step"] == nv
    # the shards partition the global walker ids and walk them bit-exactly
    i1, l1, p1, _ = _load(tmp_path / "one", 1)
    i2, l2, p2, parts = _load(tmp_path / "two", 2)
    assert np.array_equal(i1, np.arange(nv)) and np.array_equal(i2, np.arange(nv))
    assert all(0.4 * nv < len(p["qids"]) < 0.6 * nv for p in parts)
    assert np.array_equal(l1, l2) and np.array_equal(p1, p2)
    assert one["walker_steps_per_step"] == two["walker_steps_per_step"]
    # the end-of-run gather saw every walker; the e2e leg ran on both ranks
    assert two["gather"]["walkers"] == nv
    assert two["gather"]["walk_steps_check"] == two["walker_steps_per_step"]
    assert two["e2e"]["value"] > 0 and two["e2e"]["h2d_bytes_per_step"] == nv * 12


def test_weak_scaling_two_ranks(tmp_path):
    two = _bench(["--gpus", "2", "--device", "0", "--backend", "gloo", "--weak",
                  "--dump", str(tmp_path / "w")], tmp_path)
    assert two["scaling"] == "weak" and two["walkers_per_step"] == 2 * (1 << 12)
    _, _, _, parts = _load(tmp_path / "w", 2)
    assert np.array_equal(parts[1]["qids"], parts[0]["qids"] + (1 << 12))


def test_too_many_gpus_fails_loudly(tmp_path):
    import torch
    n = torch.cuda.device_count()
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus",
                          str(n + 1)] + ARGS, capture_output=True, text=True, env=env,
                         cwd=tmp_path, timeout=300)
    assert out.returncode == 2
    assert "CUDA device(s) visible" in out.stdout
