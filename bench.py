#!/usr/bin/env python
"""Benchmark: walker-steps/sec for node2vec on R-MAT scale-24 (BASELINE.json configs[1]).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config C]

--config selects another BASELINE.json config (1: s16 node2vec (2, 0.5); 3:
MetaPath s22; 4: PR2 on Pareto-weighted s25); the default is the headline, 2.

One step = one full walk batch: every vertex of the R-MAT s24 ef16 graph
(uniform [1,5) weights) starts one node2vec walker (a=p=0.5, b=q=2, 80
steps, adaptive eRJS/eRVS with the device-calibrated cost ratio).  One
process per GPU, graph replicated, no collective in the hot loop.

--gpus N: N ranks, one per GPU.  Launched without torchrun, bench.py re-executes
itself under torch.distributed.run (fails if fewer than N GPUs are visible).
Scaling is strong by default (BASELINE configs[1]: "walkers sharded across
2/4/8"): the V global walker ids are hash-partitioned over the ranks
(paper_2512_00705_b200.shard_of; hash beats range partitioning)
and each walker keeps its global id as RNG key, so the union of the shards is
exactly the 1-GPU run.  --weak: every rank walks one walker per vertex with
global ids rank * V + v.  `value` is the walker-steps of all ranks over the
slowest rank's time.  --gather: after timing, NCCL-gathers every rank's path
shard to rank 0 (the optional end-of-run gather) and reports
its time.  Inputs are resident in HBM when
the timed region starts; the graph (2.7 GB) is far larger than L2 (126 MB),
so no L2 flush is needed between steps.

--impl reference times the reference's own CPU run_queries
(oracle/_ref/libdynwalk_ref.so, compiled from the reference sources) on the
host cores, on a bounded walker sample of the same graph (rank 0 only).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "walker-steps/sec (node2vec, R-MAT s24) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "walker-steps/s"
# BASELINE.json configs (1-based, as listed there).  The driver runs the
# default, configs[1] = 2; the others are for DESIGN.md's per-config table.
CONFIGS = {
    1: dict(scale=16, model="node2vec", a=2.0, b=0.5, weights="uniform", labels=None,
            desc="node2vec p=2 q=0.5, length 80, one walker per node, weighted R-MAT s16 ef16"),
    2: dict(scale=24, model="node2vec", a=0.5, b=2.0, weights="uniform", labels=None,
            desc="node2vec p=0.5 q=2, walk length 80, one walker per vertex, weighted R-MAT "
                 "scale-24 ef16 (BASELINE configs[1])"),
    3: dict(scale=22, model="metapath", schema=(0, 1, 2, 3) * 20, weights="uniform",
            labels=(0, 3), cheaper_mix=True,
            desc="MetaPath schema (0,1,2,3) repeated to length 80, R-MAT s22 ef16, labels "
                 "uniform [0,3], uniform [1,5) weights"),
    # tier-2 sampling (erjs_handoff = 0.05): the reference's PR2 bounds run
    # ~6,100 trials per step at s20 and more at larger scales, so
    # an eRJS step hands off to the reservoir after trials worth 1/20 of a
    # pass over the row; the distribution is exact (chi-square tested), the
    # random stream differs from the reference's
    4: dict(scale=25, model="pr2", gamma=0.15, weights="pareto", labels=None, handoff=0.05,
            cheaper_mix=True, steps=2, e2e_steps=1,
            desc="second-order PR gamma=0.15 (no restart in the reference, SURVEY 7.3), "
                 "R-MAT/Kronecker s25 ef16, Pareto alpha=1 weights, tier-2 eRJS hand-off"),
    # 10 walkers per vertex (qid = r*V + v): 1.34B walkers, 435 GB of padded
    # paths per pass: one round of 134M walkers (43.5 GB) at a time in HBM
    5: dict(scale=27, model="node2vec", a=0.5, b=2.0, weights="uniform", labels=None,
            walkers_per_vertex=10,
            desc="node2vec p=0.5 q=2, walk length 80, 10 walkers per vertex, weighted R-MAT "
                 "s27 ef16 (2.1B edges in one GPU's HBM); paths written to HBM per walker "
                 "round (timed), streamed to host per round (e2e)"),
}
TOPO_SEED, WEIGHT_SEED, WALK_SEED, PROFILE_SEED, LABEL_SEED = 1, 2, 7, 5, 3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed passes (default 5; config 4: 2, an 81 s pass at s25)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS),
                    help="BASELINE.json config (2 = the headline)")
    ap.add_argument("--scale", type=int, default=0, help="override the config's R-MAT scale")
    ap.add_argument("--walk-length", type=int, default=80)
    ap.add_argument("--discard-paths", action="store_true",
                    help="experiments: walk without writing paths (lengths only)")

    ap.add_argument("--mode", default="adaptive")
    ap.add_argument("--handoff", type=float, default=-1.0,
                    help="tier-2 eRJS hand-off (dw_run_opts.erjs_handoff); default: the "
                         "config's (1 for config 4, else 0 = the reference's rule)")
    ap.add_argument("--ratio", type=float, default=0.0, help="override the calibrated ratio")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="timed end-to-end passes (default 3; config 4: 1)")
    ap.add_argument("--calib", default="micro", choices=["tune", "micro"],
                    help="ratio calibration: K4 micro-passes (profile_edge_cost_ratio, the "
                         "reference's method), or those refined by walking (dw_tune_ratio)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true",
                    help="build + 1 warm walk + 1 walk, for ncu (no JSON line)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank walks one walker per vertex")
    ap.add_argument("--gather", action="store_true",
                    help="gather the path shards to rank 0 after timing (NCCL)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: tests, several ranks on one GPU)")
    ap.add_argument("--device", type=int, default=-1,
                    help="CUDA device of every rank (tests); default LOCAL_RANK")
    ap.add_argument("--dump", default="",
                    help="directory: each rank saves its shard's global ids, lengths and "
                         "paths of the last timed step (tests)")
    a = ap.parse_args()
    a.cfg = dict(CONFIGS[a.config])
    if a.scale:
        a.cfg["scale"] = a.scale
    a.scale = a.cfg["scale"]
    if a.handoff < 0:
        a.handoff = a.cfg.get("handoff", 0.0)
    # per-config pass counts so that every default run ends within minutes
    if a.steps is None:
        a.steps = a.cfg.get("steps", 5)
    if a.e2e_steps is None:
        a.e2e_steps = a.cfg.get("e2e_steps", 3)
    return a


def metric(args) -> str:
    if args.config == 2 and args.scale == 24:
        return METRIC
    c = args.cfg
    return f"walker-steps/sec ({c['model']}, R-MAT s{args.scale}, BASELINE config {args.config})"


def model_kw(cfg) -> dict:
    if cfg["model"] == "node2vec":
        return dict(a=cfg["a"], b=cfg["b"])
    if cfg["model"] == "metapath":
        return dict(schema=tuple(cfg["schema"]))
    return dict(gamma=cfg["gamma"])


def workload(args) -> dict:
    c = args.cfg
    w = "uniform[1,5) f32 weights" if c["weights"] == "uniform" else "Pareto alpha=1 f32 weights"
    if c["labels"]:
        w += f", labels uniform [{c['labels'][0]},{c['labels'][1]}]"
    return {"workload": c["desc"] if args.scale == CONFIGS[args.config]["scale"]
            else c["desc"] + f" (run at scale {args.scale})",
            "graph": f"rmat s{args.scale} ef16 (A,B,C,D)=(.57,.19,.19,.05), mirrored, {w}",
            "model": c["model"], **{k: v for k, v in model_kw(c).items() if k != "schema"},
            "walk_length": args.walk_length, "mode": args.mode,
            "sampling": (f"tier-2: eRJS hand-off after max(32, ceil({args.handoff:g} d / ratio)) "
                         "trials (dw_run_opts.erjs_handoff; distribution-exact, chi-square "
                         "tested; paths equal the oracle with the same rule)" if args.handoff > 0
                         else "tier-1: the reference's decision rule and trial cap (bit-exact)"),
            "walkers": c.get("walkers_per_vertex", 1) * 2 ** args.scale,
            "l2": "inputs larger than L2 (graph >= 2 GB vs 126 MB L2), no flush"}


# ---------------------------------------------------------------- distributed
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def dist_init(world, local, backend):
    import torch
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return dist if world > 1 else None


def reduce_max(x: float, dist, device) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: int, dist, device) -> int:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def self_launch(args) -> None:
    """`bench.py --gpus N` outside torchrun: re-execute under torch.distributed.run
    with N ranks (one per GPU), or fail loudly if N GPUs are not visible."""
    import socket
    if args.device < 0:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) "
                                       "visible"}), flush=True)
            sys.exit(2)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "WARN")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def shard_ids(torch, lo: int, hi: int, world: int, rank: int, dev):
    """Global walker ids in [lo, hi) that rank `rank` walks: the device twin of
    paper_2512_00705_b200.shard_of (Fibonacci hashing; int64 products wrap
    like the uint64 ones, and the mask makes the shift logical)."""
    q = torch.arange(lo, hi, dtype=torch.int64, device=dev)
    if world == 1:
        return q
    h = ((q * (0x9E3779B97F4A7C15 - (1 << 64))) >> 32) & 0xFFFFFFFF
    return q[(h % world) == rank]


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def lib_sha16() -> str:
    """Build identity of the product library: sha256 over its sources, Makefile and
    public header (deterministic, unlike the linked .so)."""
    import glob
    import hashlib
    h = hashlib.sha256()
    pkg = os.path.join(ROOT, "paper_2512_00705_b200")
    files = sorted(glob.glob(os.path.join(pkg, "csrc", "*"))) + [
        os.path.join(pkg, "Makefile"), os.path.join(ROOT, "include", "dynwalk_b200.h")]
    for fn in files:
        h.update(os.path.relpath(fn, ROOT).encode())
        with open(fn, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def ncu_traffic(scale: int, sha: str):
    """Per-launch DRAM bytes of the walk kernel from the committed ncu --set full capture
    (tools/ncu_profile_json.py), only when that capture was taken of this very library
    build (same lib_sha16) on this scale; otherwise null."""
    p = os.path.join(ROOT, "profiles", "ncu_walk_kernel.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    if d.get("scale") != scale or d.get("lib_sha16") != sha:
        return None
    return d.get("dram_bytes_per_launch")


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} in a world of {world} rank(s)")
    devno = args.device if args.device >= 0 else local
    torch.cuda.set_device(devno)
    dev = torch.device("cuda", devno)
    dist = dist_init(world, devno, args.backend)
    cdev = dev if args.backend == "nccl" else torch.device("cpu")  # collective tensors
    import paper_2512_00705_b200 as dw

    t0 = time.perf_counter()
    cfg = args.cfg
    dg = dw.DeviceGraph.rmat(args.scale, 16, seed=TOPO_SEED, weights=cfg["weights"], low=1.0,
                             high=5.0, alpha=1.0, weight_seed=WEIGHT_SEED, labels=cfg["labels"],
                             label_seed=LABEL_SEED, devices=[devno])
    info = dg.info()
    build_s = time.perf_counter() - t0
    model = dw.Model(cfg["model"], **model_kw(cfg))
    # one calibration (rank 0), broadcast so every shard makes the same decisions:
    # K4's micro-pass ratio (profile_edge_cost_ratio), optionally refined by
    # timing the walk kernel at a few thresholds around it (--calib tune)
    ratio = args.ratio
    t0 = time.perf_counter()
    micro = None
    calib = args.calib
    if ratio <= 0:
        ratio = 0.0
        if rank == 0:
            pc = dw.ProfileConfig(seed=PROFILE_SEED)
            micro = dw.profile_edge_cost_ratio(dg, model, cfg=pc)
            ratio = (dw.tune_edge_cost_ratio(dg, model, cfg=pc, walk_length=args.walk_length)
                     if calib == "tune" else micro)
        if dist is not None:
            t = torch.tensor([ratio], dtype=torch.float64, device=cdev)
            dist.broadcast(t, 0)
            ratio = float(t.item())
    calib_s = time.perf_counter() - t0

    nv = info["num_vertices"]
    L = args.walk_length
    wpv = cfg.get("walkers_per_vertex", 1)
    discard = cfg.get("discard_paths", False) or args.discard_paths
    strong = world > 1 and not args.weak
    # one launch per walker round r: global ids r * V + v (weak: (rank * wpv + r) * V + v)
    rounds = []
    for r in range(wpv):
        if strong:
            qid = shard_ids(torch, r * nv, (r + 1) * nv, world, rank, dev)
            queries = (qid - r * nv).to(torch.int32)
            rounds.append((queries, qid, 0))
        else:
            queries = torch.arange(0, nv, dtype=torch.int64, device=dev).to(torch.int32)
            rounds.append((queries, None, (rank * wpv + r) * nv if world > 1 else r * nv))
    n = max(len(q) for q, _, _ in rounds)
    lib = dw.load_library()
    paths = None if discard else torch.empty((max(n, 1), L + 1), dtype=torch.int32, device=dev)
    lengths = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    mdesc = model.c()
    odescs = [dw.RunOptions(mode=args.mode, walk_length=L, seed=WALK_SEED, edge_cost_ratio=ratio,
                            qid_base=base, erjs_handoff=args.handoff,
                            qids=None if qid is None else qid.data_ptr()).c()
              for _, qid, base in rounds]
    graph_bytes = torch.cuda.mem_get_info(dev)

    def step():
        agg = None
        for (q, _, _), od in zip(rounds, odescs):
            rc = lib.dw_run_device(dg.h, 0, C.byref(mdesc), C.c_void_p(q.data_ptr()), len(q),
                                   C.byref(od), C.c_void_p(paths.data_ptr() if paths is not None
                                                           else None),
                                   C.c_void_p(lengths.data_ptr()), C.c_void_p(stream.cuda_stream))
            if rc:
                raise dw.DynwalkError(rc, lib.dw_last_error().decode())
            st = dw.RunStatsC()
            rc = lib.dw_run_device_sync(dg.h, 0, C.byref(st))
            if rc:
                raise dw.DynwalkError(rc, lib.dw_last_error().decode())
            if agg is None:
                agg = st
            else:
                for k in ("steps", "select_erjs", "select_ervs", "trials", "weight_reads",
                          "rng_draws", "erjs_fallbacks", "dead_ends", "algorithmic_bytes",
                          "kernel_launches"):
                    setattr(agg, k, getattr(agg, k) + getattr(st, k))
                agg.kernel_ms += st.kernel_ms
        return agg

    if args.profile_only:
        step()
        step()
        torch.cuda.synchronize()
        return
    for _ in range(args.warmup):
        step()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kms, stats = [], None
    with ClockSampler(devno) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            st = step()
            kms.append(st.kernel_ms)
            stats = st
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    elapsed_ms = reduce_max(elapsed_ms, dist, cdev)
    walker_steps_rank = int(stats.steps - stats.dead_ends)
    walker_steps = reduce_sum(walker_steps_rank, dist, cdev)  # per step, all ranks
    value = walker_steps * args.steps / (elapsed_ms / 1e3)
    kernel_ms = reduce_max(float(np.mean(kms)), dist, cdev)
    alg_bytes = reduce_sum(int(stats.algorithmic_bytes), dist, cdev)
    walkers_total = reduce_sum(sum(len(q) for q, _, _ in rounds), dist, cdev)
    walkers_min = -reduce_max(-float(n), dist, cdev)
    walkers_max = reduce_max(float(n), dist, cdev)

    if args.dump and paths is not None and wpv == 1:
        q0, qid0, base0 = rounds[0]
        ids = (qid0 if qid0 is not None else
               torch.arange(base0, base0 + len(q0), dtype=torch.int64, device=dev))
        os.makedirs(args.dump, exist_ok=True)
        np.savez(os.path.join(args.dump, f"rank{rank}.npz"), qids=ids.cpu().numpy(),
                 lengths=lengths[:len(q0)].cpu().numpy(), paths=paths[:len(q0)].cpu().numpy(),
                 steps=walker_steps_rank)

    # ---- optional end-of-run gather of the path shards to rank 0
    gather = None
    if args.gather and dist is not None and paths is not None and wpv == 1:
        gather = gather_shards(torch, dist, cdev, rounds[0], lengths, paths, rank, world, nv)

    # ---- e2e through the C ABI with pinned host buffers (H2D + D2H timed):
    # dw_run_compact returns RunResult.paths flattened (offsets + ids), so only
    # ids that exist cross PCIe
    e2e = None
    if args.e2e_steps > 0 and n > 0 and not discard:
        # free the device paths of the timed region first (config 5: 43.5 GB)
        del paths
        torch.cuda.empty_cache()
        # one pinned host region per distinct query array (walker rounds share
        # theirs unless hash-sharded) and one output region reused by every
        # round: a streaming sink, each round's compact paths land in host
        # memory before the next round overwrites them
        nqmax = max(len(q) for q, _, _ in rounds)
        cap = nqmax * (L + 1)
        ho = C.c_void_p()
        hf = C.c_void_p()
        for buf, nbytes in ((ho, (nqmax + 1) * 8), (hf, cap * 4)):
            rc = lib.dw_host_alloc(nbytes, C.byref(buf))
            if rc:
                raise dw.DynwalkError(rc, lib.dw_last_error().decode())
        oa = np.ctypeslib.as_array(C.cast(ho, dw.u64p), (nqmax + 1,))
        hqs, rounds_h = [], []
        for k, (q, qid, base) in enumerate(rounds):
            if k == 0 or strong:
                hq = C.c_void_p()
                rc = lib.dw_host_alloc(len(q) * 4, C.byref(hq))
                if rc:
                    raise dw.DynwalkError(rc, lib.dw_last_error().decode())
                np.ctypeslib.as_array(C.cast(hq, dw.u32p), (len(q),))[:] = \
                    q.cpu().numpy().astype(np.uint32)
                hqs.append(hq)
            hqid = None if qid is None else np.ascontiguousarray(qid.cpu().numpy().astype(np.uint64))
            od = dw.RunOptions(mode=args.mode, walk_length=L, seed=WALK_SEED,
                               edge_cost_ratio=ratio, qid_base=base, qids=hqid,
                               erjs_handoff=args.handoff)
            rounds_h.append((hqs[-1], len(q), od, od.c(), hqid))
        st = dw.RunStatsC()
        out_ids = [0]

        def e2e_step():
            ids = 0
            for hq, nq, _, odc, _ in rounds_h:
                rc = lib.dw_run_compact(dg.h, C.byref(mdesc), C.cast(hq, dw.u32p), nq,
                                        C.byref(odc), C.cast(ho, dw.u64p), C.cast(hf, dw.u32p),
                                        cap, C.byref(st))
                if rc:
                    raise dw.DynwalkError(rc, lib.dw_last_error().decode())
                ids += int(oa[nq])
            out_ids[0] = ids

        e2e_step()  # warm
        if dist is not None:
            dist.barrier()
        ts = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            e2e_step()
            ts.append(time.perf_counter() - t0)
        t_e2e = reduce_max(float(np.mean(ts)), dist, cdev)
        nq_all = sum(nq for _, nq, _, _, _ in rounds_h)
        e2e = {"value": walker_steps / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": reduce_sum(
                   sum(nq * (4 + (8 if hqid is not None else 0))
                       for _, nq, _, _, hqid in rounds_h), dist, cdev),
               "d2h_bytes_per_step": reduce_sum((nq_all + len(rounds_h)) * 8 + out_ids[0] * 4,
                                                dist, cdev),
               "ms_per_step": t_e2e * 1e3,
               "api": "dw_run_compact (C ABI): pinned host queries in, offsets + path ids out"
                      + (f", {len(rounds_h)} walker rounds streamed through one reused host "
                         "region" if len(rounds_h) > 1 else "")}
        for buf in hqs + [ho, hf]:
            lib.dw_host_free(buf)

    # ---- §8(d) cheaper-mix denominator (configs 3 and 4)
    mix = None
    if cfg.get("cheaper_mix") and args.mode == "adaptive":
        mix = mix_bytes(lib, dw, dg, mdesc, nv, L, ratio, stream, torch, dev)

    # ---- CPU baseline (oracle port, host cores), rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and host_fits(info):
        cpu = cpu_baseline_port(dg, args, ratio, nv)

    if rank != 0:
        return
    pk = peaks()
    own_bytes = alg_bytes
    bytes_model = "SURVEY.md §8(d) minimal-sector model, counted per step on the device"
    if mix is not None:
        per_step = min(mix["reference_adaptive"], mix["all_ervs"])
        alg_bytes = int(per_step * walker_steps)
        bytes_model = ("SURVEY.md §8(d) cheaper-mix rule: min(reference adaptive mix, all-eRVS "
                       "mix) bytes per walker-step, each counted by the device on the same "
                       f"{mix['sample_walkers']}-walker sample, x this run's walker-steps")
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    sha = lib_sha16()
    traffic = ncu_traffic(args.scale, sha)
    if strong:
        par = (f"walker-parallel x{world}: the {walkers_total} global walker ids hash-"
               "partitioned over the ranks (Fibonacci hashing), graph replicated, no collective "
               "in the walk")
    else:
        par = (f"walker-parallel x{world} (one walker per vertex per GPU, graph replicated)"
               if world > 1 else "1 GPU, graph resident")
    out = {
        "metric": metric(args), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if (strong or world == 1) else "weak",
        "vs_baseline": None, "dtype": "f64 (bit-exact reference arithmetic), u32 ids",
        "data": "synthetic R-MAT (deterministic Philox generator, on-device)",
        "config": dict(workload(args), parallelism=par,
                       edge_cost_ratio=ratio, edge_cost_ratio_source=(
                           "override" if args.ratio > 0 else
                           "device-calibrated: K4 micro-passes refined by walking (dw_tune_ratio)"
                           if calib == "tune" else "device-calibrated: K4 micro-passes"),
                       edge_cost_ratio_micro=micro),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                     "peak_source": pk["source"],
                     "kernel": f"walk_kernel<{cfg['model']} model, adaptive, "
                               + ("32 B fat records>" if cfg["model"] == "node2vec" and not cfg["labels"]
                                  else "fat records>"),
                     "kernel_ms_per_launch": kernel_ms,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "algorithmic_bytes_per_walker_step": alg_bytes / max(walker_steps, 1),
                     "bytes_model": bytes_model,
                     "this_run_bytes_per_walker_step": own_bytes / max(walker_steps, 1),
                     "mix_bytes_per_walker_step": mix},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "build": {"lib_sha16": sha, "traffic_source": (
            "profiles/ncu_walk_kernel.json (ncu --set full of this build)" if traffic is not None
            else "null: no committed capture of this library build")},
        "clocks": clk.summary(),
        "gpu_launches": int(stats.kernel_launches) * args.steps,
        "walker_steps_per_step": walker_steps,
        "walkers_per_step": walkers_total,
        "stats": {k: int(getattr(stats, k)) for k in (
            "steps", "select_erjs", "select_ervs", "trials", "weight_reads", "rng_draws",
            "erjs_fallbacks", "dead_ends")},
        "setup_s": {"graph_build": build_s, "calibration": calib_s},
        "graph": dict(info, device_free_after_build_gb=graph_bytes[0] / 1e9,
                      device_total_gb=graph_bytes[1] / 1e9),
    }
    if world > 1:
        out["shards"] = {"min_walkers": int(walkers_min), "max_walkers": int(walkers_max)}
    if gather is not None:
        out["gather"] = gather
    print(json.dumps(out), flush=True)


def gather_shards(torch, dist, cdev, round0, lengths, paths, rank, world, nv,
                  keep=False) -> dict:
    """End-of-run gather of every rank's path shard (global ids, lengths, padded
    paths) to rank 0, which scatters them back into query order.  Shards have
    different sizes, so they are padded to the largest.  keep: rank 0 returns
    the gathered lengths and paths in query order (tests)."""
    def sync():
        if q0.device.type == "cuda":
            torch.cuda.synchronize()
    q0, qid0, base0 = round0
    n = len(q0)
    ids = (qid0 if qid0 is not None else
           torch.arange(base0, base0 + n, dtype=torch.int64, device=q0.device))
    sizes = [torch.zeros(1, dtype=torch.int64, device=cdev) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([n], dtype=torch.int64, device=cdev))
    m = int(max(int(x.item()) for x in sizes))
    stride = paths.shape[1]
    sync()
    t0 = time.perf_counter()
    pack = torch.full((m, stride + 3), -1, dtype=torch.int32, device=q0.device)
    pack[:n, 0] = (ids & 0xFFFFFFFF).to(torch.int32)
    pack[:n, 1] = (ids >> 32).to(torch.int32)
    pack[:n, 2] = lengths[:n]
    pack[:n, 3:] = paths[:n]
    pack = pack.to(cdev)
    bufs = [torch.empty_like(pack) for _ in range(world)] if rank == 0 else None
    dist.gather(pack, bufs, dst=0)
    out = {}
    if rank == 0:
        total = sum(int(x.item()) for x in sizes)
        full_len = torch.empty(total, dtype=torch.int32, device=q0.device)
        full_paths = torch.empty((total, stride), dtype=torch.int32, device=q0.device)
        for k, b in enumerate(bufs):
            nk = int(sizes[k].item())
            b = b[:nk].to(q0.device)
            gid = (b[:, 0].to(torch.int64) & 0xFFFFFFFF) | (b[:, 1].to(torch.int64) << 32)
            at = gid - base0 if qid0 is None else gid
            full_len[at] = b[:, 2]
            full_paths[at] = b[:, 3:]
        sync()
        out = {"ms": (time.perf_counter() - t0) * 1e3, "walkers": total,
               "bytes": total * (stride + 3) * 4,
               "backend": f"{dist.get_backend()} gather (padded shards), scattered into query "
                          "order on rank 0",
               "walk_steps_check": int((full_len.to(torch.int64) - 1).clamp(min=0).sum().item())}
        if keep:
            out["lengths"], out["paths"] = full_len, full_paths
    dist.barrier()
    return out


def mix_bytes(lib, dw, dg, mdesc, nv, L, ratio, stream, torch, dev, n=1 << 15) -> dict:
    """SURVEY §8(d) cheaper-mix rule (configs 3 and 4): algorithmic bytes per
    walker-step of the reference's adaptive mix (its decision rule and trial
    cap, no hand-off) and of the all-eRVS mix, each counted by the device on
    the same evenly spaced walker sample with the same per-event costs.  The
    denominator is the cheaper of the two, so bytes the reference wastes on
    loose bounds are not credited."""
    stride = max(1, nv // n)
    q = torch.arange(0, nv, stride, dtype=torch.int64, device=dev)[:n].to(torch.int32)
    lengths = torch.empty(max(len(q), 1), dtype=torch.int32, device=dev)
    out = {"sample_walkers": int(len(q))}
    for name, mode in (("reference_adaptive", "adaptive"), ("all_ervs", "force-ervs")):
        od = dw.RunOptions(mode=mode, walk_length=L, seed=WALK_SEED, edge_cost_ratio=ratio).c()
        t0 = time.perf_counter()
        rc = lib.dw_run_device(dg.h, 0, C.byref(mdesc), C.c_void_p(q.data_ptr()), len(q),
                               C.byref(od), None, C.c_void_p(lengths.data_ptr()),
                               C.c_void_p(stream.cuda_stream))
        if rc:
            raise dw.DynwalkError(rc, lib.dw_last_error().decode())
        st = dw.RunStatsC()
        rc = lib.dw_run_device_sync(dg.h, 0, C.byref(st))
        if rc:
            raise dw.DynwalkError(rc, lib.dw_last_error().decode())
        out[name] = st.algorithmic_bytes / max(st.steps - st.dead_ends, 1)
        out[name + "_s"] = time.perf_counter() - t0
    return out


def host_fits(info) -> bool:
    """The CPU leg copies the graph to the host twice (download + oracle CSR):
    run it when that fits in 1/2 of the available host memory."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        return False
    need = 2 * (info["num_vertices"] * 8 + info["num_edges"] * 10)
    return need < avail / 2


def cpu_baseline_port(dg, args, ratio, nv) -> dict:
    """The oracle (C restatement of the reference path, pthreads over all host
    cores) on a bounded walker sample of the same graph and ratio."""
    import oracle
    a = dg.download()
    og = oracle.Graph.from_csr(a["row"], a["col"], a["prop"], a["label"])
    del a
    cores = os.cpu_count() or 1
    m = oracle.Model(args.cfg["model"], **model_kw(args.cfg))
    n = 1 << 14
    rate = None
    while True:
        stride = max(1, nv // n)
        q = np.arange(0, nv, stride, dtype=np.uint32)[:n]
        t0 = time.perf_counter()
        r = oracle.run(og, m, q, mode=args.mode, walk_length=args.walk_length, seed=WALK_SEED,
                       ratio=ratio, rng="philox", threads=cores, keep_paths=False,
                       erjs_handoff=args.handoff)
        dt = time.perf_counter() - t0
        ws = r.stats["steps"] - r.stats["dead_ends"]
        rate = ws / dt
        if dt >= args.cpu_seconds * 0.5 or n >= nv:
            break
        n = min(nv, int(n * max(2.0, args.cpu_seconds / max(dt, 1e-3))))
    return {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{len(q)} walkers (every {stride}th vertex), {ws} walker-steps, "
                      f"{dt:.1f} s, same graph/ratio/seed as the GPU run"}


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    import oracle
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    # identical graph to the GPU arm, built on the CPU (oracle generator)
    cfg = args.cfg
    og = oracle.Graph.rmat_par(args.scale, 16, TOPO_SEED, 1.0, 5.0, WEIGHT_SEED, cores)
    if cfg["weights"] == "pareto":
        og.synth_philox("pareto", alpha=1.0, seed=WEIGHT_SEED)
    if cfg["labels"]:
        og.synth_philox("labels", cfg["labels"][0], cfg["labels"][1], seed=LABEL_SEED)
    a = og.arrays()
    del og
    kind = "reference" if oracle.ref_available() else "port"
    m = oracle.Model(cfg["model"], **model_kw(cfg))
    nv = len(a["row"]) - 1
    if kind == "reference":
        g = oracle.RefGraph.from_csr(a["row"], a["col"], a["prop"], a["label"])
        del a
        # the reference's own cost-model profile (cost_model.cpp:37-126), CLI seed
        ratio = oracle.ref_profile_ratio(g, m, oracle.derive_seed(WALK_SEED, PROFILE_SEED))

        def walk(q):
            r = oracle.ref_run(g, m, q, mode=args.mode, walk_length=args.walk_length,
                               seed=WALK_SEED, ratio=ratio, rng="mt19937", workers=cores,
                               keep_paths=False)
            return r.stats["steps"] - r.stats["dead_ends"], r.wall_ms / 1e3
    else:
        g = oracle.Graph.from_csr(a["row"], a["col"], a["prop"], a["label"])
        ratio = args.ratio if args.ratio > 0 else 1.2

        def walk(q):
            r = oracle.run(g, m, q, mode=args.mode, walk_length=args.walk_length,
                           seed=WALK_SEED, ratio=ratio, rng="mt19937", threads=cores,
                           keep_paths=False)
            return r.stats["steps"] - r.stats["dead_ends"], r.wall_ms / 1e3
    setup_s = time.perf_counter() - t0
    # size the per-step sample to ~4 s of walking
    n = 1 << 13
    while True:
        stride = max(1, nv // n)
        q = np.arange(0, nv, stride, dtype=np.uint32)[:n]
        ws, dt = walk(q)
        if dt > 0.5 or n >= nv:
            break
        n *= 4
    n = int(min(nv, max(n, n * 4.0 / max(dt, 1e-3))))
    stride = max(1, nv // n)
    q = np.arange(0, nv, stride, dtype=np.uint32)[:n]
    for _ in range(args.warmup):
        walk(q)
    tot_ws, tot_t = 0, 0.0
    for _ in range(args.steps):
        ws, dt = walk(q)
        tot_ws += ws
        tot_t += dt
    value = tot_ws / tot_t
    sample = (f"{len(q)} walkers per step (every {stride}th vertex), {tot_ws // args.steps} "
              f"walker-steps per step; time = RunStats.wall_ms")
    out = {"metric": metric(args), "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic R-MAT (same graph as the GPU arm, CPU-built)",
           "impl": "reference",
           "config": dict(workload(args), edge_cost_ratio=ratio,
                          sampling="the reference's own run_queries (its decision rule and cap)",
                          edge_cost_ratio_source="reference profile_edge_cost_ratio"
                          if kind == "reference" else "fixed"),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "setup_s": setup_s}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    world, _, _ = dist_env()
    if world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
