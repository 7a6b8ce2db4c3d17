"""GPU parity suite: the CUDA path (through the C ABI) against the oracle and the
reference goldens.  Bit-exact paths, lengths and RunStats counters wherever
both sides consume the same Philox walker stream; chi-square p > 0.01 of
transition frequencies against the exact probabilities otherwise."""
import json
import os

import numpy as np
import pytest

from tests.golden.make_golden import CASES, GRAPHS, MODES, build_oracle_graph, case_id, digest, \
    stats_core

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def to_device(dw, og):
    a = og.arrays()
    return dw.DeviceGraph.from_csr(a["row"], a["col"], a["prop"], a["label"])


def run_both(dw, orc, og, dg, mk, queries, mode, L, ratio, seed=7, cap=64, qid_base=0):
    r_dev = dw.run_queries(dg, dw.Model(**mk), queries,
                           dw.RunOptions(mode=mode, walk_length=L, seed=seed, edge_cost_ratio=ratio,
                                         erjs_cap_per_degree=cap, qid_base=qid_base))
    r_orc = orc.run(og, orc.Model(**mk), queries, mode=mode, walk_length=L, seed=seed,
                    ratio=ratio, cap_per_degree=cap, rng="philox", threads=4, qid_base=qid_base)
    return r_dev, r_orc


def assert_same(r_dev, r_orc, tag=""):
    assert stats_core(r_dev.stats) == stats_core(r_orc.stats), tag
    assert np.array_equal(r_dev.lengths, r_orc.lengths), tag
    assert np.array_equal(r_dev.paths, r_orc.paths), tag


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0] + ":" + c[1]["kind"])
def test_reference_goldens_on_gpu(dw, orc, case):
    """GPU == the reference's own sampler templates (tests/golden/ref_walks.json)."""
    gold = {c["id"]: c for c in json.load(open(os.path.join(GOLDEN, "ref_walks.json")))["cases"]}
    gname, mk, L, ratio = case
    og = build_oracle_graph(GRAPHS[gname])
    dg = to_device(dw, og)
    q = np.arange(og.nv, dtype=np.uint32)
    for mode in MODES:
        r = dw.run_queries(dg, dw.Model(**mk), q,
                           dw.RunOptions(mode=mode, walk_length=L, seed=7, edge_cost_ratio=ratio))
        c = gold[case_id(gname, mk, mode, L)]
        assert stats_core(r.stats) == c["stats"], mode
        assert digest(r.paths, r.lengths) == c["digest"], mode


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("mk", [dict(kind="node2vec", a=2.0, b=0.5),
                                dict(kind="node2vec", a=0.5, b=2.0),
                                # not powers of two: the device divides by a and b
                                # (Markstein from RN(1/a)), the oracle with '/'
                                dict(kind="node2vec", a=1.3, b=0.7),
                                dict(kind="node2vec", a=3.0, b=0.1),
                                dict(kind="pr2", gamma=0.2),
                                dict(kind="static", weighted=False)])
def test_rmat_bit_exact(dw, orc, mk, mode):
    """R-MAT s12 (hubs well above the warp-cooperative threshold)."""
    og = orc.Graph.rmat(12, 16, 5).synth_philox("uniform", 1.0, 5.0, seed=6)
    dg = to_device(dw, og)
    q = np.arange(og.nv, dtype=np.uint32)
    r_dev, r_orc = run_both(dw, orc, og, dg, mk, q, mode, 40, 1.2)
    assert_same(r_dev, r_orc, (mk, mode))


def test_metapath_labels_and_dead_ends(dw, orc):
    og = orc.Graph.rmat(11, 16, 8).synth_philox("uniform", 1.0, 5.0, seed=9)
    og.synth_philox("labels", 0, 3, seed=10)
    dg = to_device(dw, og)
    q = np.arange(og.nv, dtype=np.uint32)
    mk = dict(kind="metapath", schema=(0, 1, 2, 3) * 20)
    for mode in MODES:
        r_dev, r_orc = run_both(dw, orc, og, dg, mk, q, mode, 80, 1.2)
        assert_same(r_dev, r_orc, mode)
        assert r_dev.stats["dead_ends"] > 0


def test_device_rmat_builder_matches_oracle(dw, orc):
    for scale, seed in ((10, 1), (13, 77)):
        dg = dw.DeviceGraph.rmat(scale, 16, seed=seed, weights="uniform", weight_seed=seed + 1,
                                 labels=(0, 3), label_seed=seed + 2)
        og = orc.Graph.rmat(scale, 16, seed).synth_philox("uniform", 1.0, 5.0, seed=seed + 1)
        og.synth_philox("labels", 0, 3, seed=seed + 2)
        a, b = dg.download(), og.arrays()
        for k in ("row", "col", "prop", "nmax", "nsum", "label"):
            assert np.array_equal(a[k], b[k]), (scale, k)
    dg = dw.DeviceGraph.rmat(11, 16, seed=3, weights="pareto", alpha=1.0, weight_seed=4)
    og = orc.Graph.rmat(11, 16, 3).synth_philox("pareto", alpha=1.0, seed=4)
    a, b = dg.download(), og.arrays()
    for k in ("row", "col", "prop", "nmax", "nsum"):
        assert np.array_equal(a[k], b[k]), k


def test_upload_roundtrip_and_aggregates(dw, orc):
    og = build_oracle_graph(GRAPHS["ba300_labels"])
    a = og.arrays()
    # aggregates recomputed on the device (left-to-right) equal the host's
    dg = dw.DeviceGraph.from_csr(a["row"], a["col"], a["prop"], a["label"])
    b = dg.download()
    for k in ("row", "col", "prop", "nmax", "nsum", "label"):
        assert np.array_equal(a[k], b[k]), k
    info = dg.info()
    assert info["num_vertices"] == og.nv and info["num_edges"] == og.ne and info["has_labels"]
    assert info["max_degree"] == int(np.diff(a["row"]).max())


def test_edge_cases(dw, orc):
    """Isolated starts, out-of-range starts, walk_length 0, cap fallback, duplicates."""
    og = orc.Graph.build([0, 0, 0, 1, 1, 2], [1, 1, 2, 0, 2, 0], [1, 2, 3, 1, 4, 2], nv_hint=6)
    dg = to_device(dw, og)
    q = np.array([0, 3, 99, 1, 2, 5, 0, 0], np.uint32)
    for mode in MODES:
        for L in (0, 1, 7):
            r_dev, r_orc = run_both(dw, orc, og, dg, dict(kind="node2vec", a=0.5, b=2.0), q,
                                    mode, L, 1.0)
            assert_same(r_dev, r_orc, (mode, L))
            assert r_dev.lengths[2] == 0 and r_dev.stats["query_errors"] == 1
    # tiny cap: every eRJS step falls back to the reservoir
    r_dev, r_orc = run_both(dw, orc, og, dg, dict(kind="static"), q, "force-erjs", 9, 1.0, cap=0)
    assert_same(r_dev, r_orc, "cap0")
    assert r_dev.stats["erjs_fallbacks"] == r_dev.stats["steps"]
    # empty query list
    r = dw.run_queries(dg, dw.Model(), np.zeros(0, np.uint32), dw.RunOptions(walk_length=5))
    assert r.stats["queries"] == 0


def test_sharding_is_output_invariant(dw, orc):
    """Device-count analogue of worker-count invariance (test_runtime.cpp:118-138):
    walkers split by qid_base give the paths of one unsplit run."""
    og = orc.Graph.rmat(11, 16, 21).synth_philox("uniform", 1.0, 5.0, seed=22)
    dg = to_device(dw, og)
    q = np.arange(og.nv, dtype=np.uint32)
    opts = dict(mode="adaptive", walk_length=30, seed=3, edge_cost_ratio=1.2)
    full = dw.run_queries(dg, dw.Model(a=0.5, b=2.0), q, dw.RunOptions(**opts))
    parts = [dw.run_queries(dg, dw.Model(a=0.5, b=2.0), q[lo:hi],
                            dw.RunOptions(qid_base=lo, **opts))
             for lo, hi in ((0, 700), (700, 1500), (1500, og.nv))]
    assert np.array_equal(full.paths, np.concatenate([p.paths for p in parts]))
    assert full.stats["steps"] == sum(p.stats["steps"] for p in parts)


def test_large_batched_run_matches_oracle(dw, orc):
    """> 1M walkers: dw_run splits into overlapped batches; output unchanged."""
    og = orc.Graph.rmat(14, 16, 31).synth_philox("uniform", 1.0, 5.0, seed=32)
    dg = to_device(dw, og)
    rs = np.random.default_rng(0)
    q = rs.integers(0, og.nv, size=2_500_000, dtype=np.uint32)
    r_dev, r_orc = run_both(dw, orc, og, dg, dict(kind="node2vec", a=0.5, b=2.0), q, "adaptive",
                            10, 1.2)
    assert_same(r_dev, r_orc, "batched")
    assert r_dev.stats["kernel_launches"] > 1


def test_run_device_entry_point(dw, orc):
    import ctypes as C
    import torch
    og = orc.Graph.rmat(11, 16, 41).synth_philox("uniform", 1.0, 5.0, seed=42)
    dg = to_device(dw, og)
    q = np.arange(og.nv, dtype=np.uint32)
    L = 20
    dq = torch.from_numpy(q.view(np.int32)).cuda()
    dp = torch.empty((len(q), L + 1), dtype=torch.int32, device="cuda")
    dl = torch.empty(len(q), dtype=torch.int32, device="cuda")
    lib = dw.load_library()
    m = dw.Model(a=0.5, b=2.0).c()
    o = dw.RunOptions(walk_length=L, seed=4, edge_cost_ratio=1.2).c()
    torch.cuda.synchronize()
    assert lib.dw_run_device(dg.h, 0, C.byref(m), C.c_void_p(dq.data_ptr()), len(q), C.byref(o),
                             C.c_void_p(dp.data_ptr()), C.c_void_p(dl.data_ptr()), None) == 0
    st = dw.RunStatsC()
    assert lib.dw_run_device_sync(dg.h, 0, C.byref(st)) == 0
    r_orc = orc.run(og, orc.Model(a=0.5, b=2.0), q, walk_length=L, seed=4, ratio=1.2,
                    rng="philox", threads=4)
    assert np.array_equal(dp.cpu().numpy().view(np.uint32), r_orc.paths)
    assert np.array_equal(dl.cpu().numpy().view(np.uint32), r_orc.lengths)
    assert st.steps == r_orc.stats["steps"] and st.kernel_ms > 0


def _run_device(dw, dg, q, model, opts, paths=True, qids=None):
    """dw_run_device on cuda:0 (device queries, padded rows and lengths)."""
    import ctypes as C
    import torch
    L = opts.walk_length
    dq = torch.from_numpy(q.view(np.int32)).cuda()
    dp = torch.empty((len(q), L + 1), dtype=torch.int32, device="cuda") if paths else None
    dl = torch.empty(len(q), dtype=torch.int32, device="cuda")
    if qids is not None:
        dqid = torch.from_numpy(qids.view(np.int64)).cuda()
        opts.qids = dqid.data_ptr()
    lib = dw.load_library()
    m = model.c()
    o = opts.c()
    torch.cuda.synchronize()
    assert lib.dw_run_device(dg.h, 0, C.byref(m), C.c_void_p(dq.data_ptr()), len(q), C.byref(o),
                             C.c_void_p(dp.data_ptr() if paths else None),
                             C.c_void_p(dl.data_ptr()), None) == 0
    st = dw.RunStatsC()
    assert lib.dw_run_device_sync(dg.h, 0, C.byref(st)) == 0
    opts.qids = None
    return (dp.cpu().numpy().view(np.uint32) if paths else None,
            dl.cpu().numpy().view(np.uint32), st.as_dict())


@pytest.mark.parametrize("mode", ["adaptive", "force-erjs"])
def test_run_device_listed_walkers(dw, orc, mode, tmp_path):
    """dw_run_device walks only the walkers that can move when every length
    is known before the walk (trace "L nq ok"): padded rows, lengths and
    counters equal the every-walker launch (DW_DIRECT=0) and the oracle,
    with invalid and isolated starts, explicit walker ids, qid_base and
    discarded paths; on a graph with sinks, forced listing (DW_DIRECT=2) is
    detected and re-run on every walker ("L nq retry")."""
    og = orc.Graph.rmat(13, 16, 21).synth_philox("uniform", 1.0, 5.0, seed=22)
    dg = to_device(dw, og)
    rng = np.random.default_rng(12)
    q = rng.integers(0, og.nv + 40, 1_200_000).astype(np.uint32)  # listing needs >= 2^20
    model = dw.Model(kind="node2vec", a=0.5, b=2.0)
    trace = str(tmp_path / "trace.txt")
    qids = rng.permutation(4 * len(q))[:len(q)].astype(np.uint64)
    for kw, qd in ((dict(), None), (dict(qid_base=77_777), None), (dict(), qids)):
        opts = dw.RunOptions(mode=mode, walk_length=30, seed=6, edge_cost_ratio=1.3, **kw)
        if os.path.exists(trace):
            os.remove(trace)
        a = _with_env({"DW_ENGINE_TRACE": trace}, lambda: _run_device(dw, dg, q, model, opts,
                                                                      qids=qd))
        assert open(trace).read().split() == ["L", str(len(q)), "ok"]
        b = _with_env({"DW_DIRECT": "0"}, lambda: _run_device(dw, dg, q, model, opts, qids=qd))
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), kw
        assert stats_core(a[2]) == stats_core(b[2]), kw
        assert a[2]["queries"] == b[2]["queries"] and a[2]["query_errors"] == b[2]["query_errors"]
    r_orc = orc.run(og, orc.Model(kind="node2vec", a=0.5, b=2.0), q[:30_000], mode=mode,
                    walk_length=30, seed=6, ratio=1.3, rng="philox", threads=4)
    opts = dw.RunOptions(mode=mode, walk_length=30, seed=6, edge_cost_ratio=1.3)
    p, l, st1 = _run_device(dw, dg, q, model, opts)  # listed; walker ids = indices
    assert np.array_equal(p[:30_000], r_orc.paths) and np.array_equal(l[:30_000], r_orc.lengths)
    _, l2, st2 = _run_device(dw, dg, q, model, opts, paths=False)
    assert np.array_equal(l2, l) and st2["steps"] == st1["steps"]
    # a directed graph with sinks: listing forced, detected, re-run
    src = rng.integers(0, 3000, 20000).astype(np.uint32)
    dst = rng.integers(0, 3000, 20000).astype(np.uint32)
    keep = src % 5 != 0
    g2 = orc.Graph.build(src[keep], dst[keep], rng.uniform(1, 5, keep.sum()).astype(np.float32),
                         mirror=False, nv_hint=3000)
    dg2 = to_device(dw, g2)
    q2 = np.arange(g2.nv, dtype=np.uint32).repeat(400)
    opts = dw.RunOptions(mode=mode, walk_length=25, seed=2, edge_cost_ratio=1.3)
    if os.path.exists(trace):
        os.remove(trace)
    a = _with_env({"DW_DIRECT": "2", "DW_ENGINE_TRACE": trace},
                  lambda: _run_device(dw, dg2, q2, model, opts))
    assert open(trace).read().split() == ["L", str(len(q2)), "retry"]
    b = _with_env({"DW_DIRECT": "0"}, lambda: _run_device(dw, dg2, q2, model, opts))
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert stats_core(a[2]) == stats_core(b[2])


def test_chi_square_transition_frequencies(dw, orc):
    """Per-(prev,cur) transition counts vs oracle_enumerate (samplers.hpp:272-288), p > 0.01."""
    from scipy.stats import chisquare
    # second-order fixture (test_util.hpp:22-36) reached from prev=0 -> cur=1
    og = orc.Graph.build([0, 0, 1, 1, 1, 1], [1, 2, 0, 2, 3, 4], [1, 1, 1, 1, 3, 1], nv_hint=5)
    dg = to_device(dw, og)
    n = 400_000
    for mk in (dict(kind="node2vec", a=2.0, b=0.5), dict(kind="pr2", gamma=0.2)):
        probs = orc.transition_probs(og, orc.Model(**mk), 1, 0, 1)
        for mode in MODES:
            r = dw.run_queries(dg, dw.Model(**mk), np.zeros(n, np.uint32),
                               dw.RunOptions(mode=mode, walk_length=2, seed=11,
                                             edge_cost_ratio=0.5))
            sel = r.paths[:, 1] == 1  # walks that went 0 -> 1
            nxt = r.paths[sel, 2]
            counts = np.array([(nxt == t).sum() for t in (0, 2, 3, 4)])
            assert chisquare(counts, probs * counts.sum()).pvalue > 0.01, (mk, mode)


def test_calibration(dw, orc):
    dg = dw.DeviceGraph.rmat(14, 16, seed=5)
    for mk in (dict(kind="node2vec", a=0.5, b=2.0), dict(kind="static")):
        r = dw.profile_edge_cost_ratio(dg, dw.Model(**mk), seed=1)
        assert np.isfinite(r) and r > 0


def test_calibration_positive_and_stable(dw, orc):
    """test_runtime.cpp:87-105 restated: the reference's bench fixture (BA
    n=3000 deg=6 mirrored, uniform weights), node2vec (2, 0.5), ProfileConfig
    with 5 repetitions and seed 1: a positive, finite ratio, the same within
    4x on a second call, and node_fraction = 0 rejected."""
    og = orc.Graph.ba(3000, 6, 77).synth("uniform", seed=78)
    a = og.arrays()
    dg = dw.DeviceGraph.from_csr(a["row"], a["col"], a["prop"])
    model = dw.Model(kind="node2vec", a=2.0, b=0.5)
    cfg = dw.ProfileConfig(repetitions=5, seed=1)
    p1 = dw.profile_edge_cost_ratio(dg, model, cfg=cfg)
    assert p1 > 0 and np.isfinite(p1)
    p2 = dw.profile_edge_cost_ratio(dg, model, cfg=cfg)
    assert abs(np.log(p1 / p2)) < np.log(4.0)
    with pytest.raises(dw.DynwalkError, match="node_fraction must be in"):
        dw.profile_edge_cost_ratio(dg, model, cfg=dw.ProfileConfig(node_fraction=0.0))
    with pytest.raises(dw.DynwalkError, match="repetitions must be >= 1"):
        dw.profile_edge_cost_ratio(dg, model, cfg=dw.ProfileConfig(repetitions=0))
    with pytest.raises(dw.DynwalkError, match="repetitions must be >= 1"):
        dw.profile_edge_cost_ratio(dg, model, cfg=dw.ProfileConfig(neighbors_per_node=0))
    # every ProfileConfig field reaches the device passes
    for c in (dw.ProfileConfig(node_fraction=1.0, seed=3), dw.ProfileConfig(min_nodes=1000),
              dw.ProfileConfig(neighbors_per_node=1), dw.ProfileConfig(repetitions=1)):
        r = dw.profile_edge_cost_ratio(dg, model, cfg=c)
        assert r > 0 and np.isfinite(r)


def test_tuned_ratio_is_near_the_micro_pass_ratio(dw):
    """dw_tune_ratio walks the kernel at r0 x {1/2 .. 2} around the
    micro-pass ratio r0 and returns a threshold inside that range."""
    dg = dw.DeviceGraph.rmat(14, 16, seed=5, weights="uniform", weight_seed=6)
    model = dw.Model(kind="node2vec", a=0.5, b=2.0)
    cfg = dw.ProfileConfig(seed=3)
    r0 = dw.profile_edge_cost_ratio(dg, model, cfg=cfg)
    rt = dw.tune_edge_cost_ratio(dg, model, cfg=cfg, walk_length=20)
    assert np.isfinite(rt) and r0 * 0.5 * (1 - 1e-9) <= rt <= r0 * 2.0 * (1 + 1e-9)
    with pytest.raises(dw.DynwalkError, match="node_fraction"):
        dw.tune_edge_cost_ratio(dg, model, cfg=dw.ProfileConfig(node_fraction=2.0))


def test_calibration_degree_one_ring(dw):
    """test_runtime.cpp:107-118 restated: a directed 64-node ring (every
    degree 1), StaticWalk weighted, seed 2: positive and finite."""
    n = 64
    row = np.arange(n + 1, dtype=np.uint64)
    col = ((np.arange(n) + 1) % n).astype(np.uint32)
    dg = dw.DeviceGraph.from_csr(row, col, np.ones(n, np.float32))
    r = dw.profile_edge_cost_ratio(dg, dw.Model(kind="static"), cfg=dw.ProfileConfig(seed=2))
    assert r > 0 and np.isfinite(r)


def test_errors(dw):
    with pytest.raises(dw.DynwalkError, match="not supported"):
        dg = dw.DeviceGraph.rmat(8, 16, seed=1)
        dw.run_queries(dg, dw.Model(), [0], dw.RunOptions(mode="force-its"))
    with pytest.raises(dw.DynwalkError, match="strictly positive"):
        dw.DeviceGraph.from_csr([0, 1, 1], [1], [0.0])
    with pytest.raises(dw.DynwalkError, match="not sorted"):
        dw.DeviceGraph.from_csr([0, 2, 2, 2], [2, 1], [1.0, 1.0])


def _with_env(env: dict, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("env", [{"DW_FAT": "2", "DW_FAT32_BAND": "10"},
                                 {"DW_FAT": "2", "DW_SCREEN": "0"}],
                         ids=["band-wide", "no-screen"])
def test_compact_records_exact_fallback(dw, orc, env):
    """The compact records' f32 row sum decides only outside a relative band;
    inside it (here: every decision, band 10) or without the one-multiply
    screen, the exact node record decides, and the return-edge range the
    record carried survives that refetch.  Paths and counters stay equal to
    the oracle (this path was only checked by a manual rebuild)."""
    og = orc.Graph.rmat(12, 16, 11).synth_philox("uniform", 1.0, 5.0, seed=12)
    dg = _with_env({"DW_FAT": env["DW_FAT"]}, lambda: to_device(dw, og))
    q = np.arange(og.nv, dtype=np.uint32)
    for mk in (dict(kind="node2vec", a=0.5, b=2.0), dict(kind="node2vec", a=2.0, b=0.5)):
        for mode in ("adaptive", "force-erjs"):
            r_dev, r_orc = _with_env(env, lambda: run_both(dw, orc, og, dg, mk, q, mode, 60, 1.6))
            assert_same(r_dev, r_orc, (env, mk, mode))


@pytest.mark.parametrize("scale", [3.0e38, 1.0e-38])
@pytest.mark.parametrize("layout", ["fat", "fat32", "slim"])
def test_extreme_prop_magnitudes(dw, orc, scale, layout):
    """Edge properties near FLT_MAX (row sums overflow f32: the compact
    record stores NaN and the exact node record decides) and near FLT_MIN
    (subnormal-range sums, exact in f32) walk bit-exactly on every layout."""
    base = orc.Graph.rmat(11, 16, 21).synth_philox("uniform", 1.0, 5.0, seed=22)
    a = base.arrays()
    prop = (a["prop"].astype(np.float64) / 5.0 * scale).astype(np.float32)
    assert np.all(prop > 0) and np.all(np.isfinite(prop))
    og = orc.Graph.from_csr(a["row"], a["col"], prop)
    env = {"DW_FAT": {"fat": "1", "fat32": "2"}.get(layout, "0")}
    dg = _with_env(env, lambda: dw.DeviceGraph.from_csr(a["row"], a["col"], prop))
    q = np.arange(og.nv, dtype=np.uint32)
    for mk in (dict(kind="node2vec", a=0.5, b=2.0), dict(kind="node2vec", a=2.0, b=0.5)):
        for mode in ("adaptive", "force-erjs", "force-ervs"):
            r_dev, r_orc = run_both(dw, orc, og, dg, mk, q, mode, 40, 1.6)
            assert_same(r_dev, r_orc, (scale, layout, mk, mode))


@pytest.mark.parametrize("layout", ["fat", "fat32", "slim", "slim-notwin"])
@pytest.mark.parametrize("shortcut", ["1", "0"])
@pytest.mark.parametrize("mk", [dict(kind="node2vec", a=0.5, b=2.0),
                                dict(kind="node2vec", a=2.0, b=0.5),
                                dict(kind="node2vec", a=0.3, b=1.7),
                                dict(kind="pr2", gamma=0.2)])
def test_layouts_and_free_rejections(dw, orc, mk, shortcut, layout):
    """Fat records (dw_common.cuh FatRec) and free rejections
    (nonreturn_max) must not change a single path or counter: the same run on
    the slim layout, with and without the shortcut, equals the oracle."""
    og = orc.Graph.rmat(12, 16, 11).synth_philox("uniform", 1.0, 5.0, seed=12)
    env = {"DW_FAT": {"fat": "1", "fat32": "2"}.get(layout, "0")}
    if layout == "slim-notwin":
        env["DW_TWIN"] = "0"
    dg = _with_env(env, lambda: to_device(dw, og))
    q = np.arange(og.nv, dtype=np.uint32)
    for mode in ("adaptive", "force-erjs"):
        r_dev, r_orc = _with_env({"DW_SHORTCUT": shortcut},
                                 lambda: run_both(dw, orc, og, dg, mk, q, mode, 60, 1.2))
        assert_same(r_dev, r_orc, (mk, mode, layout, shortcut))


def test_directed_multigraph_without_twins(dw, orc):
    """A directed graph with duplicate edges and self-loops: return-edge ranges
    are empty or multi-edge, so free rejections and the fat twin range are
    exercised on their edge cases."""
    rng = np.random.default_rng(5)
    n = 3000
    src = rng.integers(0, n, 40000).astype(np.uint32)
    dst = (src + rng.integers(-40, 40, 40000)).clip(0, n - 1).astype(np.uint32)
    src = np.concatenate([src, src[:3000], np.arange(0, n, 7, dtype=np.uint32)])
    dst = np.concatenate([dst, dst[:3000], np.arange(0, n, 7, dtype=np.uint32)])
    prop = rng.uniform(1.0, 5.0, len(src)).astype(np.float32)
    og = orc.Graph.build(src, dst, prop, mirror=False, nv_hint=n)
    dg = to_device(dw, og)
    q = np.arange(og.nv, dtype=np.uint32)
    for mk in (dict(kind="node2vec", a=0.5, b=2.0), dict(kind="pr2", gamma=0.3)):
        for mode in MODES:
            r_dev, r_orc = run_both(dw, orc, og, dg, mk, q, mode, 50, 1.1)
            assert_same(r_dev, r_orc, (mk, mode))
    # the slim layout with its twin[] ranges on the same edge cases
    dg = _with_env({"DW_FAT": "0"}, lambda: to_device(dw, og))
    for mk in (dict(kind="node2vec", a=0.5, b=2.0), dict(kind="pr2", gamma=0.3)):
        for mode in ("adaptive", "force-erjs"):
            r_dev, r_orc = run_both(dw, orc, og, dg, mk, q, mode, 50, 1.1)
            assert_same(r_dev, r_orc, (mk, mode, "slim"))


def test_compact_output_matches_padded(dw, orc):
    """dw_run_compact (flattened RunResult.paths) carries exactly the padded
    run's paths, including empty paths for query errors, over several batches."""
    og = orc.Graph.rmat(13, 16, 21).synth_philox("uniform", 1.0, 5.0, seed=22)
    dg = to_device(dw, og)
    rng = np.random.default_rng(3)
    q = rng.integers(0, og.nv + 50, 2_300_000).astype(np.uint32)  # > 2 batches, some invalid
    opts = dw.RunOptions(mode="adaptive", walk_length=30, seed=5, edge_cost_ratio=1.3)
    model = dw.Model(a=0.5, b=2.0)
    r = dw.run_queries(dg, model, q, opts)
    offs, flat, st = dw.run_queries_compact(dg, model, q, opts)
    lens = np.diff(offs.astype(np.int64))
    assert np.array_equal(lens, r.lengths.astype(np.int64))
    mask = np.arange(r.paths.shape[1])[None, :] < r.lengths[:, None]
    assert np.array_equal(flat, r.paths[mask])
    for k in ("steps", "trials", "rng_draws", "dead_ends", "query_errors"):
        assert st[k] == r.stats[k], k


def _compact_pair(dw, dg, model, q, opts, env, trace):
    """dw_run_compact under `env` and under the batched engine (DW_DIRECT=0);
    returns both results and the run engine trace lines of the first."""
    if os.path.exists(trace):
        os.remove(trace)
    a = _with_env(dict(env, DW_ENGINE_TRACE=trace),
                  lambda: dw.run_queries_compact(dg, model, q, opts))
    lines = open(trace).read().split() if os.path.exists(trace) else []
    b = _with_env({"DW_DIRECT": "0"}, lambda: dw.run_queries_compact(dg, model, q, opts))
    return a, b, lines


def _assert_compact_equal(a, b, tag):
    assert np.array_equal(a[0], b[0]), tag
    assert np.array_equal(a[1], b[1]), tag
    for k in ("steps", "select_erjs", "select_ervs", "trials", "weight_reads", "rng_draws",
              "dead_ends", "query_errors", "erjs_fallbacks", "queries"):
        assert a[2][k] == b[2][k], (tag, k)


@pytest.mark.parametrize("layout", ["default", "slim", "fat64"])
@pytest.mark.parametrize("mk", [dict(kind="node2vec", a=0.5, b=2.0),
                                dict(kind="node2vec", a=2.0, b=0.5, weighted=False)],
                         ids=["weighted", "unweighted"])
def test_direct_compact_output(dw, orc, mk, layout, tmp_path):
    """dw_run_compact's direct engine (one launch writing every path at its
    predicted flat offset, chunks copied while the walk runs) gives the
    batched engine's offsets, ids and counters: mirrored graph, invalid starts
    (empty paths), isolated starts (length 1), several chunks, every record
    layout, adaptive and force-erjs; other models keep the batched engine."""
    og = orc.Graph.rmat(13, 16, 21).synth_philox("uniform", 1.0, 5.0, seed=22)
    env = {"default": {}, "slim": {"DW_FAT": "0"}, "fat64": {"DW_FAT": "1"}}[layout]
    dg = _with_env(env, lambda: to_device(dw, og))
    rng = np.random.default_rng(4)
    q = rng.integers(0, og.nv + 50, 1_500_000).astype(np.uint32)
    model = dw.Model(**mk)
    trace = str(tmp_path / "trace.txt")
    for mode, L in (("adaptive", 30), ("adaptive", 1), ("adaptive", 0), ("force-erjs", 12)):
        opts = dw.RunOptions(mode=mode, walk_length=L, seed=5, edge_cost_ratio=1.3)
        a, b, lines = _compact_pair(dw, dg, model, q, opts, {}, trace)
        assert lines[:3] == ["X", str(len(q)), "ok"], (mk, mode, L, lines[:6])
        _assert_compact_equal(a, b, (mk, mode, L))
    # the padded run agrees too (lengths = offset differences)
    opts = dw.RunOptions(mode="adaptive", walk_length=20, seed=9, edge_cost_ratio=1.3)
    r = dw.run_queries(dg, model, q[:200_000], opts)
    offs, flat, _ = dw.run_queries_compact(dg, model, q[:200_000], opts)
    assert np.array_equal(np.diff(offs.astype(np.int64)), r.lengths.astype(np.int64))
    mask = np.arange(r.paths.shape[1])[None, :] < r.lengths[:, None]
    assert np.array_equal(flat, r.paths[mask])
    # PR2 and the reservoir-only modes stay on the batched engine
    for m2, mode in ((dw.Model(kind="pr2", gamma=0.15), "adaptive"), (model, "force-ervs")):
        opts = dw.RunOptions(mode=mode, walk_length=10, seed=5, edge_cost_ratio=1.3)
        a, b, lines = _compact_pair(dw, dg, m2, q[:300_000], opts, {}, trace)
        assert "X" not in lines, (mode, lines[:6])
        _assert_compact_equal(a, b, ("batched", mode))


def test_direct_compact_global_walker_ids(dw, orc, tmp_path):
    """Direct compact runs keyed by explicit global walker ids (dw_run_opts.qids,
    as the hash-sharded multi-GPU bench passes them) and by qid_base: equal to
    the batched engine and to the oracle with the same ids."""
    og = orc.Graph.rmat(12, 16, 31).synth_philox("uniform", 1.0, 5.0, seed=32)
    dg = to_device(dw, og)
    rng = np.random.default_rng(9)
    q = rng.integers(0, og.nv, 300_000).astype(np.uint32)
    qids = rng.permutation(10 * len(q))[:len(q)].astype(np.uint64)
    model = dw.Model(kind="node2vec", a=0.5, b=2.0)
    trace = str(tmp_path / "trace.txt")
    for kw in (dict(qids=qids), dict(qid_base=123_456_789)):
        opts = dw.RunOptions(mode="adaptive", walk_length=40, seed=11, edge_cost_ratio=1.1, **kw)
        a, b, lines = _compact_pair(dw, dg, model, q, opts, {}, trace)
        assert lines[:3] == ["X", str(len(q)), "ok"], lines[:6]
        _assert_compact_equal(a, b, kw.keys())
        r_orc = orc.run(og, orc.Model(kind="node2vec", a=0.5, b=2.0), q[:20_000], mode="adaptive",
                        walk_length=40, seed=11, ratio=1.1, rng="philox", threads=4,
                        qids=qids[:20_000] if "qids" in kw else None,
                        qid_base=kw.get("qid_base", 0))
        o = a[0].astype(np.int64)
        mask = np.arange(r_orc.paths.shape[1])[None, :] < r_orc.lengths[:, None]
        assert np.array_equal(a[1][:o[20_000]], r_orc.paths[mask]), kw.keys()


def test_direct_compact_falls_back_on_sinks(dw, orc, tmp_path):
    """A directed graph with sinks: walks stop early, so the direct engine is
    not used (no X trace line); forced (DW_DIRECT=2) it detects the shorter
    walks, and the batched re-run gives the same output."""
    rng = np.random.default_rng(6)
    n = 4000
    src = rng.integers(0, n, 30000).astype(np.uint32)
    dst = rng.integers(0, n, 30000).astype(np.uint32)
    keep = src % 5 != 0  # vertices 0, 5, 10 ... have in-edges only: sinks
    src, dst = src[keep], dst[keep]
    prop = rng.uniform(1.0, 5.0, len(src)).astype(np.float32)
    og = orc.Graph.build(src, dst, prop, mirror=False, nv_hint=n)
    dg = to_device(dw, og)
    q = np.arange(og.nv, dtype=np.uint32).repeat(40)
    model = dw.Model(kind="node2vec", a=0.5, b=2.0)
    opts = dw.RunOptions(mode="adaptive", walk_length=40, seed=3, edge_cost_ratio=1.3)
    trace = str(tmp_path / "trace.txt")
    a, b, lines = _compact_pair(dw, dg, model, q, opts, {"DW_DIRECT": "2"}, trace)
    assert lines[:3] == ["X", str(len(q)), "retry"], lines[:6]
    _assert_compact_equal(a, b, "forced")
    a, b, lines = _compact_pair(dw, dg, model, q, opts, {}, trace)
    assert "X" not in lines, lines[:6]
    _assert_compact_equal(a, b, "default")
    r = dw.run_queries(dg, model, q, opts)
    assert r.stats["steps"] > 0 and (r.lengths < 41).any()
    assert np.array_equal(np.diff(a[0].astype(np.int64)), r.lengths.astype(np.int64))


def _write_dwg1(path, row, col, prop, label=None):
    """DWG1 as dynwalk::save_binary writes it (graph.cpp:243-256)."""
    with open(path, "wb") as f:
        f.write(b"DWG1" + (1).to_bytes(4, "little") + bytes([1 if label is not None else 0]))
        for a in (np.asarray(row, np.uint64), np.asarray(col, np.uint32),
                  np.asarray(prop, np.float32)) + (() if label is None
                                                   else (np.asarray(label, np.uint16),)):
            f.write(len(a).to_bytes(8, "little"))
            f.write(a.tobytes())


def test_dwg1_loader_matches_reference(dw, orc, tmp_path):
    """A DWG1 file streamed to the device equals dynwalk::load_binary's graph,
    including unsorted slices (stable-sorted on load) and targets beyond the
    offsets array (they extend the vertex count), and walks equal the oracle."""
    og = build_oracle_graph(GRAPHS["ba300_labels"])
    a = og.arrays()
    p1 = str(tmp_path / "g1.dwg1")
    _write_dwg1(p1, a["row"], a["col"], a["prop"], a["label"])
    dg = dw.DeviceGraph.load_dwg1(p1)
    b = dg.download()
    for k in ("row", "col", "prop", "label", "nmax", "nsum"):
        assert np.array_equal(a[k], b[k]), k
    q = np.arange(og.nv, dtype=np.uint32)
    r_dev, r_orc = run_both(dw, orc, og, dg, dict(kind="node2vec", a=0.5, b=2.0), q, "adaptive",
                            30, 1.2)
    assert_same(r_dev, r_orc)
    # unsorted slices with duplicates, and a target id past the offsets array
    rng = np.random.default_rng(9)
    row = np.array([0, 4, 4, 9, 12], np.uint64)
    col = np.array([3, 1, 3, 0, 2, 7, 2, 2, 1, 0, 5, 0], np.uint32)
    prop = rng.uniform(1.0, 5.0, len(col)).astype(np.float32)
    lab = rng.integers(0, 4, len(col)).astype(np.uint16)
    p2 = str(tmp_path / "g2.dwg1")
    _write_dwg1(p2, row, col, prop, lab)
    b = dw.DeviceGraph.load_dwg1(p2).download()
    if orc.ref_available():
        ref = orc.RefGraph.load_binary(p2).arrays()
        for k in ("row", "col", "prop", "label", "nmax", "nsum"):
            assert np.array_equal(ref[k], b[k]), k
    assert len(b["row"]) == 9  # vertex 7 referenced: 8 vertices
    assert list(b["col"][0:4]) == [0, 1, 3, 3] and b["prop"][2] == prop[0] and b["prop"][3] == prop[2]
    # truncated and corrupt files
    p3 = str(tmp_path / "trunc.dwg1")
    open(p3, "wb").write(open(p1, "rb").read()[:-10])
    with pytest.raises(dw.DynwalkError, match="truncated binary graph file"):
        dw.DeviceGraph.load_dwg1(p3)
    p4 = str(tmp_path / "corrupt.dwg1")
    _write_dwg1(p4, np.array([0, 3], np.uint64), col[:2], prop[:2])
    with pytest.raises(dw.DynwalkError, match="corrupt binary graph file"):
        dw.DeviceGraph.load_dwg1(p4)


def test_write_paths_text_sink(dw, orc, tmp_path):
    """dw_run_write_paths is byte-identical to write_paths (runtime.cpp:280-291)
    applied to the same paths, over many ring batches and with query errors."""
    og = orc.Graph.rmat(13, 16, 31).synth_philox("uniform", 1.0, 5.0, seed=32)
    dg = to_device(dw, og)
    rng = np.random.default_rng(8)
    q = rng.integers(0, og.nv + 40, 2_300_000).astype(np.uint32)
    opts = dw.RunOptions(mode="adaptive", walk_length=12, seed=9, edge_cost_ratio=1.3)
    model = dw.Model(a=0.5, b=2.0)
    out = str(tmp_path / "paths.txt")
    st = dw.run_write_paths(dg, model, q, opts, out)
    r = dw.run_queries(dg, model, q, opts)
    lines = [" ".join(map(str, r.paths[i, :r.lengths[i]])) for i in range(len(q))]
    want = ("\n".join(lines) + "\n").encode()
    got = open(out, "rb").read()
    assert got == want
    assert st["steps"] == r.stats["steps"] and st["query_errors"] == r.stats["query_errors"] > 0
    with pytest.raises(dw.DynwalkError, match="cannot open paths output file"):
        dw.run_write_paths(dg, model, q[:10], opts, str(tmp_path / "no" / "such" / "dir.txt"))


def test_two_replicas_on_one_device(dw, orc, tmp_path, monkeypatch):
    """The multi-device engine (batches round-robin over the replicas, drains
    in query order, offset fix-up) exercised with two replicas of the graph on
    device 0: padded, compact and text outputs equal the single-replica run,
    and replica 1 starts walking before replica 0 is drained (no cross-device
    drain chain)."""
    og = orc.Graph.rmat(12, 16, 51).synth_philox("uniform", 1.0, 5.0, seed=52)
    a = og.arrays()
    one = dw.DeviceGraph.from_csr(a["row"], a["col"], a["prop"], devices=[0])
    two = dw.DeviceGraph.from_csr(a["row"], a["col"], a["prop"], devices=[0, 0])
    rng = np.random.default_rng(4)
    q = rng.integers(0, og.nv + 9, 3_000_000).astype(np.uint32)
    model = dw.Model(a=0.5, b=2.0)
    opts = dw.RunOptions(mode="adaptive", walk_length=16, seed=21, edge_cost_ratio=1.2)
    r1 = dw.run_queries(one, model, q, opts)
    r2 = dw.run_queries(two, model, q, opts)
    assert np.array_equal(r1.paths, r2.paths) and np.array_equal(r1.lengths, r2.lengths)
    for k in ("steps", "trials", "rng_draws", "query_errors"):
        assert r1.stats[k] == r2.stats[k], k
    o1, f1, _ = dw.run_queries_compact(one, model, q, opts)
    trace = tmp_path / "engine.trace"
    monkeypatch.setenv("DW_ENGINE_TRACE", str(trace))
    o2, f2, _ = dw.run_queries_compact(two, model, q, opts)
    monkeypatch.delenv("DW_ENGINE_TRACE")
    assert np.array_equal(o1, o2) and np.array_equal(f1, f2)
    ev = [ln.split() for ln in open(trace).read().splitlines()]
    first_drain0 = next(i for i, e in enumerate(ev) if e[0] == "D" and e[2] == "0")
    first_enq1 = next(i for i, e in enumerate(ev) if e[0] == "E" and e[2] == "1")
    assert first_enq1 < first_drain0
    drains = [e[2] for e in ev if e[0] == "D"]
    assert len(drains) >= 4 and drains[:4] == ["0", "1", "0", "1"]
    dw.run_write_paths(one, model, q[:200_000], opts, str(tmp_path / "a.txt"))
    dw.run_write_paths(two, model, q[:200_000], opts, str(tmp_path / "b.txt"))
    assert open(tmp_path / "a.txt", "rb").read() == open(tmp_path / "b.txt", "rb").read()


def test_calibration_with_and_without_free_rejections(dw):
    """The calibration's random pass skips the edge read of a trial above the
    row's non-return maximum (the kernel's free rejection) and runs with the
    screen switched off as well.  Both give a positive, finite ratio; their
    order is a timing matter and is not asserted (K4)."""
    import os
    dg = dw.DeviceGraph.rmat(16, 16, seed=5)
    m = dw.Model(kind="node2vec", a=0.5, b=2.0)
    with_screen = dw.profile_edge_cost_ratio(dg, m, seed=1)
    os.environ["DW_SHORTCUT"] = "0"
    try:
        without = dw.profile_edge_cost_ratio(dg, m, seed=1)
    finally:
        del os.environ["DW_SHORTCUT"]
    assert np.isfinite(with_screen) and with_screen > 0
    assert np.isfinite(without) and without > 0


@pytest.mark.parametrize("batch", [None, 37_000])
def test_batched_engine_equals_one_launch(dw, batch):
    """The run engine's batches (default plan with its geometric tail, or
    DW_BATCH-forced small batches cycling the three ring slots many times)
    give the same paths, lengths and counters as one device-resident launch
    over all queries: per-batch qid bases, slot reuse and the offset chain
    are invisible in the output."""
    import ctypes as C
    import os
    import torch
    dg = dw.DeviceGraph.rmat(12, 16, seed=31)
    rng = np.random.default_rng(9)
    q = rng.integers(0, 1 << 12, 620_000).astype(np.uint32)  # > 2 default batches
    L = 12
    model = dw.Model(a=0.5, b=2.0)
    opts = dw.RunOptions(walk_length=L, seed=3, edge_cost_ratio=1.4)
    dq = torch.from_numpy(q.view(np.int32)).cuda()
    dp = torch.empty((len(q), L + 1), dtype=torch.int32, device="cuda")
    dl = torch.empty(len(q), dtype=torch.int32, device="cuda")
    lib = dw.load_library()
    m, o = model.c(), opts.c()
    torch.cuda.synchronize()
    assert lib.dw_run_device(dg.h, 0, C.byref(m), C.c_void_p(dq.data_ptr()), len(q), C.byref(o),
                             C.c_void_p(dp.data_ptr()), C.c_void_p(dl.data_ptr()), None) == 0
    st = dw.RunStatsC()
    assert lib.dw_run_device_sync(dg.h, 0, C.byref(st)) == 0
    one_paths = dp.cpu().numpy().view(np.uint32)
    one_len = dl.cpu().numpy().view(np.uint32)
    if batch:
        os.environ["DW_BATCH"] = str(batch)
    try:
        r = dw.run_queries(dg, model, q, opts)
        offs, flat, st2 = dw.run_queries_compact(dg, model, q, opts)
    finally:
        os.environ.pop("DW_BATCH", None)
    assert np.array_equal(r.lengths, one_len)
    mask = np.arange(L + 1)[None, :] < one_len[:, None]
    assert np.array_equal(r.paths[mask], one_paths[mask])
    assert np.array_equal(np.diff(offs.astype(np.int64)), one_len.astype(np.int64))
    assert np.array_equal(flat, one_paths[mask])
    for k in ("steps", "trials", "rng_draws", "weight_reads", "select_erjs", "select_ervs"):
        assert r.stats[k] == getattr(st, k) == st2[k], k


@pytest.mark.parametrize("fat", ["1", "0"])
@pytest.mark.parametrize("mode", ["adaptive", "force-erjs"])
def test_pr2_pareto_cooperative_erjs(dw, orc, mode, fat):
    """Second-order PageRank on Pareto weights: steps run thousands of trials,
    so lanes hand their steps to the warp-cooperative eRJS (32 trials per
    round, first acceptance in trial order).  Paths and counters stay
    bit-exact, in the fat and the slim layout."""
    import os
    og = orc.Graph.rmat(11, 16, 3).synth_philox("pareto", alpha=1.0, seed=4)
    os.environ["DW_FAT"] = fat
    try:
        dg = dw.DeviceGraph.rmat(11, 16, seed=3, weights="pareto", alpha=1.0, weight_seed=4)
    finally:
        del os.environ["DW_FAT"]
    q = np.arange(og.nv, dtype=np.uint32)
    r_dev, r_orc = run_both(dw, orc, og, dg, dict(kind="pr2", gamma=0.15), q, mode, 30, 1.2)
    assert r_orc.stats["trials"] > 50 * r_orc.stats["steps"]  # heavy-tailed steps: CJS engaged
    assert_same(r_dev, r_orc, (mode, fat))


def _hub_graph(orc, n=120_000, seed=31):
    """Hubs far above one warp chunk: node 0 joined to every node, node 1 to
    every 3rd, node 2 to every 7th, the hubs joined to each other, plus a ring
    and random chords; mirrored, Philox weights.  A hub scan's prev is a small
    node (membership from prev's side, corr_ranges) or another hub (hash
    probes)."""
    rng = np.random.default_rng(seed)
    v = np.arange(3, n, dtype=np.uint32)
    src = np.concatenate([np.zeros(n - 3, np.uint32), np.ones(len(v[::3]), np.uint32),
                          np.full(len(v[::7]), 2, np.uint32), v[:-1]])
    dst = np.concatenate([v, v[::3], v[::7], v[1:]])
    extra = rng.integers(3, n, size=(2, n), dtype=np.uint32)  # a few random chords
    # hub-hub edges (a hub's scan with a hub as prev: hash probes) and a
    # multi-edge (one target repeated in a hub row)
    src = np.concatenate([src, extra[0], np.array([0, 0, 1, 0, 0], np.uint32)])
    dst = np.concatenate([dst, extra[1], np.array([1, 2, 2, 5, 5], np.uint32)])
    return orc.Graph.build(src, dst, mirror=True, nv_hint=n).synth_philox(
        "uniform", 1.0, 5.0, seed=seed + 1)


@pytest.mark.parametrize("slack", ["1", "1e13"], ids=["band", "replay"])
@pytest.mark.parametrize("mode", ["force-ervs", "ervs-nojump"])
@pytest.mark.parametrize("mk", [dict(kind="node2vec", a=0.5, b=2.0),
                                dict(kind="node2vec", a=2.0, b=0.5),
                                dict(kind="pr2", gamma=0.2),
                                dict(kind="static", weighted=True)])
def test_hub_rows_warp_reservoir(dw, orc, mk, mode, slack):
    """The warp reservoir (dw_walk_kernel.cuh ervs_warp) on rows of 17K-120K
    neighbours: the parallel jump chain decides every crossing from prefix
    sums and a rigorous rounding band, and replays the exact chain only when
    the band straddles 0.  DW_ERVS_SLACK=1e13 widens the band so that almost
    every crossing goes through the replay.  Both are bit-exact against the
    oracle's sequential chain (samplers.hpp:65-137)."""
    og = _hub_graph(orc)
    dg = to_device(dw, og)
    # walkers on and next to the hubs: every step of theirs scans a hub row
    q = np.concatenate([np.zeros(32, np.uint32), np.ones(32, np.uint32),
                        np.full(32, 2, np.uint32), np.arange(3, 3 + 160, dtype=np.uint32)])
    r_dev, r_orc = _with_env({"DW_ERVS_SLACK": slack},
                             lambda: run_both(dw, orc, og, dg, mk, q, mode, 16, 1.2))
    assert_same(r_dev, r_orc, (mk, mode, slack))
    assert r_dev.stats["weight_reads"] > 50 * 100_000


@pytest.mark.parametrize("layout", ["fat", "slim"])
@pytest.mark.parametrize("mode", ["adaptive", "force-erjs"])
def test_tier2_handoff_bit_exact_and_chi_square(dw, orc, mode, layout):
    """Tier-2 eRJS hand-off (dw_run_opts.erjs_handoff): PR2 gamma=0.15 on
    Pareto weights, the config-4 pathology.  The device equals the oracle
    run with the same rule in paths and counters, the hand-off fires, and the
    device's per-(prev, cur) transition frequencies on hub and non-hub rows
    pass chi-square against the exact probabilities."""
    from tests.chisq import transition_pvalues
    og = orc.Graph.rmat(12, 16, 3).synth_philox("pareto", alpha=1.0, seed=4)
    dg = _with_env({"DW_FAT": "1" if layout == "fat" else "0"}, lambda: to_device(dw, og))
    mk = dict(kind="pr2", gamma=0.15)
    q = np.arange(og.nv, dtype=np.uint32)
    o = dict(mode=mode, walk_length=40, seed=7, edge_cost_ratio=1.0)
    r_dev = dw.run_queries(dg, dw.Model(**mk), q, dw.RunOptions(erjs_handoff=1.0, **o))
    r_orc = orc.run(og, orc.Model(**mk), q, mode=mode, walk_length=40, seed=7, ratio=1.0,
                    rng="philox", threads=os.cpu_count() or 1, erjs_handoff=1.0)
    assert_same(r_dev, r_orc, (mode, layout))
    assert r_dev.stats["erjs_fallbacks"] > 100
    deg = np.diff(og.arrays()["row"])
    hubs = np.argsort(deg)[-3:]
    small = np.flatnonzero((deg >= 2) & (deg <= 8))[:3]
    starts = np.repeat(np.concatenate([hubs, small]).astype(np.uint32), 40_000)
    r = dw.run_queries(dg, dw.Model(**mk), starts,
                       dw.RunOptions(erjs_handoff=1.0, **dict(o, walk_length=2, seed=13)))
    ps, pooled = transition_pvalues(orc, og, orc.Model(**mk), r.paths, starts)
    assert len(ps) >= 10 and pooled > 0.01 and min(ps) > 1e-4, (len(ps), pooled, min(ps))


def test_libdevice_log_exp_against_host_libm(dw, orc):
    """eRVS keys, thresholds and floors use log/exp (samplers.hpp:82-97).  The
    device computes them with CUDA libdevice, the reference with glibc.  Over
    the inputs the samplers form -- open01 values and floor + open01 (1 -
    floor) for log, w * key <= 0 for exp -- the two never differ by more than
    1 ulp.  An outcome can then flip only when two keys, or a threshold and
    the chain, fall within ~2 ulp of each other (probability ~2^-51 per
    comparison); the measured disagreement rates are printed for DESIGN.md."""
    import ctypes as C
    rng = np.random.default_rng(17)
    n = 1 << 22
    u = rng.integers(0, 2**64, size=n, dtype=np.uint64)
    x_log = ((u >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0**-53
    fl = np.exp(-rng.exponential(3.0, size=n))
    x_log2 = fl + x_log * (1.0 - fl)
    x_exp = -np.exp(rng.uniform(-30.0, 6.0, size=n))
    lib = dw.load_library()
    for fn, x in ((0, x_log), (0, x_log2), (1, x_exp)):
        x = np.ascontiguousarray(x)
        yd = np.empty_like(x)
        yh = np.empty_like(x)
        assert lib.dw_selftest_math(fn, x.ctypes.data_as(dw.f64p), yd.ctypes.data_as(dw.f64p),
                                    n) == 0
        orc.lib().orc_libm(fn, x.ctypes.data_as(C.POINTER(C.c_double)),
                           yh.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint64(n))
        ok = np.isfinite(yh) & (yh != 0)
        assert np.array_equal(np.isfinite(yd), np.isfinite(yh))
        ulp = np.abs(yd[ok].view(np.int64) - yh[ok].view(np.int64))
        print(f"fn={fn} differ={np.count_nonzero(ulp) / ok.sum():.3e} max_ulp={ulp.max()}")
        assert ulp.max() <= 1


@pytest.mark.parametrize("lab2", ["1", "0"], ids=["packed-labels", "no-screen"])
@pytest.mark.parametrize("labels,schema", [((0, 3), (0, 1, 2, 3) * 20),
                                           ((0, 3), (2, 0, 7, 1) * 10),
                                           ((0, 5), (0, 4, 5, 1) * 20)],
                         ids=["4-labels", "absent-label", "6-labels"])
def test_metapath_label_screen(dw, orc, labels, schema, lab2):
    """MetaPath trials are judged on a 2-bit packed label (DevGraph::lab2,
    built when every label is < 4) before their record is gathered; a label
    miss is a rejection with no gather.  Paths and counters equal the oracle
    with the screen (packed labels), without it (DW_LAB2=0) and when labels
    do not fit 2 bits (no packing), including a schema label that no edge
    carries (dead rows)."""
    og = orc.Graph.rmat(12, 16, 8).synth_philox("uniform", 1.0, 5.0, seed=9)
    og.synth_philox("labels", labels[0], labels[1], seed=10)
    dg = _with_env({"DW_LAB2": lab2, "DW_FAT": "1"}, lambda: to_device(dw, og))
    q = np.arange(og.nv, dtype=np.uint32)
    mk = dict(kind="metapath", schema=schema)
    for mode in ("adaptive", "force-erjs"):
        r_dev, r_orc = run_both(dw, orc, og, dg, mk, q, mode, len(schema), 1.2)
        assert_same(r_dev, r_orc, (labels, schema, lab2, mode))
