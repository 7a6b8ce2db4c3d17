"""Parity at the headline's scale and layout, and against the reference's own
sampler templates on hub-heavy R-MAT graphs (-m gpu).

* The bench's own device-generated graph (R-MAT ef16, seeds 1/2, uniform
  [1,5) weights) at scale 20, default layout (compact 32 B fat records for
  node2vec), at the calibrated ratio the headline runs with (~2.3) and at
  1.6: 50K sampled walkers of length 80, adaptive and force-erjs, bit-exact
  against the oracle in paths, lengths and every RunStats counter.
* The same graph through dw_run_compact's direct engine (every vertex a
  start, ratio 0.5 as calibrated at s24): equal to the padded run and, on a
  sample, to the oracle.
* R-MAT s13 / s14 (max degree in the thousands): the GPU against
  ref_run_philox, i.e. the reference's samplers.hpp / models.hpp /
  runtime.cpp templates driven by the same Philox stream, for node2vec
  (0.5, 2) and (2, 0.5) and second-order PageRank in all four modes."""
import os

import numpy as np
import pytest

from tests.golden.make_golden import stats_core

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 4


def _same(r_dev, r_ref, tag):
    assert stats_core(r_dev.stats) == stats_core(r_ref.stats), tag
    assert np.array_equal(r_dev.lengths, r_ref.lengths), tag
    assert np.array_equal(r_dev.paths, r_ref.paths), tag


@pytest.fixture(scope="module")
def bench_s20(dw, orc):
    import bench
    dg = dw.DeviceGraph.rmat(20, 16, seed=bench.TOPO_SEED, weights="uniform", low=1.0, high=5.0,
                             weight_seed=bench.WEIGHT_SEED)
    a = dg.download()
    og = orc.Graph.from_csr(a["row"], a["col"], a["prop"])
    return dg, og


@pytest.mark.parametrize("ratio", [2.33, 1.6])
@pytest.mark.parametrize("mode", ["adaptive", "force-erjs"])
def test_bench_graph_s20_parity(dw, orc, bench_s20, ratio, mode):
    import bench
    dg, og = bench_s20
    nv = og.nv
    q = np.arange(0, nv, nv // 50_000, dtype=np.uint32)[:50_000]
    mk = dict(kind="node2vec", a=0.5, b=2.0)
    r_dev = dw.run_queries(dg, dw.Model(**mk), q,
                           dw.RunOptions(mode=mode, walk_length=80, seed=bench.WALK_SEED,
                                         edge_cost_ratio=ratio))
    r_orc = orc.run(og, orc.Model(**mk), q, mode=mode, walk_length=80, seed=bench.WALK_SEED,
                    ratio=ratio, rng="philox", threads=THREADS)
    _same(r_dev, r_orc, (ratio, mode))
    # the sample exercises both samplers and hub rows
    assert r_dev.stats["steps"] > 1_000_000
    if mode == "adaptive":
        assert r_dev.stats["select_ervs"] > 1000 and r_dev.stats["select_erjs"] > 100_000


def test_bench_graph_s20_direct_compact(dw, orc, bench_s20, tmp_path):
    """The headline's end-to-end path at scale 20: dw_run_compact on the
    bench graph takes the direct engine (trace line "X nq ok"), and its
    offsets and ids equal the padded run's for every vertex as a start, and
    the oracle's on a sample."""
    import bench
    dg, og = bench_s20
    nv = og.nv
    q = np.arange(nv, dtype=np.uint32)
    model = dw.Model(kind="node2vec", a=0.5, b=2.0)
    opts = dw.RunOptions(mode="adaptive", walk_length=80, seed=bench.WALK_SEED,
                         edge_cost_ratio=0.5)
    trace = str(tmp_path / "trace.txt")
    os.environ["DW_ENGINE_TRACE"] = trace
    try:
        offs, flat, st = dw.run_queries_compact(dg, model, q, opts)
    finally:
        os.environ.pop("DW_ENGINE_TRACE", None)
    assert open(trace).read().split()[:3] == ["X", str(nv), "ok"]
    r = dw.run_queries(dg, model, q, opts)
    assert np.array_equal(np.diff(offs.astype(np.int64)), r.lengths.astype(np.int64))
    mask = np.arange(r.paths.shape[1])[None, :] < r.lengths[:, None]
    assert np.array_equal(flat, r.paths[mask])
    assert stats_core(st) == stats_core(r.stats)
    qs = q[::nv // 20_000][:20_000]
    r_orc = orc.run(og, orc.Model(kind="node2vec", a=0.5, b=2.0), qs, mode="adaptive",
                    walk_length=80, seed=bench.WALK_SEED, ratio=0.5, rng="philox",
                    threads=THREADS, qids=qs.astype(np.uint64))  # walker id = vertex id
    o = offs.astype(np.int64)
    sel = np.concatenate([np.arange(o[i], o[i + 1]) for i in qs.astype(np.int64)])
    assert np.array_equal(flat[sel], r_orc.paths[np.arange(r_orc.paths.shape[1])[None, :]
                                                 < r_orc.lengths[:, None]])


@pytest.fixture(scope="module", params=[13, 14])
def rmat_pair(request, dw, ref):
    s = request.param
    og = ref.Graph.rmat(s, 16, 40 + s).synth_philox("uniform", 1.0, 5.0, seed=50 + s)
    a = og.arrays()
    rg = ref.RefGraph.from_csr(a["row"], a["col"], a["prop"])
    dg = dw.DeviceGraph.from_csr(a["row"], a["col"], a["prop"])
    return s, og.nv, rg, dg


@pytest.mark.parametrize("mode", ["adaptive", "force-erjs", "force-ervs", "ervs-nojump"])
@pytest.mark.parametrize("mk", [dict(kind="node2vec", a=0.5, b=2.0),
                                dict(kind="node2vec", a=2.0, b=0.5),
                                dict(kind="pr2", gamma=0.2)],
                         ids=["n2v-0.5-2", "n2v-2-0.5", "pr2"])
def test_gpu_matches_reference_templates_rmat(dw, ref, rmat_pair, mk, mode):
    s, nv, rg, dg = rmat_pair
    q = np.arange(nv, dtype=np.uint32)
    L = 80 if s == 13 else 40
    r_dev = dw.run_queries(dg, dw.Model(**mk), q,
                           dw.RunOptions(mode=mode, walk_length=L, seed=9, edge_cost_ratio=1.3))
    r_ref = ref.ref_run(rg, ref.Model(**mk), q, mode=mode, walk_length=L, seed=9, ratio=1.3,
                        rng="philox", workers=THREADS)
    _same(r_dev, r_ref, (s, mk, mode))
