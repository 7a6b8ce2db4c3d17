"""CPU suite: pins the oracle (oracle/) against the reference's golden vectors,
known-answer tests and the reference code itself (oracle/_ref)."""
import json
import os

import numpy as np
import pytest

from tests.golden.make_golden import CASES, GRAPHS, MODES, build_oracle_graph, case_id, digest, \
    stats_core

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---- RNG -------------------------------------------------------------------

def test_philox_known_answers(orc):
    """Random123 kat_vectors for philox4x32-10."""
    import ctypes as C
    kat = [
        ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
        ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
        ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
         (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
    ]
    for ctr, key, want in kat:
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        orc.lib().orc_philox4x32_10(c, k, o)
        assert tuple(o) == want


def test_mt19937_64_standard_value(orc):
    """[rand.predef]: the 10000th draw of a default mt19937_64 is 9981545732273789042."""
    out = np.empty(10000, np.uint64)
    orc.lib().orc_mt19937_64(5489, 10000, out.ctypes.data_as(orc.u64p))
    assert int(out[-1]) == 9981545732273789042


def test_derive_seed_matches_splitmix(orc):
    def py_derive(seed, stream):
        M = 2**64 - 1
        st = (seed ^ ((stream * 0x9e3779b97f4a7c15 + 0x2545f4914f6cdd1d) & M)) & M

        def nxt():
            nonlocal st
            st = (st + 0x9e3779b97f4a7c15) & M
            z = st
            z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M
            z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M
            return z ^ (z >> 31)
        nxt()
        return nxt()
    for s, t in [(0, 0), (13, 1), (13, 2), (2**63 + 5, 0x70726f66)]:
        assert orc.derive_seed(s, t) == py_derive(s, t)


def test_walker_stream_layout(orc):
    """draw 2k / 2k+1 are the low / high 64-bit halves of Philox block k."""
    import ctypes as C
    seed, qid, step = 0x1234_5678_9abc_def0, 77, 5
    for k in range(3):
        c = (C.c_uint32 * 4)(k, step, qid, 0)
        key = (C.c_uint32 * 2)(seed & 0xffffffff, seed >> 32)
        o = (C.c_uint32 * 4)()
        orc.lib().orc_philox4x32_10(c, key, o)
        assert orc.lib().orc_walker_draw(seed, qid, step, 2 * k) == o[0] | (o[1] << 32)
        assert orc.lib().orc_walker_draw(seed, qid, step, 2 * k + 1) == o[2] | (o[3] << 32)


# ---- the reference CLI golden ------------------------------------------------

def test_stats_walk_golden(orc):
    """proj/tests/golden/stats_walk.txt, counter for counter (test_cli.cpp:123-131)."""
    gold = json.load(open(os.path.join(GOLDEN, "stats_walk.json")))
    v = gold["values"]
    g = orc.Graph.ba(50, 4, orc.derive_seed(13, 1), True)
    g.synth("uniform", 1, 5, seed=orc.derive_seed(13, 2))
    assert g.nv == int(v["graph_vertices"]) and g.ne == int(v["graph_edges"])
    r = orc.run(g, orc.Model("node2vec"), np.arange(50), mode="adaptive", walk_length=10,
                seed=13, ratio=4.0, rng="mt19937", threads=2)
    s = r.stats
    for k in ("query_errors", "dead_ends", "steps", "select_ervs", "select_erjs", "trials",
              "weight_reads", "rng_draws", "erjs_fallbacks", "queries"):
        assert s[k] == int(v[k]), k
    assert int((r.lengths > 0).sum()) == int(v["paths_emitted"])
    assert int(r.lengths.sum()) == int(v["paths_total_nodes"])
    hist = [[b, e0, e1] for b, (e0, e1) in enumerate(s["selection_by_degree"]) if e0 or e1]
    assert hist == gold["selection_histogram"]


# ---- known-answer tests from the reference unit tests ------------------------

def second_order_fixture(orc):
    """test_util.hpp:22-36: prev=0, N(0)={1,2}; cur=1, N(1)={0,2,3,4}; (1,3) has prop 3."""
    src = [0, 0, 1, 1, 1, 1]
    dst = [1, 2, 0, 2, 3, 4]
    prop = [1, 1, 1, 1, 3, 1]
    return orc.Graph.build(src, dst, prop)


def test_node2vec_weights(orc):
    """test_models.cpp:13-28: weights 0.5 / 1 / 6 / 2 and first step = raw h."""
    g = second_order_fixture(orc)
    m = orc.Model("node2vec", a=2.0, b=0.5).c()
    e0 = int(g.arrays()["row"][1])
    got = [orc.lib().orc_weight(g.ptr, m, 1, 0, 1, e0 + i) for i in range(4)]
    assert got == [0.5, 1.0, 6.0, 2.0]
    assert orc.lib().orc_weight(g.ptr, m, 1, orc.INVALID, 0, e0 + 2) == 3.0


def test_pr2_weights(orc):
    """test_models.cpp:59-75: 1.2 for a neighbour of prev, 0.8 otherwise and for a return."""
    g = second_order_fixture(orc)
    m = orc.Model("pr2", gamma=0.2).c()
    e0 = int(g.arrays()["row"][1])
    w = [orc.lib().orc_weight(g.ptr, m, 1, 0, 1, e0 + i) for i in range(4)]
    assert w[1] == pytest.approx(1.2, rel=1e-12)
    assert w[3] == pytest.approx(0.8, rel=1e-12)
    assert w[0] == pytest.approx(0.8, rel=1e-12)


def test_decide_sampler_arithmetic(orc):
    """test_runtime.cpp:33-66: star est_max=4, est_sum=10 -> eRJS at ratio 1, eRVS at 3."""
    g = orc.Graph.build([0, 0, 0, 0], [1, 2, 3, 4], [3, 2, 4, 1])
    import ctypes as C
    mx, sm = C.c_double(), C.c_double()
    m = orc.Model("static").c()
    assert orc.lib().orc_decide(g.ptr, m, 0, orc.INVALID, 0, 1.0, C.byref(mx), C.byref(sm)) == 1
    assert (mx.value, sm.value) == (4.0, 10.0)
    assert orc.lib().orc_decide(g.ptr, m, 0, orc.INVALID, 0, 3.0, C.byref(mx), C.byref(sm)) == 0


def test_star_aggregates(orc):
    """test_graph.cpp:31-40: star max=4, sum=10."""
    g = orc.Graph.build([0, 0, 0, 0], [1, 2, 3, 4], [3, 2, 4, 1])
    a = g.arrays()
    assert a["nmax"][0] == 4.0 and a["nsum"][0] == 10.0


def test_dead_end_cap(orc):
    """test_samplers.cpp:262-280: all-zero row -> cap*d trials, reads = trials + d, dead end."""
    g = orc.Graph.build([0, 0], [1, 2], [1, 1], label=[2, 3])
    r = orc.run(g, orc.Model("metapath", schema=(0,)), [0], mode="force-erjs", walk_length=1,
                cap_per_degree=4, rng="mt19937", seed=8)
    s = r.stats
    assert s["trials"] == 8 and s["weight_reads"] == 8 + 2
    assert s["dead_ends"] == 1 and s["erjs_fallbacks"] == 1
    assert r.lengths[0] == 1


def test_query_errors_and_isolated(orc):
    """test_runtime.cpp:161-185: isolated start -> single-node path; out of range -> empty."""
    g = orc.Graph.build([0], [1], [1.0], nv_hint=4)
    r = orc.run(g, orc.Model("static"), [2, 3, 4999, 0], walk_length=5)
    assert list(r.lengths) == [1, 1, 0, 2]
    assert r.stats["query_errors"] == 1 and r.stats["steps"] == 1
    assert r.paths[2].tolist() == [orc.INVALID] * 6


def test_chi_square_star(orc):
    """test_samplers.cpp:63-73 analogue: each kernel matches the exact probabilities."""
    from scipy.stats import chisquare
    g = orc.Graph.build([0, 0, 0, 0], [1, 2, 3, 4], [3, 2, 4, 1])
    probs = orc.transition_probs(g, orc.Model("static"), 0)
    n = 100000
    for mode in ("force-erjs", "force-ervs", "ervs-nojump", "adaptive"):
        r = orc.run(g, orc.Model("static"), np.zeros(n, np.uint32), mode=mode, walk_length=1,
                    seed=5, ratio=2.49)
        counts = np.bincount(r.paths[:, 1].astype(np.int64) - 1, minlength=4)
        assert chisquare(counts, probs * n).pvalue > 1e-3, mode


# ---- oracle == reference, paths and counters ---------------------------------

@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0] + ":" + c[1]["kind"])
def test_oracle_matches_reference_goldens(orc, case):
    gold = {c["id"]: c for c in json.load(open(os.path.join(GOLDEN, "ref_walks.json")))["cases"]}
    gname, mk, L, ratio = case
    g = build_oracle_graph(GRAPHS[gname])
    q = np.arange(g.nv, dtype=np.uint32)
    m = orc.Model(**mk)
    for mode in MODES:
        r = orc.run(g, m, q, mode=mode, walk_length=L, seed=7, ratio=ratio, rng="philox",
                    threads=3)
        c = gold[case_id(gname, mk, mode, L)]
        assert stats_core(r.stats) == c["stats"], mode
        assert digest(r.paths, r.lengths) == c["digest"], mode
    r = orc.run(g, m, q, mode="adaptive", walk_length=L, seed=7, ratio=ratio, rng="mt19937",
                threads=3)
    c = gold[case_id(gname, mk, "adaptive", L) + "|mt19937"]
    assert stats_core(r.stats) == c["stats"]
    assert digest(r.paths, r.lengths) == c["digest"]


def test_oracle_matches_live_reference(ref):
    """Fresh randomized graphs against the reference run_queries (mt19937) and
    its sampler templates under Philox streams."""
    rs = np.random.default_rng(3)
    for trial in range(3):
        n, deg, seed = int(rs.integers(50, 400)), int(rs.integers(2, 9)), int(rs.integers(1e9))
        og = ref.Graph.ba(n, deg, seed, True).synth("pareto" if trial == 2 else "uniform",
                                                     alpha=1.5, seed=seed + 1)
        og.synth("labels", 0, 2, seed=seed + 2)
        rg = ref.RefGraph.gen("ba", n, deg, seed).synth("pareto" if trial == 2 else "uniform",
                                                         alpha=1.5, seed=seed + 1)
        rg.synth("labels", 0, 2, seed=seed + 2)
        for mk in (dict(kind="node2vec", a=0.7, b=1.9), dict(kind="pr2", gamma=0.3),
                   dict(kind="metapath", schema=(0, 1, 2) * 4, weighted=False),
                   dict(kind="static", weighted=False)):
            m = ref.Model(**mk)
            for mode in MODES:
                for rng in ("philox", "mt19937"):
                    a = ref.run(og, m, np.arange(n), mode=mode, walk_length=12, seed=trial,
                                ratio=1.1, rng=rng, threads=2)
                    b = ref.ref_run(rg, m, np.arange(n), mode=mode, walk_length=12, seed=trial,
                                    ratio=1.1, rng=rng, workers=2)
                    assert a.stats == b.stats, (mk, mode, rng)
                    assert np.array_equal(a.paths, b.paths), (mk, mode, rng)


def test_reference_generators_match(ref):
    """The oracle's BA / uniform generators + synthesize_weights equal the reference's."""
    for kind in ("ba", "uniform"):
        for mirror in (True, False):
            og = (ref.Graph.ba if kind == "ba" else ref.Graph.uniform)(500, 6, 99, mirror)
            og.synth("uniform", 1, 5, seed=5).synth("labels", 0, 4, seed=6)
            rg = ref.RefGraph.gen(kind, 500, 6, 99, mirror).synth("uniform", 1, 5, seed=5)
            rg.synth("labels", 0, 4, seed=6)
            a, b = og.arrays(), rg.arrays()
            for k in ("row", "col", "prop", "nmax", "nsum", "label"):
                assert np.array_equal(a[k], b[k]), (kind, mirror, k)
    og = ref.Graph.ba(300, 4, 7, True).synth("degree")
    rg = ref.RefGraph.gen("ba", 300, 4, 7).synth("degree")
    assert np.array_equal(og.arrays()["prop"], rg.arrays()["prop"])


# ---- the synthetic R-MAT workload ------------------------------------------

def test_rmat_graph_properties(orc):
    g = orc.Graph.rmat(10, 16, 42).synth_philox("uniform", 1.0, 5.0, seed=43)
    a = g.arrays()
    nv, row, col = g.nv, a["row"], a["col"]
    assert nv == 1024
    src = np.repeat(np.arange(nv), np.diff(row).astype(np.int64))
    # mirrored: the multiset of (u,v) equals that of (v,u) once self-loops are counted once
    fwd = np.sort(src.astype(np.uint64) << 32 | col)
    rev = np.sort(col.astype(np.uint64) << 32 | src.astype(np.uint64))
    assert np.array_equal(fwd, rev)
    for v in range(nv):
        s = col[row[v]:row[v + 1]]
        assert np.all(s[:-1] <= s[1:])
    assert a["prop"].min() >= 1.0 and a["prop"].max() < 5.0
    deg = np.diff(row)
    assert deg.max() > 20 * deg.mean()  # skewed


def test_tier2_handoff_keeps_the_distribution(orc):
    """Tier-2 eRJS hand-off (dw_run_opts.erjs_handoff, oracle.c erjs_cap): a
    step that runs max(32, ceil(h/ratio*d)) trials without acceptance falls
    back to the reservoir pass, as the reference's cap overrun does.  PR2 on
    Pareto weights (config 4's pathology: bounds far above the weights) with
    the hand-off: per-(prev, cur) transition frequencies over hub and
    non-hub rows pass chi-square against the exact probabilities, and the
    hand-off really fires."""
    from tests.chisq import transition_pvalues
    og = orc.Graph.rmat(10, 16, 3).synth_philox("pareto", alpha=1.0, seed=4)
    a = og.arrays()
    deg = np.diff(a["row"])
    # starts: the 4 largest rows and 4 rows of degree 2-8
    hubs = np.argsort(deg)[-4:]
    small = np.flatnonzero((deg >= 2) & (deg <= 8))[:4]
    starts = np.repeat(np.concatenate([hubs, small]).astype(np.uint32), 30_000)
    m = orc.Model("pr2", gamma=0.15)
    r = orc.run(og, m, starts, mode="adaptive", walk_length=2, seed=9, ratio=1.0,
                rng="philox", threads=os.cpu_count() or 1, erjs_handoff=1.0)
    base = orc.run(og, m, starts[:2000], mode="adaptive", walk_length=2, seed=9, ratio=1.0,
                   rng="philox", threads=os.cpu_count() or 1)
    assert r.stats["erjs_fallbacks"] > 1000 and base.stats["erjs_fallbacks"] == 0
    ps, pooled = transition_pvalues(orc, og, m, r.paths, starts)
    assert len(ps) >= 20
    assert pooled > 0.01 and min(ps) > 1e-4, (pooled, min(ps))
