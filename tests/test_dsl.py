"""DSL walk models compiled into the walk kernel.

The product's codegen (paper_2512_00705_b200/host/dsl_codegen.hpp) turns the
reference's own parse + analysis of a DslWalk program into a CUDA model
functor; dw_model_compile() builds it with NVRTC into walk_kernel.  The GPU
runs must equal the reference's DslWalk (its interpreter and derived
estimators) driven through the reference's sampler templates on the same
Philox stream: paths and every counter bit-exact.  The programs below are
written for these tests and cover dist (all three values), labels and an
array parameter indexed by step, walk_length, min/max/let, logical operators,
label aggregates in the estimators, and a loop (estimation flag NONE)."""
import numpy as np
import pytest

PROGRAMS = {
    "second_order": """
param p = 0.25;
param q = 4.0;
fn weight() {
    if (dist == 0) { return h / p; }
    if (dist == 1) { return h; }
    return h / q;
}
""",
    "schema": """
param order = [1, 0, 3, 2, 1, 0];
param walk_length = 6;
fn weight() {
    if (label == order[step]) { return h * 2.0; }
    if (label < 2 && step > 2) { return h * 0.5; }
    return 0.0;
}
""",
    "label_degree": """
param boost = 0.3;
fn weight() {
    let m = max(deg_cur, deg_prev);
    let base = h + label;
    if (dist == 1 || dist == 0) { return base * (1.0 + boost) / m * deg_cur; }
    return min(base, 3.0) / m * deg_cur;
}
""",
    "loop": """
fn weight() {
    let acc = 1.0;
    let i = 0;
    while (i < 2) { acc = acc * h; i = i + 1; }
    return acc + step;
}
""",
    "unweighted_not": """
param a = 2.0;
fn weight() {
    if (!(dist == 2)) { return 1.0 / a; }
    return 1.0;
}
""",
}


@pytest.fixture(scope="module")
def codegen(ref):
    return {k: ref.dsl_codegen(v) for k, v in PROGRAMS.items()}


def test_codegen_compiles_with_nvrtc(dw, codegen):
    """Every program generates a functor that NVRTC compiles into the walk
    kernel for all four sampler modes (no GPU needed to compile)."""
    for name, (src, ms, fl) in codegen.items():
        try:
            m = dw.CustomModel(src, ms, fl)
        except dw.DynwalkError as e:
            if e.code == -4:  # DW_EUNSUPPORTED: no NVRTC on this machine
                pytest.skip(str(e))
            raise
        del m
    assert codegen["schema"][1] == 6 and codegen["label_degree"][2] == 1
    assert "dsl_weight" in codegen["second_order"][0]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_dsl_models_match_reference(dw, ref, codegen, name):
    og = ref.Graph.rmat(11, 16, 41).synth_philox("uniform", 1.0, 5.0, seed=42)
    og.synth_philox("labels", 0, 3, seed=43)
    a = og.arrays()
    dg = dw.DeviceGraph.from_csr(a["row"], a["col"], a["prop"], a["label"])
    rg = ref.RefGraph.from_csr(a["row"], a["col"], a["prop"], a["label"])
    src, ms, fl = codegen[name]
    cm = dw.CustomModel(src, ms, fl)
    q = np.arange(og.nv, dtype=np.uint32)
    ref.set_dsl_source(PROGRAMS[name])
    for mode in ("adaptive", "force-erjs", "force-ervs", "ervs-nojump"):
        r_dev = dw.run_queries(dg, dw.Model("custom", custom=cm), q,
                               dw.RunOptions(mode=mode, walk_length=20, seed=11,
                                             edge_cost_ratio=1.3))
        r_ref = ref.ref_run(rg, ref.Model("dsl"), q, mode=mode, walk_length=20, seed=11,
                            ratio=1.3, rng="philox", workers=4)
        for k in ("steps", "select_erjs", "select_ervs", "trials", "weight_reads", "rng_draws",
                  "erjs_fallbacks", "dead_ends", "query_errors"):
            assert r_dev.stats[k] == r_ref.stats[k], (name, mode, k)
        assert np.array_equal(r_dev.lengths, r_ref.lengths), (name, mode)
        assert np.array_equal(r_dev.paths, r_ref.paths), (name, mode)
