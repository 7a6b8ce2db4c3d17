"""The product C++ shim (host/dynwalk_gpu.hpp) with the reference's own
signature dynwalk::gpu::run_queries, driven from reference types
(oracle/_ref/shim_check), must reproduce the reference goldens exactly."""
import json
import os
import subprocess

import numpy as np
import pytest

from tests.golden.make_golden import CASES, GRAPHS, case_id, digest, stats_core

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "oracle", "_ref", "shim_check")
GOLDEN = os.path.join(ROOT, "tests", "golden", "ref_walks.json")


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0] + ":" + c[1]["kind"])
def test_shim_reproduces_reference_goldens(case, tmp_path):
    if not os.path.exists(SHIM):
        pytest.skip("oracle/_ref/shim_check not built (needs /root/reference at build time)")
    gold = {c["id"]: c for c in json.load(open(GOLDEN))["cases"]}
    gname, mk, L, ratio = case
    spec = GRAPHS[gname]
    args = [SHIM, f"graph={spec['kind']}", f"n={spec['n']}", f"deg={spec['deg']}",
            f"gseed={spec['seed']}", f"weights={spec['weights'][0]}",
            f"low={spec['weights'][1]}", f"high={spec['weights'][2]}",
            f"alpha={spec['weights'][3]}", f"model={mk['kind']}",
            f"weighted={int(mk.get('weighted', True))}", f"a={mk.get('a', 2.0)}",
            f"b={mk.get('b', 0.5)}", f"gamma={mk.get('gamma', 0.2)}",
            "schema=" + ",".join(map(str, mk.get("schema", (0, 1, 2, 3, 4)))),
            f"L={L}", f"ratio={ratio}", "seed=7"]
    if spec["labels"]:
        args.append(f"labels={spec['labels'][0]},{spec['labels'][1]}")
    for mode in ("adaptive", "force-erjs", "force-ervs", "ervs-nojump"):
        out = str(tmp_path / mode)
        p = subprocess.run(args + [f"mode={mode}", f"out={out}"], capture_output=True, text=True,
                           timeout=300)
        assert p.returncode == 0, p.stderr
        stats = json.loads(p.stdout.strip().splitlines()[-1])
        paths = np.fromfile(out + ".paths", dtype=np.uint32).reshape(-1, L + 1)
        lengths = np.fromfile(out + ".lengths", dtype=np.uint32)
        c = gold[case_id(gname, mk, mode, L)]
        assert stats_core(stats) == c["stats"], mode
        assert digest(paths, lengths) == c["digest"], mode


def test_shim_rejects_unsupported_options(tmp_path):
    if not os.path.exists(SHIM):
        pytest.skip("oracle/_ref/shim_check not built")
    p = subprocess.run([SHIM, "mode=force-its", f"out={tmp_path}/x"], capture_output=True,
                       text=True, timeout=120)
    assert p.returncode == 2 and "not supported" in p.stderr


def test_shim_runs_dsl_models(ref, tmp_path):
    """A DslWalk handed to dynwalk::gpu::run_queries is compiled into the walk
    kernel by the shim (dsl_codegen.hpp + dw_model_compile) and equals the
    reference DslWalk on the Philox stream."""
    if not os.path.exists(SHIM):
        pytest.skip("oracle/_ref/shim_check not built")
    from tests.test_dsl import PROGRAMS
    g = ref.RefGraph.gen("ba", 400, 6, 13).synth("uniform", 1.0, 5.0, seed=113)
    g.synth("labels", 0, 3, seed=213)
    q = np.arange(400, dtype=np.uint32)
    for name in ("second_order", "label_degree"):
        src = tmp_path / f"{name}.wf"
        src.write_text(PROGRAMS[name])
        out = str(tmp_path / name)
        p = subprocess.run([SHIM, "graph=ba", "n=400", "deg=6", "gseed=13", "labels=0,3",
                            f"dsl={src}", "L=25", "ratio=1.4", "seed=7", "mode=adaptive",
                            f"out={out}"], capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        stats = json.loads(p.stdout.strip().splitlines()[-1])
        paths = np.fromfile(out + ".paths", dtype=np.uint32).reshape(-1, 26)
        ref.set_dsl_source(PROGRAMS[name])
        r = ref.ref_run(g, ref.Model("dsl"), q, mode="adaptive", walk_length=25, seed=7,
                        ratio=1.4, rng="philox", workers=2)
        assert stats_core(stats) == stats_core(r.stats), name
        assert np.array_equal(paths, r.paths), name


def test_shim_selection_ratio_sweep(ref):
    """dynwalk::gpu::selection_ratio_sweep (runtime.hpp:99-103 signature):
    per alpha, Pareto(alpha) properties drawn with the shared sweep seed
    (runtime.cpp:263) and an adaptive walk; every row's eRJS / eRVS split
    equals the reference samplers on the Philox stream."""
    if not os.path.exists(SHIM):
        pytest.skip("oracle/_ref/shim_check not built")
    alphas = (0.5, 1.0, 2.0, 4.0)
    p = subprocess.run([SHIM, "graph=ba", "n=300", "deg=5", "gseed=11", "L=20", "ratio=1.2",
                        "seed=7", "model=node2vec", "sweep=" + ",".join(map(str, alphas))],
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    rows = json.loads(p.stdout.strip().splitlines()[-1])
    assert [r["alpha"] for r in rows] == list(alphas)
    q = np.arange(300, dtype=np.uint32)
    sweep_seed = ref.derive_seed(7, 0x7377656570)
    for row, alpha in zip(rows, alphas):
        g = ref.RefGraph.gen("ba", 300, 5, 11).synth("uniform", 1.0, 5.0, seed=111)
        g.synth("pareto", alpha=alpha, seed=sweep_seed)
        r = ref.ref_run(g, ref.Model("node2vec", a=2.0, b=0.5), q, mode="adaptive",
                        walk_length=20, seed=7, ratio=1.2, rng="philox", workers=2)
        assert row["erjs_steps"] == r.stats["select_erjs"], alpha
        assert row["ervs_steps"] == r.stats["select_ervs"], alpha
        total = row["erjs_steps"] + row["ervs_steps"]
        assert total and abs(row["pct_erjs"] - 100.0 * row["erjs_steps"] / total) < 1e-3
    # the rows differ: the shape changes the selection split
    assert len({r["erjs_steps"] for r in rows}) > 1


def test_shim_run_queries_write_paths(tmp_path):
    """dynwalk::gpu::run_queries_write_paths writes the same bytes as the
    reference's write_paths over gpu::run_queries paths (runtime.cpp:280-291)."""
    if not os.path.exists(SHIM):
        pytest.skip("oracle/_ref/shim_check not built")
    out = str(tmp_path / "walks.txt")
    for mk in ("node2vec", "metapath"):
        extra = ["labels=0,3", "schema=0,1,2,3"] if mk == "metapath" else []
        p = subprocess.run([SHIM, "graph=ba", "n=500", "deg=6", "gseed=5", "L=15", "ratio=1.2",
                            "seed=9", f"model={mk}", f"write={out}"] + extra,
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        st = json.loads(p.stdout.strip().splitlines()[-1])
        assert st["steps"] == st["steps_rq"] > 0
        a, b = open(out, "rb").read(), open(out + ".ref", "rb").read()
        assert a == b and a.count(b"\n") == 500, mk
