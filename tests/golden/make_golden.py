"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference and oracle/_ref):
    python tests/golden/make_golden.py

* stats_walk.json  -- the reference CLI golden (proj/tests/golden/stats_walk.txt,
                      checked by proj/tests/test_cli.cpp:123-131) parsed to JSON,
                      with the CLI configuration that produces it.
* ref_walks.json   -- paths digests + RunStats of the reference's own sampler
                      templates (decide_sampler / sample_erjs / sample_ervs /
                      sample_ervs_nojump, oracle/ref_harness.cpp ref_run_philox)
                      under the Philox walker stream, and of the stock
                      run_queries (mt19937), on graphs built by the reference
                      generators.  The GPU tests rebuild the same graphs with the
                      oracle (bit-identical generators, tests/test_oracle.py) and
                      must reproduce these digests exactly.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

REF_GOLDEN = "/root/reference/proj/tests/golden/stats_walk.txt"

# graph recipes shared with tests/test_gpu_parity.py
GRAPHS = {
    "ba300": dict(kind="ba", n=300, deg=5, seed=11, weights=("uniform", 1.0, 5.0, 0.0), labels=None),
    "ba300_labels": dict(kind="ba", n=300, deg=6, seed=12, weights=("uniform", 1.0, 5.0, 0.0),
                         labels=(0, 3)),
    "ba400_pareto": dict(kind="ba", n=400, deg=8, seed=13, weights=("pareto", 0.0, 0.0, 1.0),
                         labels=None),
    "uni200": dict(kind="uniform", n=200, deg=40, seed=14, weights=("uniform", 1.0, 5.0, 0.0),
                   labels=None),
}

CASES = [
    # (graph, model kwargs, walk_length, ratio)
    ("ba300", dict(kind="node2vec", a=2.0, b=0.5), 20, 1.2),
    ("ba300", dict(kind="node2vec", a=0.5, b=2.0), 20, 1.2),
    ("ba300", dict(kind="node2vec", a=0.5, b=2.0, weighted=False), 20, 1.2),
    ("ba300", dict(kind="static"), 20, 1.0),
    ("ba300_labels", dict(kind="metapath", schema=(0, 1, 2, 3) * 5), 20, 1.2),
    ("ba400_pareto", dict(kind="pr2", gamma=0.15), 20, 1.3),
    ("uni200", dict(kind="node2vec", a=0.5, b=2.0), 30, 3.0),
]
MODES = ("adaptive", "force-erjs", "force-ervs", "ervs-nojump")


def build_oracle_graph(spec):
    g = (O.Graph.ba if spec["kind"] == "ba" else O.Graph.uniform)(spec["n"], spec["deg"],
                                                                  spec["seed"], True)
    kind, lo, hi, alpha = spec["weights"]
    g.synth(kind, lo, hi, alpha, seed=spec["seed"] + 100)
    if spec["labels"]:
        g.synth("labels", spec["labels"][0], spec["labels"][1], seed=spec["seed"] + 200)
    return g


def build_ref_graph(spec):
    g = O.RefGraph.gen(spec["kind"], spec["n"], spec["deg"], spec["seed"], True)
    kind, lo, hi, alpha = spec["weights"]
    g.synth(kind, lo, hi, alpha, seed=spec["seed"] + 100)
    if spec["labels"]:
        g.synth("labels", spec["labels"][0], spec["labels"][1], seed=spec["seed"] + 200)
    return g


def digest(paths: np.ndarray, lengths: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(paths, np.uint32).tobytes())
    h.update(np.ascontiguousarray(lengths, np.uint32).tobytes())
    return h.hexdigest()


def stats_core(st: dict) -> dict:
    keys = ("queries", "query_errors", "dead_ends", "steps", "select_ervs", "select_erjs",
            "trials", "weight_reads", "rng_draws", "erjs_fallbacks")
    out = {k: int(st[k]) for k in keys}
    out["selection_by_degree"] = [list(x) for x in st["selection_by_degree"]]
    return out


def case_id(gname, mk, mode, L):
    m = ",".join(f"{k}={v}" for k, v in sorted(mk.items()) if k != "schema")
    return f"{gname}|{m}|{mode}|L{L}"


def main():
    # 1. CLI golden
    vals = {}
    hist = []
    for line in open(REF_GOLDEN):
        line = line.strip()
        if line.startswith("deg_bucket="):
            parts = dict(p.split("=") for p in line.split())
            hist.append([int(parts["deg_bucket"].split("^")[1]), int(parts["ervs"]),
                         int(parts["erjs"])])
        elif "=" in line and not line.startswith("["):
            k, v = line.split("=", 1)
            vals[k] = v
    golden = {
        "source": "proj/tests/golden/stats_walk.txt (test_cli.cpp:123-131)",
        "cli": "dynwalk walk --gen ba:n=50,deg=4 --undirected --weights uniform:low=1,high=5 "
               "--model node2vec --seed 13 --steps 10 --workers 2 --edge-cost-ratio 4",
        "values": {k: v for k, v in vals.items() if k != "wall_ms"},
        "selection_histogram": hist,
    }
    json.dump(golden, open(os.path.join(HERE, "stats_walk.json"), "w"), indent=1)

    # 2. reference walks
    out = {"graphs": GRAPHS, "cases": []}
    for gname, mk, L, ratio in CASES:
        spec = GRAPHS[gname]
        rg = build_ref_graph(spec)
        og = build_oracle_graph(spec)
        a, b = rg.arrays(), og.arrays()
        for k in ("row", "col", "prop", "nmax", "nsum"):
            assert np.array_equal(a[k], b[k]), (gname, k)
        nv = len(a["row"]) - 1
        queries = np.arange(nv, dtype=np.uint32)
        model = O.Model(**mk)
        for mode in MODES:
            rr = O.ref_run(rg, model, queries, mode=mode, walk_length=L, seed=7, ratio=ratio,
                           rng="philox", workers=4)
            out["cases"].append({"id": case_id(gname, mk, mode, L), "graph": gname, "model": mk,
                                 "mode": mode, "walk_length": L, "ratio": ratio, "seed": 7,
                                 "rng": "philox", "digest": digest(rr.paths, rr.lengths),
                                 "stats": stats_core(rr.stats)})
        rr = O.ref_run(rg, model, queries, mode="adaptive", walk_length=L, seed=7, ratio=ratio,
                       rng="mt19937", workers=4)
        out["cases"].append({"id": case_id(gname, mk, "adaptive", L) + "|mt19937", "graph": gname,
                             "model": mk, "mode": "adaptive", "walk_length": L, "ratio": ratio,
                             "seed": 7, "rng": "mt19937", "digest": digest(rr.paths, rr.lengths),
                             "stats": stats_core(rr.stats)})
    json.dump(out, open(os.path.join(HERE, "ref_walks.json"), "w"), indent=0)
    print(f"wrote {len(out['cases'])} reference walk cases")


if __name__ == "__main__":
    main()
