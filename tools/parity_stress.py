"""Bit-exact parity at larger scale than the test suite: the device-generated
R-MAT graph (the bench's generator) against the oracle's copy of it, every
model and sampler mode, a sample of walkers at walk length 80.

    python tools/parity_stress.py [scale] [walkers] [mode,mode,...] [model,model,...]

Prints one JSON line per (model, mode) with the walker-steps compared and
whether paths, lengths and counters were identical.  TEST INFRASTRUCTURE:
the oracle is the checker here, as in tests/.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle  # noqa: E402
import paper_2512_00705_b200 as dw  # noqa: E402
from tests.golden.make_golden import stats_core  # noqa: E402

MODELS = [dict(kind="node2vec", a=0.5, b=2.0), dict(kind="node2vec", a=2.0, b=0.5),
          dict(kind="node2vec", a=1.3, b=0.7), dict(kind="pr2", gamma=0.15),
          dict(kind="static"), dict(kind="metapath", schema=(0, 1, 2, 3) * 20)]
MODES = ("adaptive", "force-erjs", "force-ervs", "ervs-nojump")


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 18
    nw = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    modes = sys.argv[3].split(",") if len(sys.argv) > 3 else MODES
    kinds = sys.argv[4].split(",") if len(sys.argv) > 4 else None
    # labels only when MetaPath runs (a labelled graph has no compact records)
    labels = (0, 3) if kinds is None or "metapath" in kinds else None
    dg = dw.DeviceGraph.rmat(scale, 16, seed=1, weights="uniform", weight_seed=2, labels=labels,
                             label_seed=3)
    a = dg.download()
    og = oracle.Graph.from_csr(a["row"], a["col"], a["prop"], a["label"])
    nv = len(a["row"]) - 1
    q = np.random.default_rng(5).integers(0, nv, nw).astype(np.uint32)
    threads = os.cpu_count() or 4
    ok_all = True
    for mk in MODELS:
        if kinds and mk["kind"] not in kinds:
            continue
        for mode in modes:
            opts = dw.RunOptions(mode=mode, walk_length=80, seed=11, edge_cost_ratio=1.6)
            r = dw.run_queries(dg, dw.Model(**mk), q, opts)
            o = oracle.run(og, oracle.Model(**mk), q, mode=mode, walk_length=80, seed=11,
                           ratio=1.6, rng="philox", threads=threads)
            same = (stats_core(r.stats) == stats_core(o.stats)
                    and np.array_equal(r.lengths, o.lengths) and np.array_equal(r.paths, o.paths))
            ok_all &= same
            print(json.dumps({"scale": scale, "walkers": nw, "model": mk["kind"],
                              "params": {k: v for k, v in mk.items() if k in ("a", "b", "gamma")},
                              "mode": mode, "walker_steps": int(r.stats["steps"]),
                              "bit_exact": bool(same)}), flush=True)
    print(json.dumps({"all_bit_exact": bool(ok_all)}))


if __name__ == "__main__":
    main()
