"""Is a walk launch bound by its slowest walker?  Kernel time for all walkers
vs a 1/4 sample of the same queries (config 4 by default: PR2, Pareto weights).

    python tools/tail_probe.py [scale] [config]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2512_00705_b200 as dw  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    cfg = bench.CONFIGS[int(sys.argv[2]) if len(sys.argv) > 2 else 4]
    g = dw.DeviceGraph.rmat(scale, 16, seed=bench.TOPO_SEED, weights=cfg["weights"], low=1.0,
                            high=5.0, alpha=1.0, weight_seed=bench.WEIGHT_SEED,
                            labels=cfg["labels"], label_seed=bench.LABEL_SEED)
    nv = g.info()["num_vertices"]
    m = dw.Model(cfg["model"], **bench.model_kw(cfg))
    ratio = dw.profile_edge_cost_ratio(g, m, seed=bench.PROFILE_SEED)
    opts = dw.RunOptions(walk_length=80, seed=bench.WALK_SEED, edge_cost_ratio=ratio)
    out = {"scale": scale, "model": cfg["model"], "ratio": ratio}
    for name, q in (("all", np.arange(nv, dtype=np.uint32)),
                    ("quarter", np.arange(0, nv, 4, dtype=np.uint32))):
        os.environ["DW_BATCH"] = str(len(q))  # one launch
        r = dw.run_queries(g, m, q, opts, keep_paths=False)
        out[name] = {"walkers": len(q), "kernel_ms": r.stats["kernel_ms"],
                     "steps": r.stats["steps"], "trials": r.stats["trials"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
