"""Per-event costs of the walk kernel in forced modes, on a walker sample.

    python tools/calib_probe.py [scale] [walkers] [walk_length]

Prints kernel ms, trials and weight reads for force-erjs and force-ervs runs of
the headline model on the bench graph, and the ratio of the two per-event
costs (ms per eRJS trial / ms per eRVS weight read) -- what the cost model's
edge_cost_ratio is meant to capture -- next to dw_calibrate's value.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2512_00705_b200 as dw  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    nw = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
    L = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    cfg = bench.CONFIGS[2]
    g = dw.DeviceGraph.rmat(scale, 16, seed=bench.TOPO_SEED, weights="uniform", low=1.0,
                            high=5.0, alpha=1.0, weight_seed=bench.WEIGHT_SEED)
    nv = g.info()["num_vertices"]
    m = dw.Model("node2vec", a=cfg["a"], b=cfg["b"])
    rng = np.random.default_rng(3)
    q = rng.integers(0, nv, nw, dtype=np.uint32)
    out = {"scale": scale, "walkers": nw, "walk_length": L,
           "calibrated": dw.profile_edge_cost_ratio(g, m, seed=bench.PROFILE_SEED)}
    for mode in ("force-erjs", "force-ervs", "adaptive"):
        opts = dw.RunOptions(mode=mode, walk_length=L, seed=7, edge_cost_ratio=1.6)
        dw.run_queries(g, m, q, opts, keep_paths=False)  # warm
        best = None
        for _ in range(3):
            r = dw.run_queries(g, m, q, opts, keep_paths=False)
            if best is None or r.stats["kernel_ms"] < best["kernel_ms"]:
                best = r.stats
        out[mode] = {k: best[k] for k in ("kernel_ms", "steps", "trials", "weight_reads",
                                          "select_erjs", "select_ervs")}
    e, v = out["force-erjs"], out["force-ervs"]
    out["ms_per_trial"] = e["kernel_ms"] / max(e["trials"], 1)
    out["ms_per_read"] = v["kernel_ms"] / max(v["weight_reads"], 1)
    out["ratio_from_kernel"] = out["ms_per_trial"] / out["ms_per_read"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
