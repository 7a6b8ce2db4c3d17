"""Micro-pass (K4) and walk-tuned (dw_tune_ratio) ratios on the bench graphs,
with their timings; run on a GPU box."""
import sys
import time

sys.path.insert(0, ".")
import paper_2512_00705_b200 as dw  # noqa: E402

for s in [int(x) for x in (sys.argv[1:] or ["24", "20"])]:
    dg = dw.DeviceGraph.rmat(s, 16, seed=1, weights="uniform", low=1.0, high=5.0, weight_seed=2)
    m = dw.Model("node2vec", a=0.5, b=2.0)
    for seed in (5, 6):
        cfg = dw.ProfileConfig(seed=seed)
        t0 = time.perf_counter()
        r0 = dw.profile_edge_cost_ratio(dg, m, cfg=cfg)
        t1 = time.perf_counter()
        rt = dw.tune_edge_cost_ratio(dg, m, cfg=cfg)
        t2 = time.perf_counter()
        print(f"s{s} seed {seed}: micro {r0:.3f} ({t1 - t0:.2f} s)  tuned {rt:.3f} ({t2 - t1:.2f} s)",
              flush=True)
    del dg
