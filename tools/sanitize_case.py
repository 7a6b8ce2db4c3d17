"""Small walks for compute-sanitizer runs (memcheck / racecheck on the walk kernel)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_00705_b200 as dw  # noqa: E402

dg = dw.DeviceGraph.rmat(10, 16, seed=3, weights="uniform", weight_seed=4, labels=(0, 3))
q = np.arange(1 << 10, dtype=np.uint32)
for kind, kw in (("node2vec", dict(a=0.5, b=2.0)), ("metapath", dict(schema=(0, 1, 2, 3) * 5)),
                 ("pr2", dict(gamma=0.2))):
    for mode in ("adaptive", "force-erjs", "force-ervs"):
        try:
            r = dw.run_queries(dg, dw.Model(kind, **kw), q,
                               dw.RunOptions(mode=mode, walk_length=20, seed=7, edge_cost_ratio=2.2))
            print(kind, mode, "ok", r.stats["steps"])
        except dw.DynwalkError as e:
            print(kind, mode, "ERROR", e)
