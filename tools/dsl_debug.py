"""Debug helper: one DSL program, every mode, first differing walker."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as ref
import paper_2512_00705_b200 as dw
from tests.test_dsl import PROGRAMS
name = sys.argv[1]
og = ref.Graph.rmat(11, 16, 41).synth_philox("uniform", 1.0, 5.0, seed=42)
og.synth_philox("labels", 0, 3, seed=43)
a = og.arrays()
dg = dw.DeviceGraph.from_csr(a["row"], a["col"], a["prop"], a["label"])
rg = ref.RefGraph.from_csr(a["row"], a["col"], a["prop"], a["label"])
src, ms, fl = ref.dsl_codegen(PROGRAMS[name])
print(src)
cm = dw.CustomModel(src, ms, fl)
q = np.arange(og.nv, dtype=np.uint32)
ref.set_dsl_source(PROGRAMS[name])
for mode in ("force-erjs", "force-ervs", "adaptive"):
    r_dev = dw.run_queries(dg, dw.Model("custom", custom=cm), q, dw.RunOptions(mode=mode, walk_length=20, seed=11, edge_cost_ratio=1.3))
    r_ref = ref.ref_run(rg, ref.Model("dsl"), q, mode=mode, walk_length=20, seed=11, ratio=1.3, rng="philox", workers=4)
    diff = {k: (r_dev.stats[k], r_ref.stats[k]) for k in ("steps", "select_erjs", "select_ervs", "trials", "rng_draws") if r_dev.stats[k] != r_ref.stats[k]}
    bad = np.nonzero((r_dev.paths != r_ref.paths).any(axis=1))[0]
    print(mode, "stat diffs", diff, "walkers differing", len(bad))
    if len(bad):
        i = bad[0]
        print(" walker", i, "dev", r_dev.paths[i, :8], "ref", r_ref.paths[i, :8])
        j = int(np.argmax(r_dev.paths[i] != r_ref.paths[i]))
        v = int(r_dev.paths[i, j - 1]); p = int(r_dev.paths[i, j - 2]) if j >= 2 else -1
        lo, hi = int(a["row"][v]), int(a["row"][v + 1])
        labs = a["label"][lo:hi]
        print(" step", j, "at node", v, "prev", p, "deg", hi - lo, "hmax", a["nmax"][v], "hsum", a["nsum"][v], "lmax", labs.max(), "lsum", float(labs.astype(np.float64).sum()))
