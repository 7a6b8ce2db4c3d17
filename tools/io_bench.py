"""Throughput of the f3/f4 paths around the walk (1 B200):
  * dw_graph_load_dwg1 vs the reference's load_binary (host, oracle/_ref) on
    the same DWG1 file of the R-MAT s22 graph;
  * dw_run_write_paths (device text formatting, streamed) vs dw_run_compact +
    host formatting, node2vec s22, one walker per vertex.
Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: the reference's load_binary)
import paper_2512_00705_b200 as dw  # noqa: E402

scale = int(os.environ.get("IO_SCALE", "22"))
tmp = os.environ.get("IO_DIR", "/tmp")
out = {"scale": scale}
dg = dw.DeviceGraph.rmat(scale, 16, seed=1, weights="uniform", weight_seed=2)
a = dg.download()
path = os.path.join(tmp, f"rmat{scale}.dwg1")
with open(path, "wb") as f:
    f.write(b"DWG1" + (1).to_bytes(4, "little") + b"\0")
    for arr in (a["row"], a["col"], a["prop"]):
        f.write(len(arr).to_bytes(8, "little"))
        f.write(arr.tobytes())
size = os.path.getsize(path)
out["dwg1_bytes"] = size
del dg
t0 = time.perf_counter()
g2 = dw.DeviceGraph.load_dwg1(path)
out["load_dwg1_s"] = time.perf_counter() - t0
b = g2.download()
out["load_dwg1_identical"] = all(np.array_equal(a[k], b[k]) for k in ("row", "col", "prop", "nmax", "nsum"))
if oracle.ref_available():
    t0 = time.perf_counter()
    rg = oracle.RefGraph.load_binary(path)
    out["ref_load_binary_s"] = time.perf_counter() - t0
    del rg
nv = len(a["row"]) - 1
q = np.arange(nv, dtype=np.uint32)
model = dw.Model(a=0.5, b=2.0)
opts = dw.RunOptions(mode="adaptive", walk_length=80, seed=7, edge_cost_ratio=2.2)
txt = os.path.join(tmp, "paths.txt")
dw.run_write_paths(g2, model, q[:1000], opts, txt)  # warm
t0 = time.perf_counter()
st = dw.run_write_paths(g2, model, q, opts, txt)
out["write_paths_s"] = time.perf_counter() - t0
out["text_bytes"] = os.path.getsize(txt)
out["walker_steps"] = st["steps"] - st["dead_ends"]
out["write_paths_walker_steps_per_s"] = out["walker_steps"] / out["write_paths_s"]
t0 = time.perf_counter()
offs, flat, st2 = dw.run_queries_compact(g2, model, q, opts)
out["compact_s"] = time.perf_counter() - t0
os.remove(txt)
os.remove(path)
print(json.dumps(out), flush=True)
