"""End-to-end (host buffers) vs device-resident walk time per batch size.

    python tools/e2e_probe.py [scale] [batch sizes...]

Runs the bench workload (config 2: node2vec, R-MAT, walk length 80) through
dw_run_device (inputs resident) and through dw_run_compact (pinned host
queries in, offsets + ids out) with the run engine's batch size forced by
DW_BATCH, so the cost of the H2D/D2H pipeline can be read off per batch size.
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2512_00705_b200 as dw  # noqa: E402


def main():
    import torch
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    sizes = [int(x) for x in sys.argv[2:]] or [0]
    cfg = bench.CONFIGS[2]
    dg = dw.DeviceGraph.rmat(scale, 16, seed=bench.TOPO_SEED, weights=cfg["weights"], low=1.0,
                             high=5.0, alpha=1.0, weight_seed=bench.WEIGHT_SEED,
                             labels=cfg["labels"], label_seed=bench.LABEL_SEED, devices=[0])
    n = dg.info()["num_vertices"]
    L = 80
    model = dw.Model(cfg["model"], **bench.model_kw(cfg))
    opts = dw.RunOptions(mode="adaptive", walk_length=L, seed=bench.WALK_SEED, edge_cost_ratio=2.2)
    lib = dw.load_library()
    mdesc, odesc = model.c(), opts.c()
    q = torch.arange(0, n, dtype=torch.int64, device="cuda").to(torch.int32)
    paths = torch.empty((n, L + 1), dtype=torch.int32, device="cuda")
    lengths = torch.empty(n, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def dev_step():
        rc = lib.dw_run_device(dg.h, 0, C.byref(mdesc), C.c_void_p(q.data_ptr()), n,
                               C.byref(odesc), C.c_void_p(paths.data_ptr()),
                               C.c_void_p(lengths.data_ptr()), C.c_void_p(stream.cuda_stream))
        assert rc == 0, lib.dw_last_error()
        st = dw.RunStatsC()
        assert lib.dw_run_device_sync(dg.h, 0, C.byref(st)) == 0
        return st

    for _ in range(2):
        st = dev_step()
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        st = dev_step()
        t.append(time.perf_counter() - t0)
    steps = int(st.steps)
    out = {"scale": scale, "walkers": n, "steps": steps,
           "device_ms": 1e3 * float(np.mean(t)), "kernel_ms": float(st.kernel_ms), "e2e": []}

    hq, ho, hf = C.c_void_p(), C.c_void_p(), C.c_void_p()
    cap = n * (L + 1)
    for buf, nb in ((hq, n * 4), (ho, (n + 1) * 8), (hf, cap * 4)):
        assert lib.dw_host_alloc(nb, C.byref(buf)) == 0
    np.ctypeslib.as_array(C.cast(hq, dw.u32p), (n,))[:] = np.arange(n, dtype=np.uint32)
    for bs in sizes:
        if bs:
            os.environ["DW_BATCH"] = str(bs)
        else:
            os.environ.pop("DW_BATCH", None)
        rs = dw.RunStatsC()

        def e2e():
            rc = lib.dw_run_compact(dg.h, C.byref(mdesc), C.cast(hq, dw.u32p), n, C.byref(odesc),
                                    C.cast(ho, dw.u64p), C.cast(hf, dw.u32p), cap, C.byref(rs))
            assert rc == 0, lib.dw_last_error()

        e2e()
        t = []
        for _ in range(3):
            t0 = time.perf_counter()
            e2e()
            t.append(time.perf_counter() - t0)
        ms = 1e3 * float(np.mean(t))
        out["e2e"].append({"batch": bs or "default", "ms": ms, "walker_steps_per_s": steps / ms * 1e3,
                           "kernel_ms_sum": float(rs.kernel_ms)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
