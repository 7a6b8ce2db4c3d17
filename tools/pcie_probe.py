"""Pinned host <-> device copy bandwidth on this box (one stream, 1 GB)."""
import json
import time

import torch


def main():
    n = 1 << 30
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    out = {}
    for name, fn in (("d2h", lambda: h.copy_(d, non_blocking=True)),
                     ("h2d", lambda: d.copy_(h, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t = []
        for _ in range(5):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            t.append(time.perf_counter() - t0)
        out[name + "_gbs"] = n / min(t) / 1e9
    # both directions at once on two streams
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
    torch.cuda.synchronize()
    out["bidir_gbs_each"] = n / (time.perf_counter() - t0) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
