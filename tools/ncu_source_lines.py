"""Per-source-line instruction and stall totals from an ncu report (no GPU needed).

    python tools/ncu_source_lines.py <report.ncu-rep> [top=40] [walker_steps]

Reads `ncu -i --page source --print-source cuda,sass --csv` (needs -lineinfo and
--import-source on at capture) and sums, per CUDA source line, the warp
instructions executed, the thread instructions (-> active lanes per
instruction) and the warp-stall samples of the SASS that line produced.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    steps = float(sys.argv[3]) if len(sys.argv) > 3 else 590664320.0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
    fname, cur, hdr = "?", None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = {k: i for i, k in enumerate(r)}
            # the second "Source" column is the SASS text
            continue
        if r[0] == "Function Name" or hdr is None:
            continue
        if r[0]:  # a CUDA source line
            cur = (fname, int(r[0]))
            agg[cur][3] = r[1].strip()[:90]
            continue
        if cur is None:
            continue
        try:
            inst = float(r[hdr["Instructions Executed"]] or 0)
            thr = float(r[hdr["Thread Instructions Executed"]] or 0)
            smp = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError):
            continue
        a = agg[cur]
        a[0] += inst
        a[1] += thr
        a[2] += smp
    tot_i = sum(a[0] for a in agg.values()) or 1
    tot_s = sum(a[2] for a in agg.values()) or 1
    print(f"total warp instructions {tot_i:.4g} ({tot_i / steps:.1f}/step), "
          f"lanes/instr {sum(a[1] for a in agg.values()) / tot_i:.2f}")
    print(f"{'file:line':28s} {'inst%':>6s} {'/step':>6s} {'lanes':>5s} {'stall%':>6s}  source")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        if a[0] == 0:
            break
        print(f"{k[0] + ':' + str(k[1]):28s} {100 * a[0] / tot_i:6.2f} {a[0] / steps:6.2f} "
              f"{a[1] / a[0]:5.1f} {100 * a[2] / tot_s:6.2f}  {a[3]}")


if __name__ == "__main__":
    main()


def regions(rep, spans, steps=590664320.0):
    """Sum the per-line totals over named [lo, hi] line spans of one file."""
    import re  # noqa: F401
