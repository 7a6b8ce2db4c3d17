"""Summarise an ncu --set full capture of the walk kernel into JSON.

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep profiles/<name>.json \
        [--scale 24] [--alg-bytes N] [--note "..."]

Reads `ncu -i <rep> --page raw --csv` (no GPU needed) and keeps the counters the
roofline and DESIGN.md cite: duration, DRAM bytes, L1/L2 hit rates, occupancy,
registers, and the warp-stall breakdown.
"""
import argparse
import csv
import io
import json
import subprocess

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__sectors_read.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_read.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "local_load", "local_store",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--alg-bytes", type=float, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None,
           "scale": a.scale, "note": a.note, "metrics": {}, "stalls_pct": {}}
    for h, u, v in zip(hdr, units, vals):
        if any(h.startswith(k) for k in KEEP):
            out["metrics"][h] = {"value": v, "unit": u}
        if h.startswith("smsp__average_warp_latency_issue_stalled") or (
                h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")):
            try:
                out["stalls_pct"][h] = float(v)
            except ValueError:
                pass

    def num(name, scale=1.0):
        m = out["metrics"].get(name)
        if not m:
            return None
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
                "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(m["unit"], 1)
        return float(m["value"].replace(",", "")) * mult * scale

    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    dur = num("gpu__time_duration.sum")
    out["dram_bytes_per_launch"] = (rd or 0) + (wr or 0)
    out["duration_s"] = dur
    if dur:
        out["dram_gbs"] = out["dram_bytes_per_launch"] / dur / 1e9
    if a.alg_bytes:
        out["algorithmic_bytes_per_launch"] = a.alg_bytes
        out["traffic_over_algorithmic"] = out["dram_bytes_per_launch"] / a.alg_bytes
    # top stall reasons (pc sampling), normalised to percent of samples
    samp = {k: v for k, v in out["stalls_pct"].items() if k.startswith("smsp__pcsamp")}
    tot = sum(samp.values())
    if tot:
        out["top_stalls"] = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""),
                                     round(100 * v / tot, 1)) for k, v in samp.items()),
                                   key=lambda x: -x[1])[:8]
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in out if k not in ("metrics", "stalls_pct")}, indent=1))


if __name__ == "__main__":
    main()
