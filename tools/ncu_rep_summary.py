"""Key counters + stall breakdown from an ncu --set full report (no GPU needed).

    python tools/ncu_rep_summary.py gpurun_out/<tag>/walk_lib.ncu-rep [walker_steps]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__sectors_read.sum", "lts__t_requests_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
        "smsp__inst_executed_op_ldgsts.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_miss.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def main():
    d = raw(sys.argv[1])
    steps = float(sys.argv[2]) if len(sys.argv) > 2 else 590664320.0
    for k in KEYS:
        if k in d:
            print(f"{k:70s} {d[k][0]:>22s} {d[k][1]}")
    def f(k):
        return float(d[k][0].replace(",", ""))
    t = f("gpu__time_duration.sum") * (1e-3 if d["gpu__time_duration.sum"][1] == "ms" else 1e-9 if d["gpu__time_duration.sum"][1] == "ns" else 1e-6)
    print(f"walker-steps/s under ncu: {steps / t:.3e}")
    print(f"L2 read requests per step: {f('lts__t_requests_srcunit_tex_op_read.sum') / steps:.2f}")
    print(f"DRAM sectors per step:     {f('dram__sectors_read.sum') / steps:.2f}")
    print(f"warp instructions per step: {f('smsp__inst_executed.sum') / steps:.1f}")
    st = {k: f(k) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
    tot = sum(st.values()) or 1
    print("stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.1f}%"
                               for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]))


if __name__ == "__main__":
    main()
