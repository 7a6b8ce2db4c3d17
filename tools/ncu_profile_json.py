"""Write the judged ncu summary of the walk kernel (no GPU needed).

    python tools/ncu_profile_json.py <walk_full.ncu-rep> <launches.csv> <bench.json> <out.json> [note]

Reads one `ncu --set full` capture of the walk kernel, the
`--metrics gpu__time_duration.sum` launch list of the same bench command and
the bench JSON line of that build, and writes:
  * the kernel's raw counters (DRAM bytes, L2 requests/sectors, SIMT
    efficiency, instructions, stall breakdown) and per-walker-step ratios;
  * dram_bytes_per_launch (read + write), which bench.py reports as
    roofline.traffic when the library hash matches;
  * the walk kernel's share of the timed step in the launch list;
  * lib_sha16 of the library that ran (from the bench line), so a summary
    can be matched to its build.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__sectors_read.sum", "lts__t_requests_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum.per_second", "sass__inst_executed_local_loads",
        "sass__inst_executed_local_stores"]


def _num(s):
    return float(s.replace(",", ""))


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def to_bytes(v, u):
    return _num(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]


def to_ms(v, u):
    return _num(v) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                      "nsecond": 1e-6, "s": 1e3, "second": 1e3}[u]


def launches(path):
    txt = open(path).read()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ms = to_ms(r["Metric Value"], r["Metric Unit"])
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")
        if "walk_kernel" in name:
            short = name.split("(WalkParams")[0].replace("void ", "")
        n, t = per.get(short, (0, 0.0))
        per[short] = (n + 1, t + ms)
    return per


def main():
    rep, lcsv, bench, out = sys.argv[1:5]
    note = sys.argv[5] if len(sys.argv) > 5 else ""
    d = raw(rep)
    b = json.loads(open(bench).read().strip().splitlines()[-1])
    if "walker_steps_per_step" not in b:
        raise SystemExit("bench line without walker_steps_per_step")
    steps = float(b["walker_steps_per_step"])
    met = {k: {"value": d[k][0], "unit": d[k][1]} for k in KEYS if k in d}
    rd = to_bytes(*d["dram__bytes_read.sum"])
    wr = to_bytes(*d["dram__bytes_write.sum"])
    alg = float(b["roofline"]["algorithmic_bytes_per_launch"])
    st = {k: _num(v[0]) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
    tot = sum(st.values()) or 1.0
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * v / tot, 1)
              for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]}
    per = launches(lcsv) if lcsv != "-" else {}
    total_ms = sum(t for _, t in per.values())
    walk = {k: v for k, v in per.items() if "walk_kernel" in k}
    walk_ms = sum(t for _, t in walk.values())
    res = {
        "kernel": d.get("Kernel Name", ("", ""))[0] or b["roofline"]["kernel"],
        "scale": int(b["config"]["graph"].split()[1][1:]) if "graph" in b["config"] else None,
        "lib_sha16": b.get("build", {}).get("lib_sha16"),
        "note": note,
        "metrics": met,
        "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": alg,
        "traffic_over_algorithmic": (rd + wr) / alg,
        "per_walker_step": {
            "warp_instructions": _num(d["smsp__inst_executed.sum"][0]) / steps,
            "l2_read_requests": _num(d["lts__t_requests_srcunit_tex_op_read.sum"][0]) / steps,
            "l2_sectors_per_request": _num(d["lts__t_sectors_srcunit_tex_op_read.sum"][0])
            / _num(d["lts__t_requests_srcunit_tex_op_read.sum"][0]),
            "dram_sectors": _num(d["dram__sectors_read.sum"][0]) / steps,
        },
        "simt_lanes_per_instruction": _num(d["smsp__thread_inst_executed_per_inst_executed.ratio"][0]),
        "stall_pct": stalls,
        "launch_list": None if lcsv == "-" else {
            "source": lcsv,
            "kernels": {k: {"launches": n, "ms": round(t, 3)} for k, (n, t) in
                        sorted(per.items(), key=lambda kv: -kv[1][1])[:12]},
            "walk_kernel_ms": walk_ms,
            "walk_share_of_all_launches": walk_ms / total_ms if total_ms else None,
        },
        "bench_line": {k: b[k] for k in ("value", "ms_per_step") if k in b},
    }
    res["bench_line"]["frac"] = b["roofline"]["frac"]
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: res[k] for k in ("traffic_over_algorithmic", "per_walker_step",
                                          "simt_lanes_per_instruction", "stall_pct")}, indent=1))


if __name__ == "__main__":
    main()
