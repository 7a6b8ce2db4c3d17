"""Per-source-line instruction and stall totals for one kernel of an ncu report.

    python tools/ncu_lines.py <rep> <cubin> <mangled kernel name> [top]
Maps the SASS page of the report (kernel-relative addresses) to source lines
with nvdisasm -g on the same cubin (the build must use -lineinfo).
"""
import collections
import csv
import io
import re
import subprocess
import sys


def addr_map(cubin, kernel):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    lines = dis.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kernel + ":"))
    cur, m = None, {}
    for l in lines[start + 1:]:
        if l.startswith(".text.") and l.endswith(":"):
            break
        mm = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if mm:
            cur = (mm.group(1).split("/")[-1], int(mm.group(2)))
            continue
        ma = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if ma and cur:
            m[int(ma.group(1), 16)] = cur
    return m


def main():
    rep, cubin, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    m = addr_map(cubin, kernel)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    base = min(int(r[ix["Address"]], 16) for r in data)

    def num(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    for r in data:
        a = int(r[ix["Address"]], 16) - base
        key = m.get(a, ("?", 0))
        v = agg[key]
        v[0] += num(r[ix["Instructions Executed"]])
        v[1] += num(r[ix["Thread Instructions Executed"]])
        v[2] += num(r[ix["Warp Stall Sampling (All Samples)"]])
        v[3] += num(r[ix["stall_no_inst"]])
        v[4] += num(r[ix["stall_wait"]])
        v[5] += num(r[ix["stall_long_sb"]])
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[2] for v in agg.values()) or 1
    src = {}
    for key in agg:
        if key[0] not in src:
            try:
                src[key[0]] = open(subprocess.run(["bash", "-c", f"ls paper_2512_00705_b200/csrc/{key[0]} 2>/dev/null"], capture_output=True, text=True).stdout.strip()).read().splitlines()
            except Exception:
                src[key[0]] = []
    order = 0
    if len(sys.argv) > 5:
        order = {"inst": 0, "samp": 2, "wait": 4, "lsb": 5}[sys.argv[5]]
    print(f"{'file:line':22s} {'inst%':>6s} {'simt':>5s} {'samp%':>6s} {'noinst%':>7s} {'wait%':>6s} {'lsb%':>6s}  source")
    for key, v in sorted(agg.items(), key=lambda kv: -kv[1][order])[:top]:
        s = src.get(key[0], [])
        text = s[key[1] - 1].strip()[:60] if 0 < key[1] <= len(s) else ""
        print(f"{key[0] + ':' + str(key[1]):22s} {100 * v[0] / ti:6.2f} {v[1] / max(v[0], 1):5.1f} "
              f"{100 * v[2] / ts:6.2f} {100 * v[3] / ts:7.2f} {100 * v[4] / ts:6.2f} {100 * v[5] / ts:6.2f}  {text}")


if __name__ == "__main__":
    main()
