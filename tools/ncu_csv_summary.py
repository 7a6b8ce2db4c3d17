"""Summarise an `ncu --metrics ... --csv` launch log: one line per kernel launch."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    recs = collections.OrderedDict()
    for r in rows[i + 1:]:
        if len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        rec = recs.setdefault(d["ID"], {"name": d["Kernel Name"]})
        try:
            rec[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            rec[d["Metric Name"]] = d["Metric Value"]
    return list(recs.values())


if __name__ == "__main__":
    for rec in load(sys.argv[1]):
        req = rec.get("lts__t_requests_srcunit_tex_op_read.sum", 0) or 1
        dr = rec.get("dram__sectors_read.sum", 0)
        t = rec.get("gpu__time_duration.sum", 0)
        print(f"{rec['name'][:44]:44s} t={t/1e3:9.1f}us l2req={req:.3e} "
              f"dram_sec/l2req={dr/req:5.2f} dramGB/s={dr*32/max(t,1):7.0f} "
              f"l2hit={rec.get('lts__t_sector_hit_rate.pct', 0):5.1f}")
