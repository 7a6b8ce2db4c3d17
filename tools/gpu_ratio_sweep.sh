#!/bin/bash
# Walk throughput of the headline config as a function of the cost-model ratio
# (the calibrated value is what bench.py uses by default).
TAG=${1:-ratio}; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in "$@"; do
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 2 --ratio $r > $OUT/r$r.json 2>> $OUT/err.txt
  python - "$r" $OUT/r$r.json <<'PY' | tee -a $OUT/sweep.txt
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
s = d["stats"]
print(f"ratio={sys.argv[1]:5s} {d['value']:.4g} frac={d['roofline']['frac']:.3f} erjs={s['select_erjs']} ervs={s['select_ervs']} trials/step={s['trials']/s['steps']:.2f}")
PY
done
