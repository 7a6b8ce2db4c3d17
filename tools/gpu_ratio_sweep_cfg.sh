#!/bin/bash
# Walk throughput of one BASELINE config as a function of the cost-model ratio.
#   bash tools/gpu_ratio_sweep_cfg.sh <tag> <config> <ratio>...
TAG=$1; CFG=$2; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in "$@"; do
  timeout 600 python bench.py --config $CFG --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 2 --ratio $r > $OUT/c${CFG}_r$r.json 2>> $OUT/err.txt
  python - "$r" $OUT/c${CFG}_r$r.json <<'PY' | tee -a $OUT/sweep.txt
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
s = d["stats"]
print(f"ratio={sys.argv[1]:5s} {d['value']:.4g} frac={d['roofline']['frac']:.3f} erjs={s['select_erjs']} ervs={s['select_ervs']} trials/step={s['trials']/s['steps']:.2f}")
PY
done
