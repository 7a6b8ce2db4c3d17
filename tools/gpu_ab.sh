#!/bin/bash
# A/B runs of the headline bench on one box: each argument is "name:ENV=V,ENV2=V2"
# (runtime switches read by the library).  Results -> gpurun_out/<tag>/ab.txt
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for rep in 1 2; do
for cfg in "$@"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $(echo $envs | tr ',' ' ') timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 2 --ratio 1.6 > $OUT/ab.json 2> $OUT/ab.err
  python - "$name" $OUT/ab.json <<'PY' | tee -a $OUT/ab.txt
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:12s} {d['value']:.4g} frac={d['roofline']['frac']:.3f} kms={d['roofline']['kernel_ms_per_launch']:.1f}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
done
