#!/bin/bash
# A/B on one box: library variants x runtime switches, fixed ratio.
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
for rep in 1 2; do
for cfg in "$@"; do
  name=${cfg%%:*}; rest=${cfg#*:}; lib=${rest%%:*}; envs=${rest#*:}
  env DYNWALK_B200_LIB=$lib $(echo $envs | tr ',' ' ') timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 2 --ratio ${RATIO:-2.2} > $OUT/ab.json 2> $OUT/ab.err
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
