#!/bin/bash
# One BASELINE config across library variants at a fixed ratio:
#   bash tools/gpu_cfg_ab.sh <tag> <config> <ratio> name:libpath ...
TAG=$1; CFG=$2; R=$3; shift 3; OUT=gpurun_out/$TAG; mkdir -p $OUT
for rep in 1 2; do
for cfg in "$@"; do
  name=${cfg%%:*}; lib=${cfg#*:}
  DYNWALK_B200_LIB=$lib timeout 900 python bench.py --config $CFG --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline --ratio $R > $OUT/$name.json 2> $OUT/$name.err
  python - "$name" $OUT/$name.json <<'PY' | tee -a $OUT/ab.txt
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"{sys.argv[1]:10s} {d['value']:.4g} frac={d['roofline']['frac']:.3f} kms={d['roofline']['kernel_ms_per_launch']:.2f}")
PY
done
done
