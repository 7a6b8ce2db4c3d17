#!/bin/bash
# Config 4 (PR2, Pareto, s20) across library variants: name:libpath ...
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
for cfg in "$@"; do
  name=${cfg%%:*}; lib=${cfg#*:}
  DYNWALK_B200_LIB=$lib timeout 900 python bench.py --config 4 --scale 20 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --ratio 2.2 > $OUT/$name.json 2> $OUT/$name.err
  python - "$name" $OUT/$name.json <<'PY' | tee -a $OUT/ab.txt
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"{sys.argv[1]:10s} {d['value']:.4g} e2e={d['e2e']['value']:.4g} kms={d['roofline']['kernel_ms_per_launch']:.0f}")
PY
done
