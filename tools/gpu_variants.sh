#!/bin/bash
# Bench every built library variant (paper_2512_00705_b200/variants/*) on the
# headline config; one JSON line each into gpurun_out/<tag>/variants.txt.
TAG=${1:-var}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
ARGS=${*:-"--steps 3 --warmup 2"}
for lib in paper_2512_00705_b200/lib/libdynwalk_b200.so paper_2512_00705_b200/variants/*/libdynwalk_b200.so; do
  [ -f "$lib" ] || continue
  DYNWALK_B200_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 $ARGS > $OUT/v.json 2> $OUT/v.err
  python - "$lib" $OUT/v.json <<'PY' | tee -a $OUT/variants.txt
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], f"{d['value']:.4g}", f"frac={d['roofline']['frac']:.3f}", f"kms={d['roofline']['kernel_ms_per_launch']:.1f}", d['stats'])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
