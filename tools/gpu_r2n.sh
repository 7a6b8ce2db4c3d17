#!/bin/bash
# A/B: weights-valid-by-construction skip against the base build on one box.
TAG=${1:-r2n}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in base posw base posw; do
  export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/$v/libdynwalk_b200.so
  timeout 900 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 8 > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  python -c "import json;d=json.load(open('$OUT/bench_$v.json'));print('$v',d['value'],d['roofline']['frac'],d['roofline']['kernel_ms_per_launch'])"
done
