#!/bin/bash
TAG=${1:-r2q}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in base2 cold base2 cold; do
  export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/$v/libdynwalk_b200.so
  timeout 900 python bench.py --config 4 --scale 22 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/c4_$v.json 2> $OUT/c4_$v.err
  python -c "import json;d=json.load(open('$OUT/c4_$v.json'));print('$v',d['value'],d['roofline']['frac'])"
done
