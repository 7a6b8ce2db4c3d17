#!/bin/bash
# A/B of the bucket mask build against the committed base on one box.
TAG=${1:-r2m}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in base mask nomask base mask nomask; do
  case $v in
    base) export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/base/libdynwalk_b200.so ;;
    nomask) export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/nomask/libdynwalk_b200.so ;;
    *) unset DYNWALK_B200_LIB ;;
  esac
  timeout 900 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 8 > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  python -c "import json;d=json.load(open('$OUT/bench_$v.json'));print('$v',d['value'],d['roofline']['frac'],d['roofline']['kernel_ms_per_launch'])"
done
