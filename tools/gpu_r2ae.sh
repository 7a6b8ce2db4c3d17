#!/bin/bash
# config 5: current vs the first direct build (padded kernel with global query atomics); config 3 batch count
TAG=${1:-r2ae}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in cur r2x cur r2x; do
  if [ $v = cur ]; then unset DYNWALK_B200_LIB; else export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/$v/libdynwalk_b200.so; fi
  timeout 900 python bench.py --config 5 --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > $OUT/c5_$v.json 2> $OUT/c5_$v.err
  python -c "import json;d=json.load(open('$OUT/c5_$v.json'));print('c5 $v',d['value'],d['e2e']['value'])"
done
unset DYNWALK_B200_LIB
for div in 4 8 16; do
  DW_BATCH_DIV=$div timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/c3_div$div.json 2> $OUT/c3_div$div.err
  python -c "import json;d=json.load(open('$OUT/c3_div$div.json'));print('c3 div$div',d['value'],d['e2e']['value'],d['e2e']['ms_per_step'])"
done
