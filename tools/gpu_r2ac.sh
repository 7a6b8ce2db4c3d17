#!/bin/bash
# direct-run walk: current flat kernel vs the first direct build (4fb1f42), same box
TAG=${1:-r2ac}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export DW_VERBOSE=1
for v in cur r2x cur r2x cur r2x; do
  if [ $v = cur ]; then unset DYNWALK_B200_LIB; else export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/$v/libdynwalk_b200.so; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline > $OUT/s24_$v.json 2> $OUT/s24_$v.err
  python -c "import json;d=json.load(open('$OUT/s24_$v.json'));print('$v',d['value'],d['e2e']['value'],round(d['e2e']['ms_per_step'],2))"
  grep 'dynwalk direct' $OUT/s24_$v.err | tail -1
done
