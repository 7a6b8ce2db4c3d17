#!/bin/bash
# direct compact engine: where the walk-time difference comes from
# (m1: chunk counts without release ordering, m2: no chunk accounting; measurement only)
TAG=${1:-r2t}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "compact or direct" > $OUT/pytest.log 2>&1
tail -3 $OUT/pytest.log
export DW_VERBOSE=1
for v in new m1 m2 base new m1 m2; do
  case $v in new) unset DYNWALK_B200_LIB;; *) export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/$v/libdynwalk_b200.so;; esac
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/s24_$v.json 2> $OUT/s24_$v.err
  python -c "import json;d=json.load(open('$OUT/s24_$v.json'));print('$v',d['value'],d['e2e']['value'],d['e2e']['ms_per_step'],d['ms_per_step'])"
  grep 'dynwalk direct' $OUT/s24_$v.err | tail -2
done
