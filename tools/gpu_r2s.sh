#!/bin/bash
# direct compact engine: parity tests, then base/new A/B of the s24 bench (value + e2e)
TAG=${1:-r2s}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "compact or direct" > $OUT/pytest.log 2>&1
tail -3 $OUT/pytest.log
for v in base new base new; do
  if [ $v = base ]; then export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/base/libdynwalk_b200.so; unset DW_VERBOSE; else unset DYNWALK_B200_LIB; export DW_VERBOSE=1; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/s24_$v.json 2> $OUT/s24_$v.err
  python -c "import json;d=json.load(open('$OUT/s24_$v.json'));print('$v',d['value'],d['e2e']['value'],d['e2e']['ms_per_step'],d['ms_per_step'])"
  grep 'dynwalk direct' $OUT/s24_$v.err | tail -2
done
