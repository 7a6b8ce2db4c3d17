#!/bin/bash
# full GPU suite + configs 1, 5 and 4 on the direct compact build
TAG=${1:-r2v}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 python -m pytest tests/ -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu.log
export DW_VERBOSE=1
for c in 1 5; do
  timeout 1200 python bench.py --config $c > $OUT/c$c.json 2> $OUT/c$c.err; echo "c$c rc=$?"
  python -c "import json;d=json.load(open('$OUT/c$c.json'));print('c$c',d['value'],d['e2e'],d['ms_per_step'])"
  grep 'dynwalk direct' $OUT/c$c.err | tail -2
done
