#!/bin/bash
# configs 1 and 5 on the direct compact build (chunk floor, buffers freed for download)
TAG=${1:-r2w}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "compact or direct or dwg1" > $OUT/pytest.log 2>&1
tail -1 $OUT/pytest.log
export DW_VERBOSE=1
for c in 1 5; do
  timeout 1200 python bench.py --config $c > $OUT/c$c.json 2> $OUT/c$c.err; echo "c$c rc=$?"
  python -c "import json;d=json.load(open('$OUT/c$c.json'));print('c$c',d['value'],d['e2e'],d['ms_per_step'],d.get('cpu_baseline'))"
  grep 'dynwalk direct' $OUT/c$c.err | tail -2
done
