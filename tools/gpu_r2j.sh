#!/bin/bash
# Round-2 session j: triangle work limit and run-engine batch count.
TAG=${1:-r2j}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for tw in 1024 4096 16384; do
  DW_TRI_WORK=$tw timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 > $OUT/tw$tw.json 2> $OUT/tw$tw.err
  python -c "import json;d=json.load(open('$OUT/tw$tw.json'));print('tri_work $tw',d['value'],d['roofline']['frac'],d['e2e']['value'],d['setup_s']['graph_build'])"
done
for bd in 3 6 8; do
  DW_BATCH_DIV=$bd timeout 600 python bench.py --no-cpu-baseline --e2e-steps 3 --steps 3 > $OUT/bd$bd.json 2> $OUT/bd$bd.err
  python -c "import json;d=json.load(open('$OUT/bd$bd.json'));print('batch_div $bd',d['value'],d['e2e']['value'],d['e2e']['ms_per_step'])"
done
