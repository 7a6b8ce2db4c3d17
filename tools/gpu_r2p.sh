#!/bin/bash
TAG=${1:-r2p}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for h in 0.02 0.05 0.1; do
  timeout 900 python bench.py --config 4 --scale 22 --handoff $h --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/c4_h$h.json 2> $OUT/c4_h$h.err
  python -c "import json;d=json.load(open('$OUT/c4_h$h.json'));print('h $h',d['value'],d['roofline']['frac'],d['stats']['trials'],d['stats']['weight_reads'])"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
  -o $OUT/c4_full -f python bench.py --profile-only --config 4 --scale 20 > $OUT/ncu_c4.log 2>&1
echo "ncu c4 rc=$?"
