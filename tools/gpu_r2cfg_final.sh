#!/bin/bash
# per-config bench lines of the final round-2 build (configs 1, 3, 5; config 4 is ~8.5 min)
TAG=${1:-cfgfinal}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in 1 3 5; do
  timeout 1500 python bench.py --config $c > $OUT/c$c.json 2> $OUT/c$c.err; echo "c$c rc=$?"
  python -c "import json;d=json.load(open('$OUT/c$c.json'));print('c$c',d['value'],(d.get('roofline') or {}).get('frac'),d['e2e']['value'],d['ms_per_step'],(d.get('cpu_baseline') or {}).get('value'))"
done
