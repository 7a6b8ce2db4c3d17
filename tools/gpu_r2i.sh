#!/bin/bash
# Round-2 session i: the other BASELINE configs on the triangle-bound build.
TAG=${1:-r2i}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in 1 3 5; do
  timeout 1500 python bench.py --config $c > $OUT/c$c.json 2> $OUT/c$c.err
  echo "c$c rc=$?"; python -c "import json;d=json.load(open('$OUT/c$c.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],(d.get('e2e') or {}).get('value'),(d.get('cpu_baseline') or {}).get('value'),d['setup_s'])"
done
timeout 2400 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 > $OUT/c4.json 2> $OUT/c4.err
echo "c4 rc=$?"; python -c "import json;d=json.load(open('$OUT/c4.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['e2e']['value'],d['cpu_baseline'],d['setup_s'],d['stats'])"
