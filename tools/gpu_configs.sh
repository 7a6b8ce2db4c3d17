#!/bin/bash
# Bench lines for the non-headline BASELINE configs (both arms).
TAG=${1:-cfg}; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() {  # name, args...
  local n=$1; shift
  timeout 1200 python bench.py "$@" > $OUT/$n.json 2> $OUT/$n.err; echo "$n rc=$?"
  python - $OUT/$n.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    e = d.get("e2e") or {}
    print(f"  {d['metric']}: value={d['value']:.4g} e2e={e.get('value', 0):.4g} frac={(d.get('roofline') or {}).get('frac')} stats={d.get('stats', {})}")
except Exception as ex:
    print("  FAILED", ex)
PY
}
run c1 --config 1 --steps 3 --warmup 3
run c1ref --config 1 --impl reference --steps 2 --warmup 1
run c3 --config 3 --steps 3 --warmup 3
run c3ref --config 3 --impl reference --steps 2 --warmup 1
run c4s20 --config 4 --scale 20 --steps 2 --warmup 3 --e2e-steps 1 --cpu-seconds 10
run c4s20ref --config 4 --scale 20 --impl reference --steps 1 --warmup 0
