#!/bin/bash
# dw_run_device listed walks (default) vs every walker launched (DW_DIRECT=0), s24 value, same box
TAG=${1:-r2ag}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in listed all listed all; do
  if [ $v = all ]; then export DW_DIRECT=0; else unset DW_DIRECT; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $OUT/s24_$v.json 2> $OUT/s24_$v.err
  python -c "import json;d=json.load(open('$OUT/s24_$v.json'));r=d['roofline'];print('$v',d['value'],d['ms_per_step'],r['frac'],r['kernel_ms_per_launch'],d['e2e']['value'],d['gpu_launches'])"
done
