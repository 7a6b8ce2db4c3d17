#!/bin/bash
TAG=${1:-r2k}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['setup_s'])"
timeout 900 python bench.py --config 4 --scale 22 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/c4_s22.json 2> $OUT/c4_s22.err
echo "c4 s22 rc=$?"; python -c "import json;d=json.load(open('$OUT/c4_s22.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
timeout 2400 python bench.py --config 4 > $OUT/c4.json 2> $OUT/c4.err
echo "c4 rc=$?"; python -c "import json;d=json.load(open('$OUT/c4.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['e2e']['value'],d['setup_s'])"
