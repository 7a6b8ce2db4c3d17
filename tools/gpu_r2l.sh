#!/bin/bash
TAG=${1:-r2l}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
for v in mask nomask mask2; do
  if [ $v = nomask ]; then export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/nomask/libdynwalk_b200.so; else unset DYNWALK_B200_LIB; fi
  timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  echo "bench $v rc=$?"; python -c "import json;d=json.load(open('$OUT/bench_$v.json'));print(d['value'],d['roofline']['frac'],d['e2e']['value'])"
done
