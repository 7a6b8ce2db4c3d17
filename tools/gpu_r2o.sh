#!/bin/bash
# A/B: leaner TMA refill (precomputed shared-window addresses, one asm block, no per-refill fence)
TAG=${1:-r2o}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "hub_rows or rmat_bit_exact or goldens" > $OUT/pytest.log 2>&1
echo "pytest rc=$?"; tail -1 $OUT/pytest.log
for v in base tma2 base tma2; do
  export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/$v/libdynwalk_b200.so
  for mode in force-ervs ervs-nojump; do
    timeout 900 python bench.py --mode $mode --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/${v}_$mode.json 2> $OUT/${v}_$mode.err
    python -c "import json;d=json.load(open('$OUT/${v}_$mode.json'));print('$v $mode',d['value'],d['roofline']['frac'])"
  done
done
