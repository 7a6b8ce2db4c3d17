#!/bin/bash
# Warp-reservoir session: hub parity tests, then force-ervs / ervs-nojump at
# s24 with the parallel jump chain and with the sequential one (variant lib).
#   gpurun -- 'bash tools/gpu_ervs.sh <tag> [scale]'
TAG=${1:-ervs}; SC=${2:-24}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hub_rows or rmat_bit_exact or extreme or layouts or goldens" > $OUT/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for mode in force-ervs ervs-nojump; do
  timeout 900 python bench.py --mode $mode --scale $SC --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/par_$mode.json 2> $OUT/par_$mode.err
  echo "par $mode rc=$?"; python -c "import json;d=json.load(open('$OUT/par_$mode.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
done
DYNWALK_B200_LIB=paper_2512_00705_b200/variants/seq/libdynwalk_b200.so timeout 900 python bench.py --mode force-ervs --scale $SC --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/seq_force-ervs.json 2> $OUT/seq_force-ervs.err
echo "seq rc=$?"; python -c "import json;d=json.load(open('$OUT/seq_force-ervs.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
