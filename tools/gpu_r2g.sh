#!/bin/bash
# Round-2 session g: merge gating, nojump screen, PR2 wide kernels.
TAG=${1:-r2g}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -s -k "goldens or hub_rows or tier2 or rmat_bit_exact or pr2_pareto or layouts" > $OUT/pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|Error" $OUT/pytest.log | tail -4
for mode in force-ervs ervs-nojump; do
  timeout 900 python bench.py --mode $mode --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/$mode.json 2> $OUT/$mode.err
  echo "$mode rc=$?"; python -c "import json;d=json.load(open('$OUT/$mode.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
done
for v in wide narrow; do
  if [ $v = narrow ]; then export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/narrow/libdynwalk_b200.so; else unset DYNWALK_B200_LIB; fi
  timeout 900 python bench.py --config 4 --scale 22 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/c4_s22_$v.json 2> $OUT/c4_s22_$v.err
  echo "c4 s22 $v rc=$?"; python -c "import json;d=json.load(open('$OUT/c4_s22_$v.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['stats']['trials'])"
done
unset DYNWALK_B200_LIB
timeout 900 python bench.py --config 4 --scale 22 --handoff 0.05 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/c4_s22_h005.json 2> $OUT/c4_s22_h005.err
echo "c4 s22 h0.05 rc=$?"; python -c "import json;d=json.load(open('$OUT/c4_s22_h005.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['stats']['trials'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
  -o $OUT/ervs_full -f python bench.py --profile-only --mode force-ervs --scale 20 > $OUT/ncu_ervs.log 2>&1
echo "ncu ervs rc=$?"
