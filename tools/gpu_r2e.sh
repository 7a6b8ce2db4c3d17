#!/bin/bash
# Round-2 session e: merge membership + TMA stage fix + NOJUMP draw fix.
TAG=${1:-r2e}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -s -k "goldens or hub_rows or metapath or tier2 or rmat_bit_exact or layouts or extreme" > $OUT/pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|Error" $OUT/pytest.log | tail -4
run() {  # tag, env..., args...
  local t=$1; shift
  env "$@" > /dev/null 2>&1
}
for v in tma notma; do
  if [ $v = notma ]; then export DYNWALK_B200_LIB=paper_2512_00705_b200/variants/notma/libdynwalk_b200.so; else unset DYNWALK_B200_LIB; fi
  timeout 900 python bench.py --mode force-ervs --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/ervs_$v.json 2> $OUT/ervs_$v.err
  echo "force-ervs $v rc=$?"; python -c "import json;d=json.load(open('$OUT/ervs_$v.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
done
unset DYNWALK_B200_LIB
timeout 900 python bench.py --mode ervs-nojump --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/nojump.json 2> $OUT/nojump.err
echo "nojump rc=$?"; python -c "import json;d=json.load(open('$OUT/nojump.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
timeout 1200 python bench.py --config 4 --scale 22 --steps 3 --warmup 3 --e2e-steps 1 > $OUT/c4_s22.json 2> $OUT/c4_s22.err
echo "c4 s22 rc=$?"; python -c "import json;d=json.load(open('$OUT/c4_s22.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['stats'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
  -o $OUT/ervs_full -f python bench.py --profile-only --mode force-ervs --scale 20 > $OUT/ncu_ervs.log 2>&1
echo "ncu ervs rc=$?"
