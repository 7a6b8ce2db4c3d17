#!/bin/bash
# Round-2 session f: window-rank membership, ski-rental hand-off, config 4 at s25, ratio sweep.
TAG=${1:-r2f}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -s -k "goldens or hub_rows or tier2 or rmat_bit_exact or layouts or extreme" > $OUT/pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|Error" $OUT/pytest.log | tail -4
for mode in force-ervs ervs-nojump; do
  timeout 900 python bench.py --mode $mode --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/$mode.json 2> $OUT/$mode.err
  echo "$mode rc=$?"; python -c "import json;d=json.load(open('$OUT/$mode.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
  -o $OUT/ervs_full -f python bench.py --profile-only --mode force-ervs --scale 20 > $OUT/ncu_ervs.log 2>&1
echo "ncu ervs rc=$?"
timeout 900 python bench.py --config 4 --scale 22 --steps 3 --warmup 3 --e2e-steps 1 > $OUT/c4_s22.json 2> $OUT/c4_s22.err
echo "c4 s22 rc=$?"; python -c "import json;d=json.load(open('$OUT/c4_s22.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['stats'])"
for r in 0.35 0.5 0.7 1.0 1.4; do
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 5 --ratio $r > $OUT/sweep_$r.json 2> $OUT/sweep_$r.err
  python -c "import json;d=json.load(open('$OUT/sweep_$r.json'));print('ratio',$r,d['value'],d['roofline']['frac'])"
done
timeout 2000 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 > $OUT/c4_s25.json 2> $OUT/c4_s25.err
echo "c4 s25 rc=$?"; python -c "import json;d=json.load(open('$OUT/c4_s25.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['stats'])"; tail -2 $OUT/c4_s25.err
