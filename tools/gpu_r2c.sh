#!/bin/bash
# Round-2 session: new parity tests, force-ervs ncu capture at s20, configs 4 and 5.
TAG=${1:-r2c}
OUT=gpurun_out/$TAG; mkdir -p $OUT
{ free -g; nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; } > $OUT/host.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "tier2 or libdevice or hub_rows" > $OUT/pytest.log 2>&1
echo "pytest rc=$?"; grep -E "fn=|passed|failed" $OUT/pytest.log | tail -6
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
  -o $OUT/ervs_full -f python bench.py --profile-only --mode force-ervs --scale 20 > $OUT/ncu_ervs.log 2>&1
echo "ncu ervs rc=$?"
for sc in 22 25; do
  timeout 1500 python bench.py --config 4 --scale $sc --steps 3 --warmup 3 --e2e-steps 1 > $OUT/c4_s$sc.json 2> $OUT/c4_s$sc.err
  echo "c4 s$sc rc=$?"; tail -c 600 $OUT/c4_s$sc.json; tail -3 $OUT/c4_s$sc.err
done
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 --e2e-steps 2 > $OUT/c5.json 2> $OUT/c5.err
echo "c5 rc=$?"; tail -c 800 $OUT/c5.json; tail -3 $OUT/c5.err
