#!/bin/bash
# Final evidence of a build: GPU suite, the default bench line, the ncu launch
# list of the same command and one ncu --set full capture of the walk kernel.
TAG=${1:-final}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['build'],d['clocks'])"
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "ref rc=$?"; tail -c 300 $OUT/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
  -o $OUT/walk_full -f python bench.py --profile-only > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
