#!/bin/bash
# Round-2 session h: triangle bound -- full parity, headline, config 4 s22, ncu of the headline.
TAG=${1:-r2h}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|Error" $OUT/pytest.log | tail -4
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['stats'],d['setup_s'])"
timeout 900 python bench.py --config 4 --scale 22 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/c4_s22.json 2> $OUT/c4_s22.err
echo "c4 s22 rc=$?"; python -c "import json;d=json.load(open('$OUT/c4_s22.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['stats']['trials'])"
timeout 900 python bench.py --mode force-ervs --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/force-ervs.json 2> $OUT/force-ervs.err
echo "force-ervs rc=$?"; python -c "import json;d=json.load(open('$OUT/force-ervs.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
  -o $OUT/walk_full -f python bench.py --profile-only > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
