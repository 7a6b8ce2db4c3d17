#!/bin/bash
# Round-2 session d: TMA warp reservoir + MetaPath label screen.
TAG=${1:-r2d}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -s -k "hub_rows or metapath or goldens or tier2 or libdevice or rmat_bit_exact" > $OUT/pytest.log 2>&1
echo "pytest rc=$?"; grep -E "fn=|passed|failed|Error" $OUT/pytest.log | tail -8
for v in tma notma; do
  lib=""; [ $v = notma ] && lib=paper_2512_00705_b200/variants/notma/libdynwalk_b200.so
  DYNWALK_B200_LIB=$lib timeout 900 python bench.py --mode force-ervs --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/ervs_$v.json 2> $OUT/ervs_$v.err
  echo "force-ervs $v rc=$?"; python -c "import json;d=json.load(open('$OUT/ervs_$v.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
done
timeout 900 python bench.py --mode ervs-nojump --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/nojump_tma.json 2> $OUT/nojump_tma.err
echo "nojump rc=$?"; python -c "import json;d=json.load(open('$OUT/nojump_tma.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
for l in 1 0; do
  DW_LAB2=$l timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/c3_lab$l.json 2> $OUT/c3_lab$l.err
  echo "c3 lab2=$l rc=$?"; python -c "import json;d=json.load(open('$OUT/c3_lab$l.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['roofline'].get('mix_bytes_per_walker_step'))"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
  -o $OUT/ervs_tma_full -f python bench.py --profile-only --mode force-ervs --scale 20 > $OUT/ncu_ervs.log 2>&1
echo "ncu ervs rc=$?"
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['roofline']['frac'],d['e2e']['value'])"
