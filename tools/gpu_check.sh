#!/bin/bash
# One gpurun session: GPU parity tests, the bench (both arms), and ncu captures
# of the walk kernel.  Usage (from this container):
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tag] [steps...]'
# steps: tests bench ref l2 ncu full (default: all)
set -u
TAG=${1:-run}; shift || true
STEPS=${*:-"tests bench ref l2 ncu full"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/gpu.txt" 2>&1
has() { [[ " $STEPS " == *" $1 "* ]]; }
if has tests; then
  timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
  tail -3 "$OUT/pytest_gpu.log"
fi
if has bench; then
  timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"
  tail -c 600 "$OUT/bench.json"
fi
if has ref; then
  timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "ref rc=$?"
fi
if has l2; then
  for f in 32 64 128; do
    DW_VERBOSE=1 DW_L2_FETCH=$f timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 3 > "$OUT/bench_l2_$f.json" 2> "$OUT/bench_l2_$f.err"
    python -c "import json,sys;d=json.load(open('$OUT/bench_l2_$f.json'));print('l2',$f,d['value'],d['roofline']['frac'])"
  done
fi
if has ncu; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > "$OUT/ncu_bench.log" 2>&1
  echo "ncu launches rc=$?"
fi
if has full; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
    -o "$OUT/walk_full" -f python bench.py --profile-only > "$OUT/ncu_full.log" 2>&1
  echo "ncu full rc=$?"
fi
