#!/bin/bash
# One gpurun session with selectable steps.  From this container:
#   gpurun --timeout 2400 -- 'bash tools/gpu_session.sh <tag> <step> [<step> ...]'
# steps:
#   tests        pytest -m gpu
#   bench        python bench.py (default headline line, both legs)
#   ref          python bench.py --impl reference
#   sweep        headline walk at fixed ratios (no e2e / cpu leg)
#   launches     ncu launch list of a short bench run
#   full         ncu --set full of one walk kernel launch (+ source)
#   cfg<C>       bench.py --config C (C = 1, 3, 4, 5)
set -u
TAG=${1:-run}; shift || true
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/gpu.txt" 2>&1
for step in "$@"; do
  case $step in
    tests)
      timeout 1800 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
      echo "pytest rc=$?" | tee -a "$OUT/pytest_gpu.log"; tail -3 "$OUT/pytest_gpu.log" ;;
    bench)
      timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"
      python -c "import json;d=json.load(open('$OUT/bench.json'));print('value',d['value'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],'ratio',d['config']['edge_cost_ratio'])" ;;
    ref)
      timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "ref rc=$?" ;;
    sweep)
      for r in ${SWEEP:-1.0 1.2 1.4 1.6 2.0 2.33}; do
        timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 5 --ratio $r > "$OUT/sweep_$r.json" 2> "$OUT/sweep_$r.err"
        python -c "import json;d=json.load(open('$OUT/sweep_$r.json'));print('ratio',$r,d['value'],d['roofline']['frac'])"
      done ;;
    launches)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > "$OUT/ncu_bench.log" 2>&1
      echo "ncu launches rc=$?" ;;
    full)
      timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 \
        -o "$OUT/walk_full" -f python bench.py --profile-only ${FULL_ARGS:-} > "$OUT/ncu_full.log" 2>&1
      echo "ncu full rc=$?" ;;
    cfg*)
      c=${step#cfg}
      timeout 1500 python bench.py --config $c ${CFG_ARGS:-} > "$OUT/bench_c$c.json" 2> "$OUT/bench_c$c.err"; echo "cfg$c rc=$?"
      tail -c 300 "$OUT/bench_c$c.json" ;;
    *) echo "unknown step $step" ;;
  esac
done
