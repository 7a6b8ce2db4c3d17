bash tools/gpu_variants.sh r1e
mkdir -p gpurun_out/r1e
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 -o gpurun_out/r1e/walk_lib -f python bench.py --profile-only > gpurun_out/r1e/ncu_lib.log 2>&1
