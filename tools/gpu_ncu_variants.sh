#!/bin/bash
# ncu --set full of the walk kernel for the main library and each variant.
TAG=${1:-ncu}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in paper_2512_00705_b200/lib paper_2512_00705_b200/variants/*; do
  [ -f $v/libdynwalk_b200.so ] || continue
  n=$(basename $v)
  DYNWALK_B200_LIB=$v/libdynwalk_b200.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel -c 1 -o $OUT/walk_$n -f python bench.py --profile-only > $OUT/ncu_$n.log 2>&1
  echo "ncu $n rc=$?"
done
