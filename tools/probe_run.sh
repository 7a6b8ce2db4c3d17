#!/bin/bash
# gather_probe throughput + DRAM bytes per request (ncu), see tools/gather_probe.cu
OUT=gpurun_out/${1:-probe}
mkdir -p $OUT
[ -x tools/bin/gather_probe ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/gather_probe tools/gather_probe.cu
tools/bin/gather_probe 32 > $OUT/probe.json 2>&1
tools/bin/gather_probe 32 32 > $OUT/probe_l2fetch32.json 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__sectors_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none -c 11 --csv --log-file $OUT/probe_ncu.csv tools/bin/gather_probe 32 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -c 11 --csv --log-file $OUT/probe_ncu_l2f32.csv tools/bin/gather_probe 32 32 > /dev/null 2>&1
echo "probe done"
cat $OUT/probe.json $OUT/probe_l2fetch32.json
