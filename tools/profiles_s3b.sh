#!/bin/bash
# ncu --set full of the dominant kernel of C3 (s = 2 gather), C3HD (9-bit tile pass)
# and C2 (fused column-major pass, two columns per CTA) at the final code.
set -x
B="--no-e2e --no-cpu-baseline --no-all-workloads --no-alt-layout --no-graph --steps 1 --warmup 1"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gather_group_kernel -c 1 --launch-skip 1 \
  -o gpurun_out/s3_gather_c3 -f python bench.py --workload C3 $B > gpurun_out/s3_ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fwht_tile_kernel -c 1 --launch-skip 2 \
  -o gpurun_out/s3_tile9_c3hd -f python bench.py --workload C3HD $B > gpurun_out/s3_ncu_c3hd.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cm_gather_kernel -c 1 --launch-skip 1 \
  -o gpurun_out/s3_cmg_c2 -f python bench.py --workload C2 $B > gpurun_out/s3_ncu_c2.log 2>&1
echo done
