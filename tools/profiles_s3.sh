#!/bin/bash
# Final-state evidence for round 2 (session 3): launch lists of every workload's
# bench step, then ncu --set full of the two C5 column-major kernels.
set -x
bash tools/launch_lists.sh gpurun_out/ll_s3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cm_gather_kernel -c 1 --launch-skip 1 \
  -o gpurun_out/s3_cmg_c5 -f python tools/cm_bench.py C5 1 > gpurun_out/s3_ncu_cmg.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cm_pass1 -c 1 --launch-skip 1 \
  -o gpurun_out/s3_p1_c5 -f python tools/cm_bench.py C5 1 > gpurun_out/s3_ncu_p1.log 2>&1
echo done
