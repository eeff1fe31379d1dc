#!/bin/bash
# ncu launch lists (time + DRAM bytes per launch) of the bench step per workload:
#   bash tools/launch_lists.sh OUTDIR [workloads...]
# Each command runs once plainly (must exit 0) before it runs under ncu.
out=${1:-gpurun_out/ll}; shift
mkdir -p "$out"
for w in ${@:-C5 C2 C3HD C3 C4 C1}; do
  for lay in auto row; do
    [ "$lay" = row ] && [ "$w" != C5 ] && [ "$w" != C2 ] && continue
    cmd="python bench.py --workload $w --layout $lay --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-alt-layout --no-all-workloads --no-graph"
    $cmd > "$out/plain_${w}_${lay}.log" 2>&1 && \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --csv --log-file "$out/launches_${w}_${lay}.csv" $cmd > "$out/ncu_${w}_${lay}.log" 2>&1
    echo "$w $lay rc=$?"
  done
done
