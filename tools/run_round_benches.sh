set -x
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench_C5_row.log 2>&1
python bench.py --layout col > gpurun_out/final/bench_C5_col.log 2>&1
for w in C1 C2 C3 C3HD C4; do python bench.py --workload $w --steps 10 > gpurun_out/final/bench_${w}_row.log 2>&1; done
for w in C1 C2 C3 C3HD; do python bench.py --workload $w --layout col --steps 10 > gpurun_out/final/bench_${w}_col.log 2>&1; done
for w in C2 C3HD C5; do timeout 300 python tools/bench_lls.py $w 2 >> gpurun_out/final/lls_bench.log 2>&1; done
for w in C2 C3HD C5; do timeout 300 python tools/cm_bench.py $w 2 >> gpurun_out/final/cm_bench.log 2>&1; done
mkdir -p gpurun_out/sketches
for w in C2 C3HD; do for sk in dht srdht; do python bench.py --workload $w --sketch $sk --steps 10 --no-alt-layout > gpurun_out/sketches/bench_${w}_${sk}.log 2>&1; done; done
for w in C2 C3 C3HD C4 C5; do python bench.py --workload $w --sketch variant --steps 10 --no-alt-layout > gpurun_out/sketches/bench_${w}_variant.log 2>&1; done
for w in C2 C3HD; do SKH_LLS_RINV=1 timeout 300 python tools/bench_lls.py $w 2 >> gpurun_out/final/lls_bench.log 2>&1; done
for w in C2 C5; do timeout 300 python tools/bench_lls.py $w 2 col >> gpurun_out/final/lls_bench.log 2>&1; done
