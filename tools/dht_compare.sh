mkdir -p gpurun_out
for w in C2 C3HD; do
  python bench.py --workload $w --sketch dht --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alt-layout 2>/dev/null | tail -1 | python -c "import json,sys;l=json.loads(sys.stdin.read());print('$w fht', l['ms_per_step'], l['value'], json.dumps(l['roofline']), l.get('stages_ms'))"
  SKH_DHT_CUFFT=1 python bench.py --workload $w --sketch dht --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alt-layout 2>/dev/null | tail -1 | python -c "import json,sys;l=json.loads(sys.stdin.read());print('$w cufft', l['ms_per_step'], l['value'], l.get('stages_ms'))"
done
