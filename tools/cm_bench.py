"""Stage timing of the column-major HRHT path (skh_rht_dense_colmajor) on a
BASELINE workload, via the library's stage trace.  Usage:
  python tools/cm_bench.py [C5|C2|C3HD|C3] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_11815_b200 as skh  # noqa: E402
from synth import configs, device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = configs.ALL[name]
At = device.dense_colmajor(cfg)
b = device.rhs(cfg)
torch.cuda.synchronize()
if cfg.hd:
    op = skh.RhtDenseColMajor(cfg.n, cfg.m, cfg.s, cfg.d)
    call = lambda: op(cfg.seed, At, b)  # noqa: E731
else:
    ws = None
    call = lambda: skh.sketch_dense_colmajor(cfg.seed, At, b, cfg.m, cfg.s)  # noqa: E731
call()
torch.cuda.synchronize()
for r in range(reps):
    with skh.Trace(16) as tr:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
    torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    abytes = cfg.n * cfg.d * 8
    st = {k: round(v, 3) for k, v in tr.durations_ms().items()}
    print(f"{name} total {tot:.3f} ms  A-GB/s {abytes / tot / 1e6:.1f}  stages {st}", flush=True)
