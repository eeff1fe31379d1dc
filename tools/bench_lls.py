"""Algorithm 1 Steps 2-5 on a BASELINE workload (NEXT-1): time the solve that
consumes SA, Sb and report the LSQR iteration rate as A-bytes streamed per
second (each iteration reads A twice: A (R^-1 v) and A^T u).
  python tools/bench_lls.py [C2|C5|C3HD] [reps] [row|col]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_11815_b200 as skh  # noqa: E402
from synth import configs, device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
layout = sys.argv[3] if len(sys.argv) > 3 else "row"
cfg = configs.ALL[name]
b = device.rhs(cfg)
cm = layout == "col"
if cm:
    A = device.dense_colmajor(cfg)
    SA, Sb = skh.RhtDenseColMajor(cfg.n, cfg.m, cfg.s, cfg.d)(cfg.seed, A, b)
else:
    A = device.dense(cfg)
    SA, Sb = skh.RhtDense(cfg.n, cfg.m, cfg.s, cfg.d)(cfg.seed, A, b)
rr = len(sys.argv) > 3 and sys.argv[3] == "rr"
solver = skh.LlsSolver(cfg.n, cfg.d, cfg.m, rcond=1e-12 if rr else None)
solver(A, b, SA, Sb, colmajor=cm)  # warm-up (handles, cuSOLVER workspace)
torch.cuda.synchronize()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6549.4)
for _ in range(reps):
    with skh.Trace(16) as tr:
        x, info = solver(A, b, SA, Sb, colmajor=cm)
    torch.cuda.synchronize()
    st = tr.durations_ms()
    it = max(info["iters"], 1)
    per_it = st.get("lsqr", 0.0) / it
    gbs = 2 * cfg.a_bytes / (per_it / 1e3) / 1e9
    print(json.dumps({"workload": name, "layout": layout, "rinv": os.environ.get("SKH_LLS_RINV") == "1", "n": cfg.n, "d": cfg.d, "m": cfg.m, "step": info["step"],
                      "iters": info["iters"], "test2": info["test2"], "stages_ms": {k: round(v, 3) for k, v in st.items()},
                      "ms_per_lsqr_iter": round(per_it, 4), "A_GBps_per_iter": round(gbs, 1),
                      "frac_of_hbm_peak": round(gbs / peak, 3)}), flush=True)
