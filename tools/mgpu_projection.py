"""Per-rank kernel times behind the multi-GPU projection of C5,
measured on ONE B200 with the column-major H.D path at the shard's shape:

  M3 (exchange-free): rank r sketches its L = n/G local rows with the folded
      lists T_r -- G s entries per local row, every local row read once and
      fanned out on chip by the fused pass 2 -- the same kernels and list
      statistics as RhtDenseColMajor(L, m, G s, d).
  M2 (butterfly all-to-all): the local transform + gather of L rows with s
      entries, RhtDenseColMajor(L, m, s, d), plus one more 2|A_r| pass for the
      log2 G cross bits (timed here as a pass-1 launch over the shard) and the
      (G-1)/G |A_r| all-to-all (bounded below by NVLink 5's 900 GB/s per
      direction, not measured: one GPU).

  python tools/mgpu_projection.py [reps]    -> one JSON line per G
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_11815_b200 as skh  # noqa: E402
from synth import configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
C5 = configs.C5
T1 = None


def timed(fn):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


g = torch.Generator(device="cuda").manual_seed(5)
for G in (1, 2, 4, 8):
    L = C5.n // G
    At = torch.randn(C5.d, L, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(L, dtype=torch.float64, device="cuda", generator=g)
    op1 = skh.RhtDenseColMajor(L, C5.m, C5.s, C5.d)
    t_m2_local = timed(lambda: op1(C5.seed, At, b))
    del op1
    torch.cuda.empty_cache()
    rec = {"G": G, "L": L, "d": C5.d, "m": C5.m}
    if G == 1:
        T1 = t_m2_local
        rec["single_gpu_ms"] = round(T1, 3)
    else:
        opG = skh.RhtDenseColMajor(L, C5.m, C5.s * G, C5.d)
        t_m3 = timed(lambda: opG(C5.seed, At, b))
        del opG
        torch.cuda.empty_cache()
        a_r = L * C5.d * 8
        cross = 2 * a_r / 6552.6e9 * 1e3  # one more read+write pass at the measured copy rate
        a2a = (G - 1) / G * a_r / 900e9 * 1e3  # NVLink 5 per-direction bound
        m2 = max(t_m2_local + cross, a2a)  # perfect overlap of the exchange with compute
        rec.update({"m3_rank_ms": round(t_m3, 3), "m3_eff": round(T1 / (G * t_m3), 3),
                    "m2_local_ms": round(t_m2_local, 3), "m2_cross_pass_ms": round(cross, 3),
                    "m2_a2a_bound_ms": round(a2a, 3), "m2_rank_ms_overlapped": round(m2, 3),
                    "m2_eff_overlapped": round(T1 / (G * m2), 3),
                    "m2_eff_serialised": round(T1 / (G * (t_m2_local + cross + a2a)), 3)})
    print(json.dumps(rec), flush=True)
    del At, b
    torch.cuda.empty_cache()
