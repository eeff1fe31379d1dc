"""Time skh_sketch_csr on C4-like shapes to separate write cost from staging/reduce."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_11815_b200 as skh  # noqa: E402
from paper_2105_11815_b200 import build  # noqa: E402
from synth import configs, device  # noqa: E402

build.build()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for (n, d, m, s, k) in [(1 << 20, 8192, 16384, 3, 8), (1024, 8192, 16384, 3, 8), (1 << 20, 4096, 16384, 3, 8),
                        (1 << 20, 2048, 16384, 3, 8), (1 << 19, 8192, 16384, 3, 8), (1 << 20, 8192, 16384, 1, 8),
                        (1 << 20, 8192, 4096, 3, 8)]:
    cfg = configs.C4.scaled(n=n, d=d, m=m)
    cfg = type(cfg)(cfg.name, "csr", n, d, m, s, 4, False, nnz_row=k)
    rp, ci, v = device.csr(cfg)
    bl = skh.hash_gen(4, m, s, n)
    SA = torch.empty(m, d, dtype=torch.float64, device="cuda")
    ms = t(lambda: skh.sketch_csr(bl, rp, ci, v, d, SA=SA))
    print(f"n={n} d={d} m={m} s={s} k={k}: {ms:.3f} ms  SA {m*d*8/1e9:.2f} GB -> {m*d*8/ms/1e6:.0f} GB/s", flush=True)
