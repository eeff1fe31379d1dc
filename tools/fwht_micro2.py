"""Time one FWHT pass of width K for several K (and the wide-pass mode from
SKH_FWHT_WIDE = fused | cluster | tile)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_11815_b200 as skh  # noqa: E402
from paper_2105_11815_b200 import build  # noqa: E402

build.build()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 19
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
Ks = [int(k) for k in sys.argv[3].split(",")] if len(sys.argv) > 3 else [7, 8, 9, 10, 11]
A = torch.randn(n, d, dtype=torch.float64, device="cuda")
Y = torch.empty_like(A)
ws = skh.api.rht_stages_workspace(n, n, 0, d)


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


gb = 2 * n * d * 8 / 1e9
mode = os.environ.get("SKH_FWHT_WIDE", "fused")
for K in Ks:
    for lo, diag, src in ((0, True, A), (0, False, Y), (8, False, Y)):
        if lo + K > n.bit_length() - 1:
            continue
        ms = t(lambda: skh.rht_stages(1, src, lo, lo + K, nrows=n, apply_diag=diag, Y=Y, ws=ws))
        print(f"[{mode}] K={K:2d} bits[{lo},{lo+K}) diag={diag} inplace={src is Y}: {ms:.3f} ms  {gb/ms*1e3:.0f} GB/s",
              flush=True)
ms = t(lambda: Y.copy_(A))
print(f"torch copy: {ms:.3f} ms {gb/ms*1e3:.0f} GB/s")
