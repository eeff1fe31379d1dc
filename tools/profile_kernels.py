"""Small, ncu-friendly invocation of each hot kernel (one launch each after a
warm-up), for `ncu --set full -k regex:<name>` captures.

    python tools/profile_kernels.py [fused|tile|gather|csr|hash] ...
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_11815_b200 as skh  # noqa: E402
from paper_2105_11815_b200 import build  # noqa: E402
from synth import configs, device  # noqa: E402

build.build()
which = sys.argv[1:] or ["fused", "tile", "gather", "csr", "hash"]
n, d = 1 << 17, 4096  # 4 GiB: C5's row length, 1/16 of its rows
if "fused" in which or "tile" in which or "gather" in which:
    cfg = configs.C5.scaled(n=n)
    A = device.dense(cfg)
    Y = torch.empty_like(A)
    ws = skh.api.rht_stages_workspace(n, n, 0, d)
    for rep in range(2):  # rep 0 = warm-up
        if "fused" in which:
            skh.rht_stages(5, A, 0, 11, nrows=n, apply_diag=True, Y=Y, ws=ws)   # fused 7+4, D fused
            skh.rht_stages(5, Y, 11, 17, nrows=n, apply_diag=False, Y=Y, ws=ws)  # tile K=6
        if "tile" in which:
            skh.rht_stages(5, A, 0, 7, nrows=n, apply_diag=True, Y=Y, ws=ws)    # tile K=7, D fused
        if "gather" in which:
            bl = skh.hash_gen(5, 7168 // 16, 1, n)
            skh.sketch_dense(bl, Y, alpha=1.0)
    torch.cuda.synchronize()
    del A, Y
if "gather2" in which:  # C3: s = 2, 64-column slices re-read through L2
    cfg = configs.C3
    A = device.dense(cfg)
    bl = skh.hash_gen(cfg.seed, cfg.m, cfg.s, cfg.n)
    for rep in range(2):
        skh.sketch_dense(bl, A)
    torch.cuda.synchronize()
    del A
if "csr" in which:
    cfg = configs.C4
    rp, ci, v = device.csr(cfg)
    b = device.rhs(cfg)
    bl = skh.hash_gen(cfg.seed, cfg.m, cfg.s, cfg.n)
    for rep in range(2):
        skh.sketch_csr(bl, rp, ci, v, cfg.d, b)
    torch.cuda.synchronize()
if "hash" in which:
    for rep in range(2):
        skh.hash_gen(5, 7168, 1, 1 << 21)
    torch.cuda.synchronize()
print("ok")
