"""One small call of every libskh entry point that launches kernels, for
compute-sanitizer (memcheck / racecheck / synccheck):
  compute-sanitizer --tool racecheck python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2105_11815_b200 as skh  # noqa: E402
from synth import configs, gen  # noqa: E402

dev = "cuda"
r = np.random.default_rng(0)
n, d, m = 4096 * 4 + 7, 24, 96
A = torch.from_numpy(r.standard_normal((n, d))).to(dev)
b = torch.from_numpy(r.standard_normal(n)).to(dev)
for s in (1, 3):
    bl = skh.hash_gen(1, m, s, n)                         # segmented transpose path (N <= 96 m)
    skh.sketch_dense(bl, A, b)
    blv = skh.hash_gen(1, 8, s, 3000, variant=True)       # radix path (m < 64)
    skh.sketch_dense(blv, A[:3000], b[:3000])
skh.rht_dense(2, A, b, m, 1)                              # FWHT tile passes + gather
Y = skh.rht_stages(3, A[:4096], 0, 12, apply_diag=True)
At = A.t().contiguous()
skh.rht_dense_colmajor(4, At, b, m, 2)                    # cm pass 1 + fused pass 2 (K2 = 2)
skh.sketch_dense_colmajor(4, At, b, m, 2)                 # cm gather (K2 = 0)
skh.rht_colmajor(5, torch.zeros(2, 1 << 22, dtype=torch.float64, device=dev)[:, :(1 << 21) + 5],
                 nrows=1 << 22)                           # mid pass (L = 22)
cfg = configs.C4.scaled(n=3000, d=300, m=50)
rp, ci, v = gen.csr(cfg)
blc = skh.hash_gen(cfg.seed, cfg.m, cfg.s, cfg.n)
skh.sketch_csr(blc, torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev), torch.from_numpy(v).to(dev), cfg.d,
               torch.from_numpy(gen.rhs(cfg)).to(dev))
skh.hrdht_dense(6, A, b, m, 1)
skh.hrdht_dense_colmajor(6, At, b, m, 1)
skh.srdht_dense(6, A, b, m)
SA, Sb = skh.rht_dense(7, A, b, m, 1)
skh.lls_solve(A, b, SA, Sb, it_max=5)
SAt, Sbt = skh.rht_dense_colmajor(7, At, b, m, 1)
skh.LlsSolver(n, d, m)(At, b, SAt, Sbt, it_max=5, colmajor=True)
parts = torch.randn(3, 5, 7, dtype=torch.float64, device=dev)
skh.ordered_sum(parts, 0.5)
torch.cuda.synchronize()
print("sanitize_small: done")
