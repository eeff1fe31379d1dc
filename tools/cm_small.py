"""C5-shaped column-major HRHT on fewer columns (for ncu): python tools/cm_small.py d"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_11815_b200 as skh  # noqa: E402
from synth import configs, device  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = configs.C5.scaled(d=d)
At = device.dense_colmajor(cfg)
op = skh.RhtDenseColMajor(cfg.n, cfg.m, cfg.s, cfg.d)
for _ in range(2):
    op(cfg.seed, At)
torch.cuda.synchronize()
