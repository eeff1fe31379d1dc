import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2105_11815_b200 as skh
from synth import configs, device
for name in ("C2", "C3HD"):
    cfg = configs.ALL[name]
    At = device.dense_colmajor(cfg); b = device.rhs(cfg)
    n, d = cfg.n, cfg.d
    ws = torch.empty(skh._lib.load().skh_hrdht_dense_colmajor_workspace_bytes(n, cfg.m, cfg.s, d), dtype=torch.uint8, device="cuda")
    SAt = torch.empty(d, cfg.m, dtype=torch.float64, device="cuda"); Sb = torch.empty(cfg.m, dtype=torch.float64, device="cuda")
    f = lambda: skh.hrdht_dense_colmajor(cfg.seed, At, b, cfg.m, cfg.s, SAt=SAt, Sb=Sb, ws=ws)
    f(); torch.cuda.synchronize()
    for _ in range(2):
        with skh.Trace(16) as tr:
            f()
        torch.cuda.synchronize()
        dd = tr.durations_ms(); print(name, round(sum(dd.values()), 4), {k: round(v, 4) for k, v in dd.items()})
    del At, ws
