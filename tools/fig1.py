"""Reproduce the paper's Fig. 1 on the GPU sketches: kappa(A R^{-1})
vs m/d for the coherent A = [I_d; 0] + 1e-8 J (eq. (7.4)), n = 4000, d = 400,
HR-DHT (hashing, s = 1; and s = 2) vs SR-DHT (Blendenpik's sampling).
Writes one JSON line per m/d.   python tools/fig1.py [seeds]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_11815_b200 as skh  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n, d = 4000, 400
A = torch.full((n, d), 1e-8, dtype=torch.float64, device="cuda")
A[torch.arange(d), torch.arange(d)] += 1.0


def kappa(SA):
    R = torch.linalg.qr(SA, mode="r")[1]
    sv = torch.linalg.svdvals(torch.linalg.solve_triangular(R, A, upper=True, left=False))
    return float(sv[0] / sv[-1]) if float(sv[-1]) > 0 else float("inf")


for ratio in (1.1, 1.25, 1.5, 1.75, 2.0, 2.5, 3.0, 4.0):
    m = int(ratio * d)
    row = {"m_over_d": ratio, "m": m}
    for name, fn in (("hashing_s1", lambda sd: skh.hrdht_dense(sd, A, None, m, 1)[0]),
                     ("hashing_s2", lambda sd: skh.hrdht_dense(sd, A, None, m, 2)[0]),
                     ("sampling", lambda sd: skh.srdht_dense(sd, A, None, m)[0])):
        ks = [kappa(fn(sd)) for sd in range(seeds)]
        row[name + "_median_kappa"] = statistics.median(ks)
        row[name + "_max_kappa"] = max(ks)
    print(json.dumps(row), flush=True)
