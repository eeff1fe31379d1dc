"""Experiment: the row-major H D path of C3HD run slab by slab (w columns at a
time) so that the transform's intermediate (n x w x 8 bytes) stays in L2
between the two FWHT passes and the gather; composed from the existing C-ABI
calls.  Times eager and CUDA-graph replays and compares SA with the
one-shot HrhtStep bit for bit.

    python tools/slab_probe.py [w ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_11815_b200 import api, pipeline  # noqa: E402
from synth import configs  # noqa: E402


class SlabStep:
    def __init__(self, seed, A, b, m, s, w):
        self.seed, self.m, self.s, self.w = seed, m, s, w
        self.A, self.b = A, b
        n, d = A.shape
        self.n, self.d = n, d
        self.L = n.bit_length() - 1
        self.plan = api.rht_pass_plan(self.L, w, True)
        dev = A.device
        self.S = torch.empty(n, w, dtype=torch.float64, device=dev)
        self.yb = torch.empty(n, 1, dtype=torch.float64, device=dev)
        self.SA = torch.empty(m, d, dtype=torch.float64, device=dev)
        self.Sb = torch.empty(m, dtype=torch.float64, device=dev)
        self.ws = api.rht_stages_workspace(n, n, 0, w, dev)
        self.wsb = api.rht_stages_workspace(n, n, 0, 1, dev)
        self.alpha = api.c_ns(n, s)
        self.bl = None

    def run(self, timer=None):
        self.bl = api.hash_gen(self.seed, self.m, self.s, self.n, out=self.bl)
        api.rht_stages(self.seed, self.b.view(-1, 1), 0, self.L, nrows=self.n, apply_diag=True, alpha=1.0,
                       Y=self.yb, ws=self.wsb)
        for c0 in range(0, self.d, self.w):
            lo = 0
            for p, k in enumerate(self.plan):
                src = self.A[:, c0:c0 + self.w] if p == 0 else self.S
                api.rht_stages(self.seed, src, lo, lo + k, nrows=self.n, apply_diag=(p == 0), alpha=1.0, Y=self.S,
                               ws=self.ws)
                lo += k
            api.sketch_dense(self.bl, self.S, None, alpha=self.alpha, SA=self.SA[:, c0:c0 + self.w])
        api.sketch_dense(self.bl, self.yb, None, alpha=self.alpha, SA=self.Sb.view(-1, 1))
        return self.SA, self.Sb


def timeit(fn, k):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def main():
    ws = [int(x) for x in sys.argv[1:]] or [32, 64]
    torch.cuda.set_device(0)
    cfg = configs.ALL["C3HD"]
    if os.environ.get("SLAB_ONLY"):  # one eager step per width (for ncu launch lists)
        from synth import device
        A, b = device.dense(cfg), device.rhs(cfg)
        for w in ws:
            st = SlabStep(cfg.seed, A, b, cfg.m, cfg.s, w)
            st.run()
            torch.cuda.synchronize()
        return
    ref_step, (A, b) = bench.build_step(cfg, torch, "row")
    for _ in range(3):
        ref_step.run()
    t_ref = timeit(ref_step.run, 10)
    SA_ref = ref_step.SA.clone()
    Sb_ref = ref_step.Sb.clone()
    print(f"C3HD HrhtStep: {t_ref:.3f} ms", flush=True)
    del ref_step
    torch.cuda.empty_cache()
    for w in ws:
        st = SlabStep(cfg.seed, A, b, cfg.m, cfg.s, w)
        for _ in range(2):
            st.run()
        t_e = timeit(st.run, 5)
        same = torch.equal(st.SA, SA_ref) and torch.equal(st.Sb, Sb_ref)
        g, per = bench.capture_step(st, torch)
        t_g = timeit(g.replay, 10)
        print(f"w={w} plan={st.plan}: eager {t_e:.3f} ms, graph {t_g:.3f} ms ({per} launches), "
              f"bit-identical {same}", flush=True)
        del g, st
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
