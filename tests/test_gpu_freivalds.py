"""Whole-matrix checks of SA at the full BASELINE sizes (SURVEY §8(c) tier 2):
Freivalds probes w^T (S A) v = (S^T w)^T (A v) over ALL m x d entries, for
the step objects bench.py times (bench.build_step, default layout).  S^T w
comes from the oracle's column lists (oracle/probes.py; for the
HRHT one oracle FWHT of an n-vector); A v is an fp64 library
matrix-vector product of the input (torch.mv / a host CSR product), not the
CUDA sketch path.  Bound: 1e-12 ||w|| ||SA||_F ||v|| per probe.
"""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2105_11815_b200.build as b
    b.build()


def freivalds(cfg, SA, Av_of, nprobe=4):
    """max over probes of |w^T SA v - (S^T w)^T (A v)| / (||w|| ||SA||_F ||v||)."""
    from oracle import probes
    rng = np.random.default_rng(12345)
    SA = np.asarray(SA, np.float64)
    worst = 0.0
    for _ in range(nprobe):
        w = rng.standard_normal(cfg.m)
        v = rng.standard_normal(cfg.d)
        lhs = float(w @ (SA @ v))
        Av = Av_of(v)
        rhs = (probes.probe_rht if cfg.hd else probes.probe_dense)(cfg.seed, cfg.n, cfg.m, cfg.s, w, Av)
        worst = max(worst, abs(lhs - rhs) / (np.linalg.norm(w) * np.linalg.norm(SA) * np.linalg.norm(v)))
    return worst


@pytest.mark.parametrize("name", ["C2", "C3", "C3HD", "C4", "C5"])
def test_freivalds_full_size(name):
    import bench
    from synth import configs, gen
    cfg = configs.ALL[name]
    layout = bench.default_layout(cfg)
    step, inputs = bench.build_step(cfg, torch, layout)
    SA, Sb = step.run()
    torch.cuda.synchronize()
    SA = SA.cpu().numpy()
    if layout == "col" and cfg.kind != "csr":
        SA = SA.T
    if cfg.kind == "csr":
        import scipy.sparse as sp
        rp, ci, v = gen.csr(cfg)
        A = sp.csr_matrix((v, ci, rp), shape=(cfg.n, cfg.d))
        Av_of = lambda x: A @ x  # noqa: E731
    else:
        X = inputs[0]  # device A (row-major n x d) or A^T (d x n) for the column-major layout
        if layout == "col":
            Av_of = lambda x: torch.mv(X.t(), torch.from_numpy(x).to(X.device)).cpu().numpy()  # noqa: E731
        else:
            Av_of = lambda x: torch.mv(X, torch.from_numpy(x).to(X.device)).cpu().numpy()  # noqa: E731
    worst = freivalds(cfg, SA, Av_of)
    assert worst <= 1e-12, f"{name}: Freivalds residual {worst:.3e}"
    assert np.isfinite(SA).all()
    del step, inputs
    torch.cuda.empty_cache()


def test_freivalds_detects_a_wrong_sketch():
    """The probe is sharp: one flipped sign of one bucket entry fails it."""
    from oracle import sketch
    from synth import configs, gen
    cfg = configs.C1
    A = gen.dense(cfg)
    SA, _ = sketch.sketch_dense(cfg.seed, A, None, cfg.m, cfg.s)
    assert freivalds(cfg, SA, lambda x: A @ x) <= 1e-13
    bad = SA.copy()
    bad[7] = -bad[7]
    assert freivalds(cfg, bad, lambda x: A @ x) > 1e-6
