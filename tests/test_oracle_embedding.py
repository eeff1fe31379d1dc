"""Statistical pins for the sketch: the subspace-embedding property (Def.
subspace_embedding_def1_statement; R11), the coherent
negative control and Algorithm 1's use of SA."""
import math

import numpy as np
import scipy.sparse.linalg

from oracle import sketch
from synth import configs, gen


def sv_band(d, m, slack=0.05):
    q = math.sqrt(d / m)
    return 1 - q - slack, 1 + q + slack


def test_embedding_C1_full_size():
    cfg = configs.C1
    A = gen.dense(cfg)
    U, _ = np.linalg.qr(A)
    SU, _ = sketch.sketch_dense(cfg.seed, U, None, cfg.m, cfg.s)
    sv = np.linalg.svd(SU, compute_uv=False)
    lo, hi = sv_band(cfg.d, cfg.m)
    assert lo <= sv.min() and sv.max() <= hi


def test_embedding_C2_replica_with_hd():
    cfg = configs.C2.scaled(n=8192, d=128, m=224)
    U, _ = np.linalg.qr(gen.dense(cfg))
    SU, _ = sketch.rht_sketch(cfg.seed, U, None, cfg.m, cfg.s)
    sv = np.linalg.svd(SU, compute_uv=False)
    lo, hi = sv_band(cfg.d, cfg.m)
    assert lo <= sv.min() and sv.max() <= hi


def test_coherent_negative_control_and_hd_recovery():
    """Coherent A (C3 structure, scaled): s=2 hashing alone loses rank at
    m = 1.75 d (Example 1 / P:L1376-1377); with H D it embeds."""
    cfg = configs.C3.scaled(n=4096, d=256, m=448)
    A = gen.dense(cfg)
    U, _ = np.linalg.qr(A)
    SU, _ = sketch.sketch_dense(cfg.seed, U, None, cfg.m, cfg.s)
    sv = np.linalg.svd(SU, compute_uv=False)
    assert sv.min() < 0.05
    SUh, _ = sketch.rht_sketch(cfg.seed, U, None, cfg.m, cfg.s)
    svh = np.linalg.svd(SUh, compute_uv=False)
    lo, hi = sv_band(cfg.d, cfg.m)
    assert lo <= svh.min() and svh.max() <= hi


def test_sketch_preconditioned_lsqr_matches_normal_equations():
    """Algorithm 1 Steps 2-5 on a C1-shaped problem: QR of SA gives R; LSQR on
    W = A R^{-1} converges to the normal-equations solution, within
    the iteration bound of the rate-of-convergence result."""
    cfg = configs.C1
    A = gen.dense(cfg)
    b = gen.rhs(cfg)
    SA, Sb = sketch.sketch_dense(cfg.seed, A, b, cfg.m, cfg.s)
    Q, R = np.linalg.qr(SA)
    x_s = np.linalg.solve(R, Q.T @ Sb)                  # Step 3 sketched solution
    Rinv = np.linalg.inv(R)
    W = A @ Rinv
    res = scipy.sparse.linalg.lsqr(W, b, atol=1e-14, btol=1e-14, iter_lim=1000)
    x = Rinv @ res[0]
    x_ne = np.linalg.solve(A.T @ A, A.T @ b)
    assert np.linalg.norm(x - x_ne) / np.linalg.norm(x_ne) < 1e-10
    # kappa(W) small: SA embeds A (P:L1707 with the measured epsilon)
    sv = np.linalg.svd(W, compute_uv=False)
    kappa = sv.max() / sv.min()
    assert kappa < 4
    eps = (kappa ** 2 - 1) / (kappa ** 2 + 1)          # kappa(W^T W) = (1+e)/(1-e)
    bound = math.ceil((math.log(2) + abs(math.log(1e-14))) / abs(math.log(eps))) + 2
    assert res[2] <= bound * 2
    # explicit-sketching guarantee: ||A x_s - b|| <= (1+e)/(1-e) ||A x* - b||
    r_s = np.linalg.norm(A @ x_s - b)
    r_star = np.linalg.norm(A @ x_ne - b)
    assert r_s <= (1 + eps) / (1 - eps) * r_star * (1 + 1e-12)
