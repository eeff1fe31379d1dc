"""Pins for oracle/lls.py: Algorithm 1 Steps 2-5 with LSQR (Paige &
Saunders) and the (7.1) stopping rule."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg

from oracle import hashing, lls, sketch


def problem(n=3000, d=40, m=120, s=2, seed=3, noise=1.0, cond=1e3):
    r = np.random.default_rng(seed)
    U, _ = np.linalg.qr(r.standard_normal((n, d)))
    V, _ = np.linalg.qr(r.standard_normal((d, d)))
    A = (U * np.logspace(0, -math.log10(cond), d)) @ V.T
    x_true = r.standard_normal(d)
    b = A @ x_true + noise * r.standard_normal(n)
    SA, Sb = sketch.sketch_dense(seed, A, b, m, s)
    return A, b, SA, Sb


def test_lsqr_matches_scipy_lsqr():
    """Independent implementation: scipy's LSQR with only its test 2 active
    (atol = tau_r, btol = 0, conlim = 0) stops at the same iteration with the
    same iterate (inconsistent system, so test 1 cannot fire)."""
    A, b, SA, Sb = problem()
    Q, R = lls.qr_sketch(SA)
    W = A @ np.linalg.inv(R)
    for tau in (1e-4, 1e-6, 1e-9):
        y, it, test2, rnorm = lls.lsqr(lambda v: W @ v, lambda u: W.T @ u, b, tau, 1000)
        ref = scipy.sparse.linalg.lsqr(W, b, atol=tau, btol=0.0, conlim=0.0, iter_lim=1000)
        assert ref[1] == 2 and ref[2] == it
        assert np.linalg.norm(y - ref[0]) <= 1e-9 * np.linalg.norm(ref[0])  # rotations computed differently
        assert abs(rnorm - ref[3]) <= 1e-12 * ref[3]


def test_estimates_are_exact_quantities():
    """At exit, phibar = ||W y - b|| and alpha |s phi| = ||W^T (W y - b)||
    (Paige & Saunders' recurrences), so test2 is the (7.1) ratio with ||W||
    replaced by the running Frobenius estimate (<= ||W||_F)."""
    A, b, SA, Sb = problem(seed=5)
    Q, R = lls.qr_sketch(SA)
    W = A @ np.linalg.inv(R)
    y, it, test2, rnorm = lls.lsqr(lambda v: W @ v, lambda u: W.T @ u, b, 1e-6, 1000)
    r = W @ y - b
    assert abs(rnorm - np.linalg.norm(r)) <= 1e-8 * np.linalg.norm(r)
    exact = np.linalg.norm(W.T @ r) / (np.linalg.norm(r))
    anorm_f = np.linalg.norm(W, "fro")
    assert test2 <= 1e-6
    assert exact / anorm_f <= test2 * 1.0001  # Frobenius estimate <= ||W||_F


def test_converged_solution_is_least_squares():
    """tau_r -> 0: x_tau is the least-squares solution (numpy lstsq, closed form)."""
    A, b, SA, Sb = problem(seed=7)
    x, info = lls.solve(A, b, SA, Sb, tau_a=0.0, tau_r=1e-15, it_max=500)
    xs = np.linalg.lstsq(A, b, rcond=None)[0]
    assert info["step"] == 4
    assert np.linalg.norm(x - xs) <= 1e-8 * np.linalg.norm(xs)


def test_step3_exit_on_consistent_system():
    """b = A x exactly: x_s (Step 3) already solves it, ||A x_s - b|| <= tau_a."""
    A, b, SA, Sb = problem(seed=9, noise=0.0)
    x, info = lls.solve(A, b, SA, Sb, tau_a=1e-8)
    assert info["step"] == 3 and info["iters"] == 0
    assert np.linalg.norm(A @ x - b) <= 1e-8


def test_iteration_bound_from_condition_number():
    """LSQR error decays like 2((sqrt k - 1)/(sqrt k + 1))^j with
    k = kappa(W^T W); the (7.1) test fires within a few iterations of that bound."""
    A, b, SA, Sb = problem(n=4000, d=60, m=110, s=1, seed=11)
    x, info = lls.solve(A, b, SA, Sb)
    R = info["R"]
    sv = np.linalg.svd(A @ np.linalg.inv(R), compute_uv=False)
    k = (sv[0] / sv[-1]) ** 2
    rate = (math.sqrt(k) - 1) / (math.sqrt(k) + 1)
    bound = math.log(1e-6 / 2) / math.log(rate)
    assert info["iters"] <= math.ceil(bound) + 3


def test_explicit_and_lsqr_residual_bounds():
    """with eps the embedding distortion of S on
    range([A b]) (squared singular values of S U in [1 - eps, 1 + eps]),
    ||A x_s - b|| <= (1+eps)/(1-eps) ||A x* - b|| and
    ||A x_tau - b|| <= (1 + 2 eps tau_r/(1-eps)) ||A x* - b||."""
    n, d, m, s, seed = 3000, 20, 400, 2, 13
    A, b, SA, Sb = problem(n=n, d=d, m=m, s=s, seed=seed)
    U, _ = np.linalg.qr(np.column_stack([A, b]))
    SU, _ = sketch.sketch_dense(seed, U, None, m, s)
    sv = np.linalg.svd(SU, compute_uv=False)
    eps = max(sv[0] ** 2 - 1, 1 - sv[-1] ** 2)
    assert eps < 1
    best = np.linalg.norm(A @ np.linalg.lstsq(A, b, rcond=None)[0] - b)
    x, info = lls.solve(A, b, SA, Sb, tau_a=0.0)
    assert info["res_s"] <= (1 + eps) / (1 - eps) * best * (1 + 1e-12)
    assert np.linalg.norm(A @ x - b) <= (1 + 2 * eps * 1e-6 / (1 - eps)) * best * (1 + 1e-12)


def test_hashing_preconditioner_at_paper_m():
    """Default m = 1.7 d with s = 1 after H D: the preconditioned system
    is well conditioned (kappa(W) modest) and LSQR needs few iterations."""
    r = np.random.default_rng(1)
    n, d = 4096, 64
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    m = int(1.7 * d)
    SA, Sb = sketch.rht_sketch(2, A, b, m, 1)
    x, info = lls.solve(A, b, SA, Sb)
    assert info["step"] == 4 and info["iters"] < 60
    assert hashing.c_s(1) == 1.0


# ------------------------------------------------------------------ R-CPQR mode
def deficient(n=2500, d=30, r=18, m=100, s=2, seed=11):
    """A of exact rank r < d: r independent columns and d - r combinations of them."""
    g = np.random.default_rng(seed)
    B = g.standard_normal((n, r))
    C = g.standard_normal((r, d - r))
    A = np.concatenate([B, B @ C], axis=1)[:, g.permutation(d)]
    b = g.standard_normal(n)
    SA, Sb = sketch.sketch_dense(seed, A, b, m, s)
    return A, b, SA, Sb, r


def test_cpqr_rank_and_factorisation():
    """SA P = Q R~ exactly (to rounding); the detected p equals rank(A) for an
    exactly rank-deficient A (S is an embedding at m = 100 >> r); r~_qq beyond
    p are at the rounding level and non-increasing |r~_qq| (Businger-Golub)."""
    A, b, SA, Sb, r = deficient()
    Q1, R11, piv, p = lls.cpqr_sketch(SA, 1e-12)
    assert p == r == np.linalg.matrix_rank(A)
    Q, R, piv2 = __import__("scipy.linalg").linalg.qr(SA, mode="economic", pivoting=True)
    assert np.allclose(SA[:, piv2], Q @ R, atol=1e-12 * np.linalg.norm(SA))
    dg = np.abs(np.diag(R))
    assert np.all(dg[1:] <= dg[:-1] * (1 + 1e-12))
    assert dg[p - 1] >= 1e-12 > dg[p] if p < len(dg) else True


def test_cpqr_solve_reaches_the_least_squares_residual():
    """Rank-deficient A: x is not unique, but the objective is.  The R-CPQR solve
    reaches the minimum residual of numpy's minimum-norm lstsq (the
    solution is optimal over the detected column space), and x_tau lies in the
    span of the p pivoted coordinates."""
    A, b, SA, Sb, r = deficient(seed=12)
    x, info = lls.solve(A, b, SA, Sb, tau_a=0.0, tau_r=1e-14, it_max=500, rcond=1e-12)
    xm = np.linalg.lstsq(A, b, rcond=None)[0]
    rmin = np.linalg.norm(A @ xm - b)
    assert info["rank"] == r and info["step"] == 4
    assert abs(np.linalg.norm(A @ x - b) - rmin) <= 1e-10 * rmin
    Q1, R11, piv, p = lls.cpqr_sketch(SA, 1e-12)
    assert np.all(x[piv[p:]] == 0.0)


def test_cpqr_equals_qr_mode_on_full_rank():
    """Full-rank A: both Step-2 modes precondition the same problem and converge
    to its unique least-squares solution."""
    A, b, SA, Sb = problem(seed=13)
    x1, i1 = lls.solve(A, b, SA, Sb, tau_a=0.0, tau_r=1e-15, it_max=500)
    x2, i2 = lls.solve(A, b, SA, Sb, tau_a=0.0, tau_r=1e-15, it_max=500, rcond=1e-12)
    assert i2["rank"] == A.shape[1]
    assert np.linalg.norm(x1 - x2) <= 1e-8 * np.linalg.norm(x1)


def test_cpqr_rcond_truncates_small_diagonals():
    """rcond above the smallest |r~_qq| drops exactly the trailing pivots below it."""
    A, b, SA, Sb = problem(seed=14, cond=1e8)
    Q, R, piv = __import__("scipy.linalg").linalg.qr(SA, mode="economic", pivoting=True)
    dg = np.abs(np.diag(R))
    rc = float(np.sqrt(dg[-3] * dg[-2]))  # between the 3rd- and 2nd-last
    assert lls.cpqr_sketch(SA, rc)[3] == len(dg) - 2
