"""Algorithm 1 Steps 2-5 (the sketch-preconditioned LLS solve), oracle side.
Two Step-2 modes: the full-rank QR mode (below) and the paper's default,
column-pivoted (R-CPQR) with rank truncation (``cpqr_sketch``, ``solve(...,
rcond=...)``).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

"Generic Sketching Algorithm" (Alg. ``alg1``), given SA and Sb from
Step 1 (oracle/sketch.py):
  Step 2  factor SA = Q R V^T.  Reading R19: the full-rank QR mode the paper
          allows "as in Blendenpik, using DGEQRF from LAPACK": V = I,
          p = d, Householder QR (numpy.linalg.qr calls LAPACK dgeqrf / dorgqr).
  Step 3  x_s = V1 R11^{-1} Q1^T Sb (a back-solve, not an inverse: P:L1081);
          terminate if ||A x_s - b||_2 <= tau_a.
  Step 4  y_tau ~ argmin ||W y - b||, W = A V1 R11^{-1}, by LSQR (Paige &
          Saunders 1982, the paper's ref. 10.1145/355984.355989) started at
          y = 0 (reading R19), stopped when the estimate of
          ||W^T (W y_k - b)|| / (||W|| ||W y_k - b||) <= tau_r  (eq. TC-lsqr,
          "(7.1)") or after it_max iterations.
  Step 5  x_tau = V1 R11^{-1} y_tau.
Defaults: tau_a = 1e-8, tau_r = 1e-6, it_max = 1e4.

LSQR below is the bidiagonalisation recurrence of Paige & Saunders written out
step by step (no reorthogonalisation, no damping): ||W|| is their running
Frobenius estimate sqrt(sum alpha^2 + beta^2), ||r|| = phibar and
||W^T r|| = alpha * |s * phi|, exactly the quantities their stopping test 2
uses.
"""
import math

import numpy as np
import scipy.linalg


def qr_sketch(SA):
    """Step 2 (reading R19): SA = Q R with Q (m x d) orthonormal, R (d x d) upper."""
    Q, R = np.linalg.qr(np.asarray(SA, np.float64), mode="reduced")
    return Q, R


def cpqr_sketch(SA, rcond=1e-12):
    """Step 2, the paper's default mode: a column-
    pivoted QR  SA P = Q R~  (LAPACK dgeqp3 via scipy: Businger-Golub
    Householder QR with column pivoting; the paper's R-CPQR randomises the pivot
    choice, reading R22), i.e. SA = Q R~ V^T with V = P, then
        p = max{q : |r~_qq| >= rcond}      (1-based q; rcond absolute, as printed)
    and R11 = R~[:p, :p], Q1 = Q[:, :p], V1 = P[:, :p] (Alg. 1 Step 2, L873-886).
    Returns (Q1, R11, piv, p) with V1 = I[:, piv[:p]]."""
    Q, R, piv = scipy.linalg.qr(np.asarray(SA, np.float64), mode="economic", pivoting=True)
    big = np.nonzero(np.abs(np.diag(R)) >= rcond)[0]
    p = int(big[-1]) + 1 if big.size else 0
    return Q[:, :p], R[:p, :p], piv, p


def solve_R(R, y):
    """R^{-1} y by back-substitution."""
    return scipy.linalg.solve_triangular(R, y, lower=False)


def solve_RT(R, y):
    """R^{-T} y (forward substitution with R^T)."""
    return scipy.linalg.solve_triangular(R, y, trans="T", lower=False)


def lsqr(Wmul, WTmul, b, tau_r, it_max):
    """LSQR on W y = b.  Wmul(v) = W v, WTmul(u) = W^T u.

    Returns (y, iters, test2, rnorm): iters = number of bidiagonalisation steps
    taken; test2 = the (7.1) estimate at exit."""
    b = np.asarray(b, np.float64)
    beta = float(np.linalg.norm(b))
    u = b / beta if beta > 0 else b.copy()
    v = WTmul(u)
    alpha = float(np.linalg.norm(v))
    if alpha > 0:
        v = v / alpha
    y = np.zeros_like(v)
    if beta == 0 or alpha == 0:  # b = 0 or W^T b = 0: y = 0 is optimal
        return y, 0, 0.0, beta
    w = v.copy()
    phibar, rhobar = beta, alpha
    anorm2 = 0.0
    test2 = math.inf
    it = 0
    while it < it_max:
        it += 1
        # bidiagonalisation: beta u = W v - alpha u, alpha v = W^T u - beta v
        u = Wmul(v) - alpha * u
        beta = float(np.linalg.norm(u))
        if beta > 0:
            u = u / beta
        anorm2 = anorm2 + alpha * alpha + beta * beta
        v = WTmul(u) - beta * v
        alpha = float(np.linalg.norm(v))
        if alpha > 0:
            v = v / alpha
        # plane rotation eliminating beta
        rho = math.sqrt(rhobar * rhobar + beta * beta)
        c = rhobar / rho
        s = beta / rho
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        # update y and the search direction w
        y = y + (phi / rho) * w
        w = v - (theta / rho) * w
        rnorm = phibar
        arnorm = alpha * abs(s * phi)
        anorm = math.sqrt(anorm2)
        if rnorm == 0.0:
            test2 = 0.0
            break
        test2 = arnorm / (anorm * rnorm)
        if test2 <= tau_r:
            break
    return y, it, test2, phibar


def solve(A, b, SA, Sb, tau_a=1e-8, tau_r=1e-6, it_max=10000, rcond=None):
    """Algorithm 1 Steps 2-5 for dense A (n x d) given Step 1's SA, Sb.

    rcond None: the full-rank QR mode (R19).  rcond given: the R-CPQR mode
    (``cpqr_sketch``): x_s = V1 R11^{-1} Q1^T Sb (L881), LSQR on
    W = A V1 R11^{-1} (L886-894), x = V1 R11^{-1} y (L896).

    Returns (x, info) with info = {"step": 3 or 4, "iters", "test2", "x_s",
    "res_s" = ||A x_s - b||, "R", "rank"}."""
    A = np.asarray(A, np.float64)
    b = np.asarray(b, np.float64)
    d = A.shape[1]
    if rcond is None:
        Q, R = qr_sketch(SA)
        piv, p = np.arange(d), d
    else:
        Q, R, piv, p = cpqr_sketch(SA, rcond)

    def V1(z):  # V1 z: the first p pivots' coordinates
        x = np.zeros(d)
        x[piv[:p]] = z
        return x

    x_s = V1(solve_R(R, Q.T @ np.asarray(Sb, np.float64)))
    res_s = float(np.linalg.norm(A @ x_s - b))
    info = {"x_s": x_s, "res_s": res_s, "R": R, "rank": p}
    if res_s <= tau_a or p == 0:
        info.update(step=3, iters=0, test2=0.0)
        return x_s, info
    Ap = A[:, piv[:p]]
    y, it, test2, _ = lsqr(lambda v: Ap @ solve_R(R, v), lambda u: solve_RT(R, Ap.T @ u), b, tau_r, it_max)
    info.update(step=4, iters=it, test2=test2)
    return V1(solve_R(R, y)), info
