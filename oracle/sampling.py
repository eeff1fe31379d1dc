"""The SR-DHT sketch S = S_s F D of Blendenpik (eq. ``eq::SR-DHT``, "(7.2)",
P:L1285-1289) and the Fig. 1 experiment, oracle side.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

"S_s in R^{m x n} is a sampling matrix, whose individual rows contain a single
non-zero entry at a random column with value 1"; F, D as in
HR-DHT (oracle/hartley.py).  The paper does not say whether the m columns are
distinct: reading R21 (as SPEC S:L171) draws them independently, with
replacement: row r of S_s selects column j_r = mulhi(u(key_SAMP, r), n),
key_SAMP = mix64(seed ^ 0x53414D50) ("SAMP"), so SA = (F D A)[j_0 .. j_{m-1}].

Fig. 1: coherent A = [I_d; 0] + 1e-8 J (eq. (7.4)),
n = 4000, d = 400; for each m/d, QR of the HR-DHT sketch and of the SR-DHT
sketch (no pivoting) and kappa(A R^{-1}); the claim: hashing reaches a given
kappa at a smaller m than sampling.
"""
import math

import numpy as np

from . import hartley, hashing, lls, rng

LABEL_SAMP = 0x53414D50


def sample_rows(seed, n, m):
    """j_r for r = 0..m-1 (reading R21)."""
    key = rng.mix64(seed ^ LABEL_SAMP)
    return rng.mulhi_np(rng.u_np(key, np.arange(m, dtype=np.uint64)), n).astype(np.int64)


def dense_Ss(seed, n, m):
    """S_s as a dense m x n 0/1 matrix (tier 0)."""
    S = np.zeros((m, n))
    S[np.arange(m), sample_rows(seed, n, m)] = 1.0
    return S


def srdht_sketch(seed, A, b, m):
    """SA = S_s F D A, Sb = S_s F D b: rows j_r of c_n * Fhat D A, c_n = 1/sqrt(n)."""
    A = np.asarray(A, np.float64)
    n = A.shape[0]
    j = sample_rows(seed, n, m)
    c = 1.0 / math.sqrt(float(n))
    SA = c * hartley.fd(seed, A)[j]
    Sb = None if b is None else c * hartley.fd(seed, np.asarray(b, np.float64))[j]
    return SA, Sb


def coherent_A(n, d):
    """Eq. (7.4): [I_d; 0] + 1e-8 J."""
    A = np.full((n, d), 1e-8)
    A[np.arange(d), np.arange(d)] += 1.0
    return A


def kappa_preconditioned(A, SA):
    """kappa(A R^{-1}) with SA = Q R (no pivoting); inf if R is singular."""
    _, R = lls.qr_sketch(SA)
    if np.min(np.abs(np.diag(R))) <= 1e-300:
        return math.inf
    sv = np.linalg.svd(A @ np.linalg.inv(R), compute_uv=False)
    return float(sv[0] / sv[-1]) if sv[-1] > 0 else math.inf


def fig1_point(seed, A, m, s=1):
    """(kappa with HR-DHT, kappa with SR-DHT) at one m."""
    SAh, _ = hartley.hrdht_sketch(seed, A, None, m, s)
    SAs, _ = srdht_sketch(seed, A, None, m)
    assert hashing.c_s(s) > 0
    return kappa_preconditioned(A, SAh), kappa_preconditioned(A, SAs)
