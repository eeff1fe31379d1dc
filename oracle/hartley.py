"""The HR-DHT sketch S = S_h F D (eq. ``eqn::HR-DHT``, "(6.1)"),
oracle side: the sketch the paper's dense solver actually uses.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

"F is a matrix representing the normalized Discrete Hartley Transform (DHT),
defined as F_ij = sqrt(1/n) [cos(2 pi (i-1)(j-1)/n) + sin(2 pi (i-1)(j-1)/n)]"
(P:L1071-1072); D is the random sign diagonal of Def. def::HRHT; S_h
the s-hashing matrix.  The DHT handles any n, so there
is no padding: S_h hashes the n rows.

DESIGN.md readings: R2 0-based indices (F_ij with (i-1)(j-1) -> ij); R7 D as
for the HRHT path; R20 the unnormalised transform Fhat = sqrt(n) F is applied
and the sketch is scaled once by c = 1/sqrt(n s) (as R10 for the HRHT); tier 1
computes Fhat x as Re(X) - Im(X) of the DFT X_k = sum_j x_j exp(-2 pi i jk/n)
(numpy.fft, a library primitive used as one step: cos(t) + sin(t) =
Re(e^{-it}) - Im(e^{-it})).
"""
import math

import numpy as np

from . import hadamard, hashing, sketch


def dht_matrix(n):
    """F of eq. (6.1) written out entrywise (tier 0), 0-based."""
    ij = np.outer(np.arange(n), np.arange(n)).astype(np.float64)
    t = 2.0 * math.pi * ((ij % n) / n)
    return (np.cos(t) + np.sin(t)) / math.sqrt(n)


def dht_unnormalised(X):
    """Fhat X = sqrt(n) F X along axis 0 via the DFT (tier 1, reading R20)."""
    X = np.asarray(X, np.float64)
    Z = np.fft.fft(X, axis=0)
    return Z.real - Z.imag


def fd(seed, A):
    """Fhat D A (unnormalised), any n."""
    A = np.asarray(A, np.float64)
    sg = hadamard.diag_signs(seed, np.arange(A.shape[0])).astype(np.float64)
    return dht_unnormalised(A * (sg if A.ndim == 1 else sg[:, None]))


def hrdht_sketch(seed, A, b, m, s, buckets=None):
    """SA = S_h F D A, Sb = S_h F D b: ascending-row signed sums of Fhat D A rows
    per bucket, times c = 1/sqrt(n s) (readings R10, R20)."""
    A = np.asarray(A, np.float64)
    n = A.shape[0]
    X = fd(seed, A)
    ptr, rows, signs = hashing.bucket_lists(seed, np.arange(n), m, s)
    c = 1.0 / math.sqrt(float(n) * float(s))
    SA = sketch.bucket_sum(X, ptr, rows, signs, c, buckets)
    Sb = None
    if b is not None:
        Sb = sketch.bucket_sum(fd(seed, np.asarray(b, np.float64)), ptr, rows, signs, c, buckets)
    return SA, Sb


def hrdht_sketch_dense_S(seed, A, b, m, s):
    """Tier 0: S_h (dense) @ F (explicit eq. (6.1)) @ D @ A."""
    A = np.asarray(A, np.float64)
    n = A.shape[0]
    Dv = hadamard.diag_signs(seed, np.arange(n)).astype(np.float64)
    S = hashing.dense_S(seed, n, m, s)
    F = dht_matrix(n)
    SA = S @ (F @ (Dv[:, None] * A))
    Sb = None if b is None else S @ (F @ (Dv * np.asarray(b, np.float64)))
    return SA, Sb
