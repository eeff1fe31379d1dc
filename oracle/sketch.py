"""Algorithm 1 Step 1: SA and Sb (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

"Randomly draw a sketching matrix S in R^{m x n} from the distribution, compute
the matrix-matrix product SA in R^{m x d} and the matrix-vector product
Sb in R^m" (Alg. 1 Step 1).  S is an s-hashing matrix for
dense and sparse A or the HRHT S_h H D for dense A.

Tier 0 (``*_dense_S``): S materialised as a dense m x n matrix and multiplied by
NumPy (BLAS order: agrees with tier 1 to rounding, not bitwise).

Tier 1 (everything else): the definition written as a sum,
    (SA)[b, :] = sum over nonzeros S[b, i] of S[b, i] * X[i, :],
with the DESIGN.md reading R10 for the rounding order: for every bucket b the
signed rows sigma * X[i, :] are added one at a time in ascending i, starting
from 0.0, and the sum is multiplied once by the constant c (c_s = 1/sqrt(s) for
plain hashing, c_ns = 1/sqrt(n_pad * s) for HRHT).  A sign flip is exact, so
this is the unique IEEE result of "exact-order signed summation, one scale".
"""
import math

import numpy as np

from . import hadamard, hashing


def c_ns(n_pad, s):
    """Combined constant n_pad^{-1/2} s^{-1/2} of S_h H (reading R10)."""
    return 1.0 / math.sqrt(float(n_pad) * float(s))


def bucket_sum(X, ptr, rows, signs, c, buckets=None):
    """out[b] = c * (((0 + s_1 X[r_1]) + s_2 X[r_2]) + ...) over bucket b's list.

    X: (n, d) or (n,) float64; ptr/rows/signs: bucket lists (hashing.bucket_lists).
    ``buckets``: optional subset of bucket ids (default all); returns
    out[len(buckets), ...].
    """
    X = np.asarray(X, dtype=np.float64)
    m = len(ptr) - 1
    if buckets is None:
        buckets = range(m)
    buckets = list(buckets)
    out = np.zeros((len(buckets),) + X.shape[1:], dtype=np.float64)
    for ob, b in enumerate(buckets):
        acc = np.zeros(X.shape[1:], dtype=np.float64)
        for t in range(ptr[b], ptr[b + 1]):
            acc += float(signs[t]) * X[rows[t]]
        out[ob] = c * acc
    return out


def sketch_dense(seed, A, b, m, s, buckets=None):
    """SA, Sb for dense A (n x d) with an s-hashing S (tier 1).  b may be None."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    ptr, rows, signs = hashing.bucket_lists(seed, np.arange(n), m, s)
    c = hashing.c_s(s)
    SA = bucket_sum(A, ptr, rows, signs, c, buckets)
    Sb = None if b is None else bucket_sum(np.asarray(b, np.float64), ptr, rows, signs, c, buckets)
    return SA, Sb


def sketch_dense_S(seed, A, b, m, s):
    """Tier 0: S materialised densely (hashing.dense_S), then S @ A, S @ b."""
    A = np.asarray(A, dtype=np.float64)
    S = hashing.dense_S(seed, A.shape[0], m, s)
    return S @ A, (None if b is None else S @ np.asarray(b, np.float64))


def csr_row(row_ptr, col_idx, val, i, d):
    """Row i of a CSR matrix as a dense length-d vector."""
    x = np.zeros(d, dtype=np.float64)
    lo, hi = int(row_ptr[i]), int(row_ptr[i + 1])
    x[np.asarray(col_idx[lo:hi], dtype=np.int64)] = val[lo:hi]
    return x


def sketch_csr(seed, row_ptr, col_idx, val, d, b, m, s, buckets=None):
    """SA (dense m x d), Sb for CSR A, same summation rule as
    ``bucket_sum`` applied to the rows of A (a missing entry is an exact 0.0,
    so adding it leaves acc unchanged except -0.0 -> +0.0, which cannot occur
    because acc starts at +0.0)."""
    n = len(row_ptr) - 1
    ptr, rows, signs = hashing.bucket_lists(seed, np.arange(n), m, s)
    c = hashing.c_s(s)
    if buckets is None:
        buckets = range(m)
    buckets = list(buckets)
    SA = np.zeros((len(buckets), d), dtype=np.float64)
    for ob, bk in enumerate(buckets):
        acc = np.zeros(d, dtype=np.float64)
        for t in range(ptr[bk], ptr[bk + 1]):
            i = rows[t]
            lo, hi = int(row_ptr[i]), int(row_ptr[i + 1])
            cols = np.asarray(col_idx[lo:hi], dtype=np.int64)
            acc[cols] += float(signs[t]) * val[lo:hi]
        SA[ob] = c * acc
    Sb = None
    if b is not None:
        Sb = bucket_sum(np.asarray(b, np.float64), ptr, rows, signs, c, buckets)
    return SA, Sb


def csr_to_dense(row_ptr, col_idx, val, d):
    n = len(row_ptr) - 1
    A = np.zeros((n, d), dtype=np.float64)
    for i in range(n):
        A[i] = csr_row(row_ptr, col_idx, val, i, d)
    return A


def hda(seed, A):
    """Normalised H D [A; 0] (Def. def::HRHT): c_n * H_hat D A."""
    A = np.asarray(A, dtype=np.float64)
    n_pad = hadamard.next_pow2(A.shape[0])
    return hadamard.c_n(n_pad) * hadamard.hd(seed, A, n_pad)


def rht_sketch(seed, A, b, m, s, buckets=None):
    """SA = S_h H D A and Sb = S_h H D b (tier 1).

    X = H_hat D [A; 0] (unnormalised fast transform, reading R9), hashed over all
    n_pad rows (reading R8), SA[b] = c_ns * (ascending-i signed sum of X rows).
    """
    A = np.asarray(A, dtype=np.float64)
    n_pad = hadamard.next_pow2(A.shape[0])
    X = hadamard.hd(seed, A, n_pad)
    ptr, rows, signs = hashing.bucket_lists(seed, np.arange(n_pad), m, s)
    c = c_ns(n_pad, s)
    SA = bucket_sum(X, ptr, rows, signs, c, buckets)
    Sb = None
    if b is not None:
        Xb = hadamard.hd(seed, np.asarray(b, np.float64), n_pad)
        Sb = bucket_sum(Xb, ptr, rows, signs, c, buckets)
    return SA, Sb


def rht_sketch_dense_S(seed, A, b, m, s):
    """Tier 0: S_h (dense) @ H (Sylvester, normalised) @ D @ [A; 0]."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    n_pad = hadamard.next_pow2(n)
    H = hadamard.hadamard_sylvester(n_pad) / math.sqrt(n_pad)
    Dv = np.array([hadamard.diag_sign_scalar(seed, i) for i in range(n)], dtype=np.float64)
    Ap = np.zeros((n_pad, A.shape[1]), dtype=np.float64)
    Ap[:n] = Dv[:, None] * A
    S = hashing.dense_S(seed, n_pad, m, s)
    SA = S @ (H @ Ap)
    Sb = None
    if b is not None:
        bp = np.zeros(n_pad, dtype=np.float64)
        bp[:n] = Dv * np.asarray(b, np.float64)
        Sb = S @ (H @ bp)
    return SA, Sb


def rht_sketch_columns(seed, column_block, n, m, s, cols):
    """SA[:, cols] of S_h H D A for an A too large to hold: ``column_block(cols)``
    returns A[:, cols] (n x len(cols)).  Columns are independent under both H
    and S_h, so this is rht_sketch restricted to those columns."""
    Ablk = np.asarray(column_block(cols), dtype=np.float64)
    if Ablk.shape[0] != n:
        raise ValueError("column_block returned the wrong number of rows")
    SA, _ = rht_sketch(seed, Ablk, None, m, s)
    return SA
