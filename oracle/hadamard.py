"""The randomised Walsh-Hadamard mix H D (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Def. ``def::HRHT``: S = S_h H D with
  * D a random n x n diagonal matrix with +-1 independent entries;
  * H the n x n Walsh-Hadamard matrix
        H_ij = n^{-1/2} (-1)^{<(i-1)_2, (j-1)_2>}
    where (i-1)_2 is the binary digit vector of i-1 (footnote: (3)_2 = (1,1)).
  * S_h an s-hashing matrix independent of D.

DESIGN.md readings:
  R2  0-based: H_ij = n^{-1/2} (-1)^{popcount(i & j)}  (natural / Sylvester
      order, not sequency order).
  R7  D_i = -1 iff bit (i & 63) of u(key_DIAG, i >> 6) is set (global row i).
  R8  n not a power of two: pad with zero rows to n_pad = 2^ceil(log2 n)
      (S:L221); D is irrelevant on padded rows (they are zero).
  R9  fast transform: unnormalised radix-2 butterflies, stage h = 1, 2, 4, ...
      (low bit to high bit), (x_i, x_{i+h}) <- (x_i + x_{i+h}, x_i - x_{i+h})
      for i with bit h clear; the normalisation n^{-1/2} is applied once at the
      end (c_n = 1.0 / sqrt(float(n_pad))).
"""
import math

import numpy as np

from . import rng


def next_pow2(n):
    """Smallest power of two >= n (R8)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    return 1 << (n - 1).bit_length()


def c_n(n_pad):
    """Normalisation n^{-1/2} of H."""
    return 1.0 / math.sqrt(float(n_pad))


def hadamard_formula(n):
    """H entrywise from the P:L796 formula, via explicit binary digit vectors."""
    k = n.bit_length() - 1
    if n != 1 << k:
        raise ValueError("n must be a power of two")
    H = np.empty((n, n), dtype=np.float64)
    for i in range(n):
        bi = [(i >> t) & 1 for t in range(k)]  # (i)_2, little-endian digits
        for j in range(n):
            bj = [(j >> t) & 1 for t in range(k)]
            dot = sum(x * y for x, y in zip(bi, bj))
            H[i, j] = (-1.0) ** dot
    return H / math.sqrt(n)


def hadamard_sylvester(n):
    """Unnormalised Sylvester recursion: H_1 = [1], H_2k = [[H, H], [H, -H]]."""
    k = n.bit_length() - 1
    if n != 1 << k:
        raise ValueError("n must be a power of two")
    H = np.ones((1, 1), dtype=np.float64)
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H


def diag_signs(seed, row_ids):
    """D_i for global rows ``row_ids`` as +-1 int8 (reading R7)."""
    row_ids = np.asarray(row_ids, dtype=np.uint64)
    w = rng.u_np(rng.key_diag(seed), row_ids >> np.uint64(6))
    bit = (w >> (row_ids & np.uint64(63))) & np.uint64(1)
    return np.where(bit == 1, -1, 1).astype(np.int8)


def diag_sign_scalar(seed, i):
    """D_i for one global row, pure Python (tier 0)."""
    w = rng.u(rng.key_diag(seed), i >> 6)
    return -1 if (w >> (i & 63)) & 1 else 1


def fwht_stages(X, bit_lo, bit_hi):
    """Apply the unnormalised butterfly stages for bits [bit_lo, bit_hi) along
    axis 0 of X (in place, low bit first, reading R9).  len(X) must be a
    multiple of 2^bit_hi."""
    if not X.flags.c_contiguous:
        raise ValueError("fwht_stages works in place on a C-contiguous array")
    n = X.shape[0]
    for bit in range(bit_lo, bit_hi):
        h = 1 << bit
        if n % (2 * h):
            raise ValueError("length not a multiple of 2^(bit+1)")
        V = X.reshape(n // (2 * h), 2, h, *X.shape[1:])
        a = V[:, 0].copy()
        b = V[:, 1]
        V[:, 0] = a + b
        V[:, 1] = a - b
    return X


def fwht(X):
    """Unnormalised H_hat X along axis 0 (all stages); X is copied."""
    X = np.array(X, dtype=np.float64, copy=True)
    n = X.shape[0]
    k = n.bit_length() - 1
    if n != 1 << k:
        raise ValueError("length must be a power of two")
    return fwht_stages(X, 0, k)


def hd(seed, A, n_pad=None, row0=0):
    """Unnormalised H_hat D [A; 0] for a block of columns (rows are global
    row0 .. row0+n-1, zero-padded to n_pad)."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    if n_pad is None:
        n_pad = next_pow2(n)
    X = np.zeros((n_pad,) + A.shape[1:], dtype=np.float64)
    sg = diag_signs(seed, np.arange(row0, row0 + n)).astype(np.float64)
    X[:n] = A * (sg if A.ndim == 1 else sg[:, None])
    return fwht(X)
