"""Freivalds probes: checks of SA at sizes the oracle cannot materialise.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

For any w in R^m and v in R^d,  w^T (S A) v = (S^T w)^T (A v)  (associativity).
The right-hand side needs only the column lists of S (Def.
def::sampling_and_hashing), not the bucket lists, and one
matrix-vector product with A, so it is independent of the transpose and of the
bucket-order summation it checks.  For the HRHT S = S_h H D,
S^T w = D H S_h^T w (H and D are symmetric), one fast transform of an n-vector.
"""
import numpy as np

from . import hadamard, hashing


def st_w(seed, n, m, s, w):
    """(S_h^T w)_i = c_s * sum_k sigma_{ik} w[h_k(i)] for i < n (column lists)."""
    rows, signs = hashing.draw_columns(seed, np.arange(n), m, s)
    w = np.asarray(w, dtype=np.float64)
    return hashing.c_s(s) * (signs.astype(np.float64) * w[rows]).sum(axis=1)


def probe_dense(seed, n, m, s, w, Av):
    """(S^T w)^T (A v) for the plain s-hashing sketch; Av = A @ v (length n)."""
    return float(np.dot(st_w(seed, n, m, s, w), np.asarray(Av, np.float64)))


def probe_rht(seed, n, m, s, w, Av):
    """(D H S_h^T w)^T (A v) for the HRHT sketch; n is the unpadded row count."""
    n_pad = hadamard.next_pow2(n)
    y = st_w(seed, n_pad, m, s, w)                     # S_h^T w, length n_pad
    y = hadamard.c_n(n_pad) * hadamard.fwht(y)          # H S_h^T w
    dsg = hadamard.diag_signs(seed, np.arange(n)).astype(np.float64)
    return float(np.dot(dsg * y[:n], np.asarray(Av, np.float64)))
