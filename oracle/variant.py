"""The s-hashing VARIANT matrix T (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definition ``def::s-hashing-variant`` ("Def. 7"): "T in R^{m x n}
is an s-hashing variant matrix if independently for each j in [n], we sample
with replacement i_1, i_2, ..., i_s in [m] uniformly at random and add
+-1/sqrt(s) to T_{i_k j}, where k = 1, 2, ..., s" (footnote: "we may have
i_k = i_l for some l < k").  Lemma ``decompose_s_hashing_varaint`` ("Lemma 8",
P:L693-718): T = s^{-1/2} (S^(1) + ... + S^(s)) with S^(k) independent
1-hashing matrices.

DESIGN.md readings used here:
  R1-R4 as for oracle/hashing.py (same generator and key), except that
        "with replacement" keeps every draw: draw k of column j is
        r_k = mulhi(u(key_HASH, j * 2^16 + k), m) for k = 0..s-1 (no rejection),
        its sign is bit k of u(key_HASH, j * 2^16 + 0xFFFF).  With s = 1 the draw
        equals the 1-hashing draw of oracle/hashing.py ("Both ... reduce
        to 1-hashing matrices when s = 1").
  R18   sketches of T: T A = c_s * (sum over the draws (j, k) with r_k(j) = b of
        sigma_k(j) A[j]) per bucket b, i.e. Lemma 8's sum of the s 1-hashing
        sketches written draw by draw.  Summation order: ascending j; the draws
        of one column into the same bucket (coincident draws) are adjacent,
        + before -.  So the bucket lists are those of oracle/hashing.py with
        repeated (bucket, row) entries allowed, and ``sketch.bucket_sum``
        evaluates them unchanged.
"""
import math

import numpy as np

from . import hashing, rng


def check_args(m, s):
    """Def. 7 needs s <= m only through SPEC; 1 <= s <= 64 (one sign word)."""
    hashing.check_args(m, s)


# ------------------------------------------------------------------ tier 0
def draw_column(seed, j, m, s):
    """Rows and signs of column j of T, pure Python, in draw order (Def. 7)."""
    check_args(m, s)
    key = rng.key_hash(seed)
    rows = [rng.mulhi(rng.u(key, (j << 16) + k), m) for k in range(s)]
    w = rng.u(key, (j << 16) + hashing.SIGN_SLOT)
    signs = [-1 if (w >> k) & 1 else 1 for k in range(s)]
    return rows, signs


def dense_T(seed, n, m, s):
    """T as a dense m x n matrix, built exactly as Def. 7 states: for each j, for
    each k, add sigma_k / sqrt(s) to T[i_k, j]."""
    T = np.zeros((m, n), dtype=np.float64)
    c = hashing.c_s(s)
    for j in range(n):
        rows, signs = draw_column(seed, j, m, s)
        for r, sg in zip(rows, signs):
            T[r, j] += sg * c
    return T


def dense_T_lemma8(seed, n, m, s):
    """T by Lemma 8 with the loops swapped: for each k, the 1-hashing
    matrix S^(k) of draw k over all columns; T = s^{-1/2} (S^(1) + ... + S^(s)).
    Integer accumulation first (exact), one scale at the end."""
    check_args(m, s)
    key = rng.key_hash(seed)
    acc = np.zeros((m, n), dtype=np.int64)
    for k in range(s):
        Sk = np.zeros((m, n), dtype=np.int64)
        for j in range(n):
            r = rng.mulhi(rng.u(key, (j << 16) + k), m)
            w = rng.u(key, (j << 16) + hashing.SIGN_SLOT)
            Sk[r, j] = -1 if (w >> k) & 1 else 1
        acc += Sk
    return acc.astype(np.float64) * hashing.c_s(s)


# ------------------------------------------------------------------ tier 1
def draw_columns(seed, cols, m, s):
    """Vectorised draw_column: (rows int64, signs int8), shape (len(cols), s)."""
    check_args(m, s)
    cols = np.asarray(cols, dtype=np.uint64)
    key = rng.key_hash(seed)
    base = cols << np.uint64(16)
    rows = np.stack([rng.mulhi_np(rng.u_np(key, base + np.uint64(k)), m).astype(np.int64) for k in range(s)],
                    axis=1).reshape(len(cols), s)
    w = rng.u_np(key, base + np.uint64(hashing.SIGN_SLOT))
    bits = (w[:, None] >> np.arange(s, dtype=np.uint64)[None, :]) & np.uint64(1)
    signs = np.where(bits == 1, -1, 1).astype(np.int8)
    return rows, signs


def bucket_lists(seed, row_ids, m, s):
    """Bucket lists of T over the given global rows (reading R18): entries sorted
    by (bucket, global row, sign with + first); a coincident draw repeats its row."""
    row_ids = np.asarray(row_ids, dtype=np.int64)
    rows, signs = draw_columns(seed, row_ids, m, s)
    b = rows.reshape(-1)
    local = np.repeat(np.arange(len(row_ids)), s)
    gid = np.repeat(row_ids, s)
    sg = signs.reshape(-1)
    perm = np.lexsort((sg < 0, gid, b))  # last key is primary: bucket, then row, then + before -
    counts = np.bincount(b, minlength=m)
    ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    return ptr, local[perm], sg[perm]


def sketch_dense(seed, A, b, m, s, buckets=None):
    """T A and T b (tier 1, reading R18)."""
    from . import sketch
    A = np.asarray(A, dtype=np.float64)
    ptr, rows, signs = bucket_lists(seed, np.arange(A.shape[0]), m, s)
    c = hashing.c_s(s)
    TA = sketch.bucket_sum(A, ptr, rows, signs, c, buckets)
    Tb = None if b is None else sketch.bucket_sum(np.asarray(b, np.float64), ptr, rows, signs, c, buckets)
    return TA, Tb


def distinct_fraction_exact(m, s):
    """P(all s draws of a column distinct) = prod_{i<s} (m - i) / m (birthday)."""
    return math.prod((m - i) / m for i in range(s))
