"""The s-hashing matrix S (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definition ``def::sampling_and_hashing``: "S in R^{m x n} is a
s-hashing matrix if independently for each j in [n], we sample without
replacement i_1, i_2, ..., i_s in [m] uniformly at random and let
S_{i_k j} = +-1/sqrt(s) for k = 1, ..., s."  s = 1 is the 1-hashing matrix
(P:L272).

DESIGN.md readings used here:
  R1  generator: rng.u on key_hash(seed)
  R2  0-based indices (the paper's [n] = {1..n})
  R3  "without replacement" = rejection of duplicates: attempt t = 0, 1, ...
      draws r_t = mulhi(u(key_HASH, j * 2^16 + t), m); r_t is accepted when it
      differs from the rows already accepted for column j; stop after s
      acceptances.  t <= 2^16 - 2, otherwise the draw fails (SKH_ERETRY).
  R4  signs independent of rows: w = u(key_HASH, j * 2^16 + 0xFFFF); the k-th
      accepted row has sign -1 iff bit k of w is set (so s <= 64).
  R5  value of an entry: sigma * c_s with c_s = 1.0 / sqrt(float(s)) (IEEE sqrt
      then IEEE divide); sketches scale the exact signed sum once at the end.
  R6  bucket lists (the CSR form of S): for bucket b, the columns j with a
      nonzero in row b, in ascending j.  Unique because a column hits a bucket at
      most once.
"""
import math

import numpy as np

from . import rng

MAX_ATTEMPTS = 0xFFFF  # attempts t = 0 .. 0xFFFE; 0xFFFF is the sign word
SIGN_SLOT = 0xFFFF


def check_args(m, s):
    """Argument rules of the hash: 1 <= s <= m, s <= 64."""
    if m < 1 or s < 1 or s > m:
        raise ValueError(f"need 1 <= s <= m (m={m}, s={s})")
    if s > 64:
        raise ValueError("s > 64 unsupported (one 64-bit sign word per column, R4)")
    if m >= (1 << 31):
        raise ValueError("m must fit in int32")


def c_s(s):
    """Entry magnitude 1/sqrt(s) of Def. def::sampling_and_hashing."""
    return 1.0 / math.sqrt(float(s))


# ------------------------------------------------------------------ tier 0
def draw_column(seed, j, m, s):
    """Rows and signs of column j of S, pure Python (reading R3/R4).

    Returns (rows, signs): lists of length s, rows distinct in [0, m), signs in
    {+1, -1}, in acceptance order.
    """
    check_args(m, s)
    key = rng.key_hash(seed)
    rows = []
    t = 0
    while len(rows) < s:
        if t >= MAX_ATTEMPTS:
            raise RuntimeError(f"column {j}: rejection attempts exhausted")
        r = rng.mulhi(rng.u(key, (j << 16) + t), m)
        if r not in rows:
            rows.append(r)
        t += 1
    w = rng.u(key, (j << 16) + SIGN_SLOT)
    signs = [-1 if (w >> k) & 1 else 1 for k in range(s)]
    return rows, signs


def dense_S(seed, n, m, s):
    """S as a dense m x n float64 matrix, one column at a time (tier 0)."""
    S = np.zeros((m, n), dtype=np.float64)
    c = c_s(s)
    for j in range(n):
        rows, signs = draw_column(seed, j, m, s)
        for r, sg in zip(rows, signs):
            S[r, j] = sg * c
    return S


# ------------------------------------------------------------------ tier 1
def draw_columns(seed, cols, m, s):
    """Vectorised ``draw_column`` for an array of global column ids.

    Returns (rows, signs) of shape (len(cols), s): int64 rows and int8 signs in
    acceptance order.  Same rule as draw_column, applied to all columns at once.
    """
    check_args(m, s)
    cols = np.asarray(cols, dtype=np.uint64)
    ncols = cols.shape[0]
    key = rng.key_hash(seed)
    rows = np.full((ncols, s), -1, dtype=np.int64)
    nacc = np.zeros(ncols, dtype=np.int64)
    base = cols << np.uint64(16)
    active = np.arange(ncols)
    t = 0
    while active.size:
        if t >= MAX_ATTEMPTS:
            raise RuntimeError("rejection attempts exhausted")
        r = rng.mulhi_np(rng.u_np(key, base[active] + np.uint64(t)), m).astype(np.int64)
        dup = (rows[active] == r[:, None]).any(axis=1)
        acc = active[~dup]
        rows[acc, nacc[acc]] = r[~dup]
        nacc[acc] += 1
        active = active[nacc[active] < s]
        t += 1
    w = rng.u_np(key, base + np.uint64(SIGN_SLOT))
    bits = (w[:, None] >> np.arange(s, dtype=np.uint64)[None, :]) & np.uint64(1)
    signs = np.where(bits == 1, -1, 1).astype(np.int8)
    return rows, signs


def bucket_lists(seed, row_ids, m, s):
    """Bucket lists (CSR of S restricted to the given columns), reading R6.

    ``row_ids`` are the global column ids of S (= global rows of A) held
    locally, in local order 0..len-1.  Returns (bucket_ptr[m+1] int64,
    bucket_rows int64 LOCAL positions, bucket_signs int8), with rows ascending
    in global id inside every bucket (a stable sort of the entries by bucket,
    the entries being listed in ascending global id).
    """
    row_ids = np.asarray(row_ids, dtype=np.int64)
    order = np.argsort(row_ids, kind="stable")  # ascending global id
    rows, signs = draw_columns(seed, row_ids[order], m, s)
    local = np.repeat(order, s)
    b = rows.reshape(-1)
    sg = signs.reshape(-1)
    perm = np.argsort(b, kind="stable")
    counts = np.bincount(b, minlength=m)
    ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    return ptr, local[perm], sg[perm]


def triples(seed, n, m, s):
    """S as explicit (bucket, column, value) triples (materialised S, BJ)."""
    rows, signs = draw_columns(seed, np.arange(n), m, s)
    c = c_s(s)
    b = rows.reshape(-1)
    j = np.repeat(np.arange(n), s)
    v = signs.reshape(-1).astype(np.float64) * c
    return b, j, v
