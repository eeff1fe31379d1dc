"""Seeded synthetic inputs (host / NumPy side).

This module is the ONLY code shared by the oracle side (tests, bench's CPU
baseline) and the CUDA side (tests, bench): it produces the inputs A, b of the
BASELINE.json workloads and holds none of the sketch's arithmetic.  The device
generator in ``synth/csrc/synth_gen.cu`` implements the same counter-based
recipe; both are integer-exact (see below) so they agree bit for bit, which
``tests/test_synth.py`` checks.

Recipe.  Every value is a pure function of (seed, label, index):
    mixS(z)        splitmix64 finaliser (this module's own copy)
    word(k, c)     = mixS(k + (c + 1) * GAMMA), k = mixS(seed ^ (label << 32))
    normal(idx)    Irwin-Hall(12) - 6: the 12 uniforms are the 32-bit halves of
                   word(k, 6 idx + t), t = 0..5; the sum of twelve 32-bit
                   integers minus 6 * 2^32 is an exact integer < 2^37, so
                   value = that integer * 2^-32 is exact in fp64 on any
                   platform.  Mean 0, variance 1, support [-6, 6] (the paper's
                   N(0,1) entries; R12 records the
                   substitution).
    uniform01(idx) = (word(k, idx) >> 11) * 2^-53
    U(a, b)        = a + (b - a) * uniform01, each operation one IEEE op.
Dense matrices are row-major, element (i, c) of an n x d matrix has index
i * d + c.
"""
import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15

LABEL_A = 0x41          # dense A entries
LABEL_B = 0x42          # right-hand side b
LABEL_DIAGU = 0x55      # U(1,10) diagonal of the coherent config
LABEL_CSR_COL = 0x43    # CSR column draws
LABEL_CSR_VAL = 0x56    # CSR values

_U64 = np.uint64


def _mix_int(z):
    z &= MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    z ^= z >> 31
    return z


def stream_key(seed, label):
    return _mix_int((seed & MASK64) ^ (label << 32))


def _mix(z):
    with np.errstate(over="ignore"):
        z = z ^ (z >> _U64(30))
        z = z * _U64(0xBF58476D1CE4E5B9)
        z = z ^ (z >> _U64(27))
        z = z * _U64(0x94D049BB133111EB)
        z = z ^ (z >> _U64(31))
    return z


def words(key, ctr):
    ctr = np.asarray(ctr, dtype=_U64)
    with np.errstate(over="ignore"):
        return _mix(_U64(key) + (ctr + _U64(1)) * _U64(GAMMA))


def normal(seed, label, idx):
    """Irwin-Hall(12) - 6 standard-normal surrogate at integer indices idx."""
    idx = np.asarray(idx, dtype=_U64)
    key = stream_key(seed, label)
    acc = np.zeros(idx.shape, dtype=_U64)
    base = idx * _U64(6)
    lo = _U64(0xFFFFFFFF)
    for t in range(6):
        w = words(key, base + _U64(t))
        acc += (w & lo) + (w >> _U64(32))
    v = acc.astype(np.int64) - np.int64(6 << 32)
    return v.astype(np.float64) * (2.0 ** -32)


def uniform01(seed, label, idx):
    w = words(stream_key(seed, label), np.asarray(idx, dtype=_U64))
    return (w >> _U64(11)).astype(np.float64) * (2.0 ** -53)


# ------------------------------------------------------------------ workloads
def dense_block(cfg, r0, r1, cols=None):
    """Rows [r0, r1) (and optionally a column subset) of the config's dense A."""
    n, d, seed = cfg.n, cfg.d, cfg.seed
    cols = np.arange(d, dtype=np.int64) if cols is None else np.asarray(cols, dtype=np.int64)
    rows = np.arange(r0, r1, dtype=np.int64)
    idx = rows[:, None] * d + cols[None, :]
    if cfg.kind == "dense_gauss":
        return normal(seed, LABEL_A, idx)
    if cfg.kind == "dense_coherent":
        eps = 1e-8 * normal(seed, LABEL_A, idx)
        diag_mask = (rows[:, None] == cols[None, :]) & (rows[:, None] < min(d, n))
        if diag_mask.any():
            ri = np.nonzero(diag_mask)
            uu = uniform01(seed, LABEL_DIAGU, rows[ri[0]])
            dv = 1.0 + 9.0 * uu            # U(1, 10): one IEEE multiply, one add
            eps[ri] = dv + eps[ri]
        return eps
    raise ValueError(f"not a dense config: {cfg.kind}")


def dense(cfg):
    return dense_block(cfg, 0, cfg.n)


def rhs(cfg):
    """b ~ N(0,1) for every config (R15)."""
    return normal(cfg.seed, LABEL_B, np.arange(cfg.n, dtype=np.int64))


def csr_rows(cfg, r0, r1):
    """CSR rows [r0, r1): cfg.nnz_row distinct sorted columns per row drawn by
    rejection (attempt t at counter (i << 8) + t), values normal at index
    i * nnz_row + k.  Returns (row_ptr local int64, col_idx int32, val f64)."""
    n, d, k, seed = cfg.n, cfg.d, cfg.nnz_row, cfg.seed
    if k > d:
        raise ValueError("nnz per row > d")
    rows = np.arange(r0, r1, dtype=np.uint64)
    nr = rows.shape[0]
    key = stream_key(seed, LABEL_CSR_COL)
    cols = np.full((nr, k), -1, dtype=np.int64)
    nacc = np.zeros(nr, dtype=np.int64)
    active = np.arange(nr)
    t = 0
    while active.size:
        if t >= 256:
            raise RuntimeError("CSR column draw exhausted")
        w = words(key, (rows[active] << _U64(8)) + _U64(t))
        c = ((w >> _U64(32)) * _U64(d)) >> _U64(32)      # floor(hi32 * d / 2^32)
        c = c.astype(np.int64)
        dup = (cols[active] == c[:, None]).any(axis=1)
        acc = active[~dup]
        cols[acc, nacc[acc]] = c[~dup]
        nacc[acc] += 1
        active = active[nacc[active] < k]
        t += 1
    cols.sort(axis=1)
    vidx = rows.astype(np.int64)[:, None] * k + np.arange(k)[None, :]
    val = normal(seed, LABEL_CSR_VAL, vidx)
    row_ptr = np.arange(nr + 1, dtype=np.int64) * k
    return row_ptr, cols.reshape(-1).astype(np.int32), val.reshape(-1)


def csr(cfg):
    return csr_rows(cfg, 0, cfg.n)


def small_int_dense(seed, n, d, lo=-3, hi=3):
    """Integer-valued test matrix (entries in [lo, hi]) for the order-independent
    bit-exact checks."""
    idx = np.arange(n * d, dtype=np.uint64)
    w = words(stream_key(seed, 0x49), idx)
    span = hi - lo + 1
    v = ((w >> _U64(32)) * _U64(span)) >> _U64(32)
    return (v.astype(np.int64) + lo).astype(np.float64).reshape(n, d)
