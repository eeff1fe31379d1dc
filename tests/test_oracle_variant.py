"""Pins for oracle/variant.py: the s-hashing variant of Def. def::s-hashing-variant
 and its Lemma 8 decomposition."""
import math

import numpy as np
import pytest
import scipy.stats

from oracle import hashing, sketch, variant


@pytest.mark.parametrize("m,s", [(1, 1), (2, 2), (5, 3), (16, 3), (64, 8), (7, 7)])
def test_def7_equals_lemma8(m, s):
    """Def. 7's accumulate-per-draw construction and Lemma 8's sum of s 1-hashing
    matrices (loops swapped, integer sums) give the same T exactly."""
    n = 150
    T = variant.dense_T(3, n, m, s)
    T8 = variant.dense_T_lemma8(3, n, m, s)
    # same integer pattern; Def. 7 accumulates c + c + ... in floating point, Lemma 8
    # scales the integer sum once, so entries of 3+ coincident draws may differ by an ulp
    assert np.array_equal(np.rint(T * math.sqrt(s)), np.rint(T8 * math.sqrt(s)))
    assert np.allclose(T, T8, rtol=0, atol=1e-15)


def test_s1_is_one_hashing():
    """both reduce to 1-hashing for s = 1 (here: the same draws)."""
    for m in (1, 3, 100):
        assert np.array_equal(variant.dense_T(7, 300, m, 1), hashing.dense_S(7, 300, m, 1))


def test_vectorised_matches_pure_python():
    rows, signs = variant.draw_columns(11, np.arange(200), 9, 4)
    for j in range(200):
        r, sg = variant.draw_column(11, j, 9, 4)
        assert list(rows[j]) == r and list(signs[j]) == sg


def test_collision_fraction_exact_probability():
    """s=3, m=16: fraction of columns with < 3 distinct rows is
    1 - 15*14/16^2 = 0.1797 (with replacement); the s-hashing matrix has none."""
    m, s, n = 16, 3, 100000
    rows, _ = variant.draw_columns(5, np.arange(n), m, s)
    distinct = np.array([len(set(r)) for r in rows])
    frac = float((distinct < s).mean())
    want = 1 - variant.distinct_fraction_exact(m, s)
    assert abs(want - (1 - 15 * 14 / 256)) < 1e-15
    assert abs(frac - want) < 0.01
    rows_h, _ = hashing.draw_columns(5, np.arange(2000), m, s)
    assert all(len(set(r)) == s for r in rows_h)


def test_s2_m2_patterns():
    """s=2, m=2: a column is either two entries +-1/sqrt2, a single entry
    +-2/sqrt2 (coincident draws, same sign) or zero (opposite signs)."""
    T = variant.dense_T(13, 4000, 2, 2)
    c = 1 / math.sqrt(2)
    seen = set()
    for j in range(T.shape[1]):
        col = T[:, j]
        nz = col[col != 0]
        if len(nz) == 2:
            assert np.allclose(np.abs(nz), c)
            seen.add("two")
        elif len(nz) == 1:
            assert np.isclose(abs(nz[0]), 2 * c)
            seen.add("double")
        else:
            assert len(nz) == 0
            seen.add("zero")
    assert seen == {"two", "double", "zero"}


def test_rows_uniform_chi2():
    m, s, n = 64, 2, 20000
    rows, _ = variant.draw_columns(17, np.arange(n), m, s)
    assert scipy.stats.chisquare(np.bincount(rows.reshape(-1), minlength=m)).pvalue > 1e-3


def test_norm_preserved_in_expectation():
    """E||T x||^2 = ||x||^2 (independent zero-mean signs; coincident draws add
    sigma_k sigma_l with mean 0).  Monte-Carlo over 400 seeds, 6 sigma."""
    m, s, n = 12, 3, 40
    x = np.random.default_rng(1).standard_normal(n)
    vals = np.array([np.sum((variant.dense_T(sd, n, m, s) @ x) ** 2) for sd in range(400)])
    z = (vals.mean() - x @ x) / (vals.std(ddof=1) / math.sqrt(len(vals)))
    assert abs(z) < 6


def test_bucket_lists_are_csr_of_T():
    """The bucket lists (reading R18) rebuild T exactly, repeated rows included."""
    n, m, s = 500, 6, 4
    ptr, rows, signs = variant.bucket_lists(21, np.arange(n), m, s)
    T = np.zeros((m, n))
    for b in range(m):
        for t in range(ptr[b], ptr[b + 1]):
            T[b, rows[t]] += signs[t] * hashing.c_s(s)
        r = rows[ptr[b]:ptr[b + 1]]
        assert np.all(np.diff(r) >= 0)
        same = np.flatnonzero(np.diff(r) == 0)
        assert np.all(signs[ptr[b] + same] >= signs[ptr[b] + same + 1])  # + before -
    assert np.allclose(T, variant.dense_T(21, n, m, s), atol=1e-15)
    assert ptr[-1] == n * s


def test_sketch_vs_dense_product_and_integer_mode():
    n, d, m, s = 700, 5, 20, 3
    A = np.random.default_rng(2).standard_normal((n, d))
    TA, _ = variant.sketch_dense(9, A, None, m, s)
    assert np.linalg.norm(TA - variant.dense_T(9, n, m, s) @ A) <= 1e-14 * np.linalg.norm(TA)
    Ai = np.random.default_rng(3).integers(-3, 4, size=(n, d)).astype(np.float64)
    TAi, _ = variant.sketch_dense(9, Ai, None, m, s)
    Tint = np.rint(variant.dense_T_lemma8(9, n, m, s) * math.sqrt(s)).astype(np.int64)
    assert np.array_equal(TAi, hashing.c_s(s) * (Tint @ Ai.astype(np.int64)).astype(np.float64))
    assert sketch is not None
