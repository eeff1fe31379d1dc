"""Pins for oracle/hashing.py: Def. def::sampling_and_hashing."""
import math

import numpy as np
import pytest
import scipy.stats

from oracle import hashing


@pytest.mark.parametrize("m,s", [(1, 1), (2, 1), (2, 2), (7, 3), (16, 16), (64, 2), (256, 5)])
def test_vectorised_matches_pure_python(m, s):
    n = 120
    rows, signs = hashing.draw_columns(11, np.arange(n), m, s)
    for j in range(n):
        r, sg = hashing.draw_column(11, j, m, s)
        assert list(rows[j]) == r
        assert list(signs[j]) == sg


@pytest.mark.parametrize("m,s", [(3, 1), (10, 2), (16, 3), (8, 8), (256, 2)])
def test_structure(m, s):
    """Exactly s distinct rows per column, entries +-1/sqrt(s), unit column norm
    (S:L140-148)."""
    n = 200
    S = hashing.dense_S(3, n, m, s)
    c = 1.0 / math.sqrt(s)
    assert ((S != 0).sum(axis=0) == s).all()
    nz = S[S != 0]
    assert np.all((nz == c) | (nz == -c))
    assert np.allclose((S * S).sum(axis=0), 1.0, rtol=0, atol=4e-16)


def test_one_hashing_single_pm1():
    """s = 1: every column one nonzero of value +-1."""
    S = hashing.dense_S(5, 1000, 3, 1)
    assert ((S != 0).sum(axis=0) == 1).all()
    assert set(np.unique(S[S != 0])) <= {-1.0, 1.0}


def test_s_equals_m_dense_columns():
    """s = m: every column dense, entries +-1/sqrt(m)."""
    S = hashing.dense_S(9, 50, 6, 6)
    assert (S != 0).all()
    assert np.allclose(np.abs(S), 1 / math.sqrt(6))


def test_uniform_buckets_chi2():
    """s=2, m=64, n=1e4: bucket marginal uniform; chi^2 p > 1e-3."""
    m, s, n = 64, 2, 10000
    rows, _ = hashing.draw_columns(17, np.arange(n), m, s)
    counts = np.bincount(rows.reshape(-1), minlength=m)
    p = scipy.stats.chisquare(counts).pvalue
    assert p > 1e-3


def test_pair_distribution_uniform():
    """Without replacement: the unordered pair {i1, i2} is uniform over the
    C(m,2) pairs (a dropped rejection would put mass on i1 == i2)."""
    m, s, n = 8, 2, 40000
    rows, _ = hashing.draw_columns(23, np.arange(n), m, s)
    assert (rows[:, 0] != rows[:, 1]).all()
    a = np.minimum(rows[:, 0], rows[:, 1])
    b = np.maximum(rows[:, 0], rows[:, 1])
    counts = np.bincount(a * m + b, minlength=m * m)
    pairs = counts[[i * m + j for i in range(m) for j in range(i + 1, m)]]
    assert pairs.sum() == n
    assert scipy.stats.chisquare(pairs).pvalue > 1e-3


def test_sign_balance():
    """Signs are fair coins independent of rows (P:L272 footnote; R4)."""
    n, m, s = 20000, 32, 3
    rows, signs = hashing.draw_columns(29, np.arange(n), m, s)
    neg = (signs == -1).sum()
    N = n * s
    assert abs(neg - N / 2) < 5 * math.sqrt(N / 4)
    # independence from the row: sign balance per bucket
    for b in range(m):
        sel = signs[rows == b]
        assert abs((sel == -1).sum() - sel.size / 2) < 5 * math.sqrt(sel.size / 4)


def test_norm_unbiased():
    """E||Sx||^2 = ||x||^2 (P:L272 footnote) within 2% over 1e4 draws."""
    x = np.linspace(-1.0, 2.0, 24)
    vals = []
    for seed in range(10000):
        rows, signs = hashing.draw_columns(seed, np.arange(24), 6, 2)
        y = np.zeros(6)
        np.add.at(y, rows.reshape(-1), (signs.astype(float) / math.sqrt(2) * x[:, None]).reshape(-1))
        vals.append(y @ y)
    assert abs(np.mean(vals) / (x @ x) - 1) < 0.02


def test_example1_birthday(golden):
    """Example 1: with 1-hashing the r columns of S_1 land in
    distinct rows with probability prod(1 - k/m) <= exp(-r(r-1)/2m)."""
    for r, m, exact, bound in golden("example1_birthday.txt"):
        r, m, exact, bound = int(r), int(m), float(exact), float(bound)
        prod = 1.0
        for k in range(1, r):
            prod *= 1 - k / m
        assert abs(prod - exact) < 1e-6 and prod <= bound
        trials = 6000
        hits = 0
        for seed in range(trials):
            rows, _ = hashing.draw_columns(1000 + seed, np.arange(r), m, 1)
            hits += len(set(rows[:, 0].tolist())) == r
        freq = hits / trials
        assert abs(freq - exact) < 4.5 * math.sqrt(exact * (1 - exact) / trials)


def test_errors():
    for m, s in [(4, 5), (4, 0), (0, 1), (100, 65)]:
        with pytest.raises(ValueError):
            hashing.draw_columns(1, np.arange(3), m, s)


def test_bucket_lists_transpose():
    """Bucket lists = CSR of S: counts sum to n s, each (i, k) once, rows ascending,
    and the round trip reproduces the column lists."""
    n, m, s = 500, 37, 3
    ptr, rows, signs = hashing.bucket_lists(8, np.arange(n), m, s)
    assert ptr[0] == 0 and ptr[-1] == n * s
    crow, csg = hashing.draw_columns(8, np.arange(n), m, s)
    seen = set()
    for b in range(m):
        seg = rows[ptr[b]:ptr[b + 1]]
        assert (np.diff(seg) > 0).all()
        for t in range(ptr[b], ptr[b + 1]):
            i = rows[t]
            k = list(crow[i]).index(b)
            assert signs[t] == csg[i, k]
            seen.add((i, k))
    assert len(seen) == n * s
    # dense S from bucket lists equals tier-0 dense S
    S = np.zeros((m, n))
    for b in range(m):
        for t in range(ptr[b], ptr[b + 1]):
            S[b, rows[t]] = signs[t] / math.sqrt(s)
    assert np.array_equal(S, hashing.dense_S(8, n, m, s))
