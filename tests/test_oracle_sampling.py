"""Pins for oracle/sampling.py: SR-DHT (eq. (7.2)) and the Fig. 1
claim."""
import math

import numpy as np
import scipy.stats

from oracle import hartley, sampling


def test_rows_uniform_with_replacement():
    n, m = 50, 200000
    j = sampling.sample_rows(3, n, m)
    assert j.min() >= 0 and j.max() < n
    assert scipy.stats.chisquare(np.bincount(j, minlength=n)).pvalue > 1e-3
    # with replacement: m = 40 draws from n = 1000 repeat with prob 1 - prod (1 - i/n)
    reps = np.mean([len(set(sampling.sample_rows(sd, 1000, 40))) < 40 for sd in range(2000)])
    want = 1 - math.prod(1 - i / 1000 for i in range(40))
    assert abs(reps - want) < 0.04


def test_sketch_equals_explicit_product():
    """Tier 0: S_s (explicit 0/1) @ F (eq. (6.1) matrix) @ D @ A."""
    n, d, m = 300, 4, 50
    A = np.random.default_rng(1).standard_normal((n, d))
    SA, _ = sampling.srdht_sketch(7, A, None, m)
    from oracle import hadamard
    Dv = hadamard.diag_signs(7, np.arange(n)).astype(float)
    ref = sampling.dense_Ss(7, n, m) @ hartley.dht_matrix(n) @ (Dv[:, None] * A)
    assert np.linalg.norm(SA - ref) <= 1e-13 * np.linalg.norm(ref)
    assert np.all(sampling.dense_Ss(7, n, m).sum(axis=1) == 1)


def test_coherent_matrix_definition():
    A = sampling.coherent_A(10, 3)
    assert A.shape == (10, 3)
    assert np.allclose(A[:3] - np.eye(3), 1e-8) and np.allclose(A[3:], 1e-8)


def test_fig1_hashing_beats_sampling():
    """'using hashing instead of sampling in randomised DHT allows the use
    of a smaller m to reach a given preconditioning quality'.  Scaled replica
    (n = 2000, d = 100, the paper's n/d = 10): at m/d = 1.5 and 2, the median
    kappa(A R^{-1}) over seeds is smaller with hashing (s = 1)."""
    n, d = 2000, 100
    A = sampling.coherent_A(n, d)
    for ratio in (1.5, 2.0):
        m = int(ratio * d)
        kh, ks = zip(*[sampling.fig1_point(sd, A, m) for sd in range(5)])
        assert np.median(kh) < np.median(ks)
        assert np.median(kh) < 20
