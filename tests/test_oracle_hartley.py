"""Pins for oracle/hartley.py: the normalized DHT of eq. (6.1) and
the HR-DHT sketch S_h F D."""
import math

import numpy as np
import pytest

from oracle import hadamard, hartley, hashing


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 12, 64, 100])
def test_fft_route_equals_definition(n):
    X = np.random.default_rng(n).standard_normal((n, 3))
    F = hartley.dht_matrix(n)
    assert np.allclose(hartley.dht_unnormalised(X) / math.sqrt(n), F @ X, rtol=0, atol=1e-13 * max(1, n))


@pytest.mark.parametrize("n", [1, 2, 7, 16, 256])
def test_involution_and_orthogonality(n):
    """F (F x) = x for this normalisation; F is symmetric orthogonal."""
    F = hartley.dht_matrix(n)
    assert np.allclose(F, F.T, atol=1e-15)
    assert np.allclose(F @ F, np.eye(n), atol=1e-12)
    x = np.random.default_rng(1).standard_normal(n)
    y = hartley.dht_unnormalised(hartley.dht_unnormalised(x)) / n
    assert np.allclose(y, x, atol=1e-12)


def test_small_cases_and_special_vectors():
    assert np.array_equal(hartley.dht_matrix(1), np.ones((1, 1)))
    # n = 2: the DHT equals the 2-point Walsh-Hadamard transform
    assert np.allclose(hartley.dht_matrix(2), hadamard.hadamard_formula(2), atol=1e-15)
    # n = 4: it does not (cas(pi/2) = 1, cas(3 pi/2) = -1 differ from the Sylvester rows)
    assert not np.allclose(hartley.dht_matrix(4), hadamard.hadamard_formula(4))
    n = 12
    e0 = np.zeros(n)
    e0[0] = 1.0
    assert np.allclose(hartley.dht_unnormalised(e0), np.ones(n))        # DHT of delta = constant
    assert np.allclose(hartley.dht_unnormalised(np.ones(n)), n * e0, atol=1e-12)  # and back
    x = np.random.default_rng(4).standard_normal(n)
    assert math.isclose(np.sum(hartley.dht_unnormalised(x) ** 2), n * np.sum(x ** 2), rel_tol=1e-13)  # Parseval


@pytest.mark.parametrize("n,d,m,s", [(7, 2, 3, 1), (100, 5, 16, 2), (257, 3, 40, 3)])
def test_sketch_tier0_matches_tier1(n, d, m, s):
    r = np.random.default_rng(n)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    SA, Sb = hartley.hrdht_sketch(9, A, b, m, s)
    SA0, Sb0 = hartley.hrdht_sketch_dense_S(9, A, b, m, s)
    assert np.linalg.norm(SA - SA0) <= 1e-13 * np.linalg.norm(SA0)
    assert np.linalg.norm(Sb - Sb0) <= 1e-13 * np.linalg.norm(Sb0)
    assert hashing.c_s(s) > 0


def test_column_norms_preserved_and_coherence_reduced():
    """F D is orthogonal (column norms of F D A equal those of A); on the coherent
    A = [I; 0] it spreads every column (max |entry| ~ sqrt(2/n) vs 1)."""
    n, d = 1024, 16
    A = np.zeros((n, d))
    A[:d, :d] = np.eye(d)
    X = hartley.fd(5, A) / math.sqrt(n)
    assert np.allclose(np.linalg.norm(X, axis=0), 1.0, atol=1e-12)
    assert np.abs(X).max() <= math.sqrt(2.0 / n) + 1e-12
