"""Pins for oracle/hadamard.py: Def. def::HRHT."""
import math

import numpy as np
import pytest

from oracle import hadamard


def test_golden_small(golden):
    rows = golden("hadamard_small.txt")
    H2 = hadamard.hadamard_formula(2)
    for r in rows:
        if r[0] == "n2":
            x = np.array([float(r[1]), float(r[2])])
            want = np.array([float(r[3]), float(r[4])]) / math.sqrt(2)
            assert np.allclose(H2 @ x, want, rtol=0, atol=1e-16)
            assert np.allclose(hadamard.fwht(x) / math.sqrt(2), want, rtol=0, atol=1e-16)
    H4 = hadamard.hadamard_formula(4) * 2
    want4 = np.array([[float(v) for v in r[2:]] for r in rows if r[0] == "n4row"])
    assert np.array_equal(H4, want4)


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16, 32, 64])
def test_sylvester_equals_formula(n):
    """Sylvester recursion (natural order) equals the P:L796 formula entrywise."""
    assert np.array_equal(hadamard.hadamard_sylvester(n) / math.sqrt(n), hadamard.hadamard_formula(n))


@pytest.mark.parametrize("n", [2, 8, 64, 256])
def test_hhat_squared_is_nI(n):
    H = hadamard.hadamard_sylvester(n)
    assert np.array_equal(H @ H, n * np.eye(n))


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256])
def test_fast_matches_dense(n):
    """FWHT vs the naive matrix to 1e-14, exact on integers."""
    r = np.random.default_rng(n)
    x = r.standard_normal((n, 3))
    H = hadamard.hadamard_formula(n)
    assert np.allclose(hadamard.fwht(x) / math.sqrt(n), H @ x, rtol=0, atol=1e-14 * np.abs(x).sum())
    xi = r.integers(-3, 4, size=(n, 5)).astype(float)
    assert np.array_equal(hadamard.fwht(xi), hadamard.hadamard_sylvester(n) @ xi)


def test_unit_vectors_and_involution():
    n = 1024
    e0 = np.zeros(n)
    e0[0] = 1
    c = hadamard.c_n(n)
    assert np.allclose(c * hadamard.fwht(e0), np.full(n, c))
    assert np.allclose(c * hadamard.fwht(np.ones(n)), math.sqrt(n) * e0)
    x = np.random.default_rng(3).standard_normal(n)
    y = c * hadamard.fwht(x)
    assert abs(np.linalg.norm(y) / np.linalg.norm(x) - 1) < 1e-13   # orthogonal
    assert np.allclose(c * hadamard.fwht(y), x, atol=1e-13)          # H(Hx) = x


def test_stage_split_is_exact():
    """Stages over bit ranges compose to the full transform bit for bit."""
    x = np.random.default_rng(4).standard_normal((512, 7))
    full = hadamard.fwht(x)
    part = np.array(x)
    hadamard.fwht_stages(part, 0, 3)
    hadamard.fwht_stages(part, 3, 6)
    hadamard.fwht_stages(part, 6, 9)
    assert np.array_equal(full, part)


def test_diag_signs():
    rows = np.arange(5000)
    dv = hadamard.diag_signs(7, rows)
    assert set(np.unique(dv)) == {-1, 1}
    assert abs((dv == -1).sum() - 2500) < 5 * math.sqrt(1250)
    assert [hadamard.diag_sign_scalar(7, i) for i in range(200)] == list(dv[:200])
    assert not np.array_equal(dv, hadamard.diag_signs(8, rows))


def test_hd_preserves_column_norms():
    """H D is orthogonal: column norms preserved (north_star oracle check)."""
    A = np.random.default_rng(5).standard_normal((1000, 6))
    n_pad = hadamard.next_pow2(1000)
    Y = hadamard.c_n(n_pad) * hadamard.hd(2, A)
    assert Y.shape == (1024, 6)
    assert np.allclose(np.linalg.norm(Y, axis=0), np.linalg.norm(A, axis=0), rtol=1e-13)


def test_tropp_coherence_bound():
    """Lemma 14 (Tropp): mu(HDU) <= sqrt(r/n) + sqrt(8 log(n/d1)/n)
    with probability >= 1 - d1, for the maximally coherent U = [I_r; 0]."""
    n, r, d1 = 1024, 8, 0.1
    U = np.zeros((n, r))
    U[:r, :r] = np.eye(r)
    bound = math.sqrt(r / n) + math.sqrt(8 * math.log(n / d1) / n)
    ok = 0
    trials = 60
    for seed in range(trials):
        Y = hadamard.c_n(n) * hadamard.hd(seed, U)
        mu = np.sqrt((Y * Y).sum(axis=1)).max()
        ok += mu <= bound
    assert ok / trials >= 1 - d1 - 0.05
    # and the transform really reduces coherence from mu(U) = 1
    assert mu < 0.5
