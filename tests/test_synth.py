"""The shared input generators (host side): shapes and value structure."""
import numpy as np

from synth import configs, gen


def test_normal_moments():
    x = gen.normal(1, gen.LABEL_A, np.arange(200000))
    assert abs(x.mean()) < 0.01 and abs(x.var() - 1) < 0.01
    assert np.abs(x).max() <= 6
    # exactness: every value is an integer multiple of 2^-32
    assert np.array_equal(np.round(x * 2**32), x * 2**32)


def test_coherent_structure():
    cfg = configs.C3.scaled(n=300, d=40)
    A = gen.dense(cfg)
    diag = np.diag(A[:40])
    assert (diag > 0.99).all() and (diag < 10.01).all()
    off = A.copy()
    off[np.arange(40), np.arange(40)] = 0
    assert np.abs(off).max() < 1e-7


def test_csr_structure():
    cfg = configs.C4.scaled(n=2000, d=100)
    rp, ci, v = gen.csr(cfg)
    assert rp[-1] == 2000 * 8
    cols = ci.reshape(2000, 8)
    assert (np.diff(cols, axis=1) > 0).all() and cols.min() >= 0 and cols.max() < 100
    # row blocks are consistent with the whole
    rp2, ci2, v2 = gen.csr_rows(cfg, 500, 900)
    assert np.array_equal(ci2, ci[500 * 8:900 * 8]) and np.array_equal(v2, v[500 * 8:900 * 8])


def test_dense_block_consistent():
    cfg = configs.C2.scaled(n=64, d=16)
    A = gen.dense(cfg)
    assert np.array_equal(gen.dense_block(cfg, 10, 20, [3, 5]), A[10:20][:, [3, 5]])
