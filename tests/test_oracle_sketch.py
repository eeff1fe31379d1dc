"""Pins for oracle/sketch.py and oracle/probes.py: Algorithm 1 Step 1."""
import math

import numpy as np
import pytest
import scipy.sparse

from oracle import hadamard, hashing, probes, sketch
from synth import configs, gen


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("n,d,m,s", [(1, 1, 1, 1), (3, 2, 2, 1), (64, 5, 7, 3), (300, 17, 40, 2), (257, 4, 256, 4)])
def test_tier0_matches_tier1(n, d, m, s):
    r = np.random.default_rng(n)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    SA, Sb = sketch.sketch_dense(4, A, b, m, s)
    SA0, Sb0 = sketch.sketch_dense_S(4, A, b, m, s)
    assert rel(SA, SA0) < 1e-14 and rel(Sb, Sb0) < 1e-14


def test_identity_gives_S():
    """A = I_n: SA = S exactly (materialisation check)."""
    n, m, s = 64, 9, 2
    SA, _ = sketch.sketch_dense(6, np.eye(n), None, m, s)
    assert np.array_equal(SA, hashing.dense_S(6, n, m, s))


def test_scipy_sparse_crosscheck():
    n, d, m, s = 400, 8, 30, 3
    A = np.random.default_rng(1).standard_normal((n, d))
    b_, j_, v_ = hashing.triples(12, n, m, s)
    S = scipy.sparse.coo_matrix((v_, (b_, j_)), shape=(m, n)).tocsr()
    SA, _ = sketch.sketch_dense(12, A, None, m, s)
    assert rel(SA, S @ A) < 1e-14


def test_linearity():
    r = np.random.default_rng(2)
    A, B = r.standard_normal((200, 6)), r.standard_normal((200, 6))
    SA, _ = sketch.sketch_dense(3, A, None, 20, 2)
    SB, _ = sketch.sketch_dense(3, B, None, 20, 2)
    SAB, _ = sketch.sketch_dense(3, A + B, None, 20, 2)
    assert rel(SAB, SA + SB) < 1e-14


def test_integer_inputs_bitexact():
    """Integer A: every bucket sum is exact, so SA == fl(c_s * (S_int @ A)) bit for
    bit, with S_int @ A computed independently in int64."""
    n, d, m, s = 333, 9, 21, 3
    A = gen.small_int_dense(5, n, d)
    SA, _ = sketch.sketch_dense(9, A, None, m, s)
    Sint = np.rint(hashing.dense_S(9, n, m, s) * math.sqrt(s)).astype(np.int64)
    T = Sint @ A.astype(np.int64)
    assert np.array_equal(SA, hashing.c_s(s) * T.astype(np.float64))


def test_empty_buckets_are_zero():
    SA, Sb = sketch.sketch_dense(2, np.ones((3, 4)), np.ones(3), 50, 1)
    ptr, _, _ = hashing.bucket_lists(2, np.arange(3), 50, 1)
    empty = np.diff(ptr) == 0
    assert empty.sum() >= 47
    assert (SA[empty] == 0).all() and (Sb[empty] == 0).all()


def test_all_ones_b():
    """b = 1 (the paper's right-hand side): Sb[b] = c_s * sum of signs."""
    n, m, s = 1000, 13, 2
    _, Sb = sketch.sketch_dense(21, np.zeros((n, 1)), np.ones(n), m, s)
    ptr, _, sg = hashing.bucket_lists(21, np.arange(n), m, s)
    want = np.array([sg[ptr[b]:ptr[b + 1]].astype(np.int64).sum() for b in range(m)]) / math.sqrt(s)
    assert np.allclose(Sb, want, rtol=0, atol=1e-12)


def test_csr_equals_dense():
    """CSR sketch equals the dense sketch of the same matrix bit for bit."""
    cfg = configs.C4.scaled(n=600, d=40, m=32)
    rp, ci, v = gen.csr(cfg)
    A = sketch.csr_to_dense(rp, ci, v, cfg.d)
    assert (np.count_nonzero(A, axis=1) == cfg.nnz_row).all()
    b = gen.rhs(cfg)
    SA, Sb = sketch.sketch_csr(cfg.seed, rp, ci, v, cfg.d, b, cfg.m, cfg.s)
    SA2, Sb2 = sketch.sketch_dense(cfg.seed, A, b, cfg.m, cfg.s)
    assert np.array_equal(SA, SA2) and np.array_equal(Sb, Sb2)


@pytest.mark.parametrize("n,d,m,s", [(1, 2, 1, 1), (5, 3, 4, 1), (64, 4, 16, 2), (100, 3, 32, 1), (256, 6, 40, 3)])
def test_rht_tier0_matches_tier1(n, d, m, s):
    r = np.random.default_rng(n + 7)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    SA, Sb = sketch.rht_sketch(13, A, b, m, s)
    SA0, Sb0 = sketch.rht_sketch_dense_S(13, A, b, m, s)
    assert rel(SA, SA0) < 1e-13 and rel(Sb, Sb0) < 1e-13


def test_hda_matches_dense():
    n = 128
    A = np.random.default_rng(8).standard_normal((n, 5))
    H = hadamard.hadamard_formula(n)
    D = np.diag(hadamard.diag_signs(3, np.arange(n)).astype(float))
    assert rel(sketch.hda(3, A), H @ D @ A) < 1e-14


def test_rht_integer_bitexact():
    """Integer A: S_h Hhat D A is an exact integer matrix; SA == fl(c_ns * T)."""
    n, d, m, s = 128, 5, 12, 2
    A = gen.small_int_dense(6, n, d)
    SA, _ = sketch.rht_sketch(17, A, None, m, s)
    Sint = np.rint(hashing.dense_S(17, n, m, s) * math.sqrt(s)).astype(np.int64)
    Hint = hadamard.hadamard_sylvester(n).astype(np.int64)
    Dint = hadamard.diag_signs(17, np.arange(n)).astype(np.int64)
    T = Sint @ (Hint @ (Dint[:, None] * A.astype(np.int64)))
    assert np.array_equal(SA, sketch.c_ns(n, s) * T.astype(np.float64))


def test_rht_padding():
    """Non-power-of-two n pads with zero rows; all n_pad columns of S_h hashed."""
    n, d, m, s = 100, 3, 10, 1
    A = np.random.default_rng(9).standard_normal((n, d))
    Ap = np.zeros((128, d))
    Ap[:n] = A
    SA, _ = sketch.rht_sketch(5, A, None, m, s)
    SAp, _ = sketch.rht_sketch(5, Ap, None, m, s)
    assert np.array_equal(SA, SAp)


def test_bucket_subset():
    A = np.random.default_rng(3).standard_normal((300, 4))
    SA, _ = sketch.sketch_dense(1, A, None, 17, 2)
    sub, _ = sketch.sketch_dense(1, A, None, 17, 2, buckets=[3, 0, 16])
    assert np.array_equal(sub, SA[[3, 0, 16]])


def test_freivalds_probes():
    r = np.random.default_rng(10)
    n, d, m, s = 500, 7, 24, 2
    A = r.standard_normal((n, d))
    w, v = r.standard_normal(m), r.standard_normal(d)
    SA, _ = sketch.sketch_dense(3, A, None, m, s)
    assert abs(w @ SA @ v - probes.probe_dense(3, n, m, s, w, A @ v)) < 1e-12 * np.linalg.norm(SA) * 10
    SAh, _ = sketch.rht_sketch(3, A, None, m, s)
    assert abs(w @ SAh @ v - probes.probe_rht(3, n, m, s, w, A @ v)) < 1e-12 * np.linalg.norm(SAh) * 10
    # a one-entry corruption is detected
    bad = SA.copy()
    bad[5, 2] += 1e-6
    assert abs(w @ bad @ v - probes.probe_dense(3, n, m, s, w, A @ v)) > 1e-9


def test_column_streaming_equals_full():
    cfg = configs.C2.scaled(n=1024, d=12, m=30)
    A = gen.dense(cfg)
    SA, _ = sketch.rht_sketch(cfg.seed, A, None, cfg.m, cfg.s)
    cols = [1, 7, 11]
    part = sketch.rht_sketch_columns(cfg.seed, lambda c: gen.dense_block(cfg, 0, cfg.n, c), cfg.n, cfg.m, cfg.s, cols)
    assert np.array_equal(part, SA[:, cols])
