"""s-hashing variant (Def. def::s-hashing-variant) through the C ABI
(skh_hash_gen_variant) vs oracle/variant.py: column draws and bucket lists
bit-exact; T A, T b, T H D A and CSR T A bit-exact (the consumers are the
s-hashing kernels, reading R18 fixes the order of coincident draws)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2105_11815_b200.build as b
    b.build()


def skh():
    import paper_2105_11815_b200 as p
    return p


def np_(t):
    return t.detach().cpu().numpy()


def assert_bits(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape
    assert np.linalg.norm(got - want) <= 1e-12 * max(np.linalg.norm(want), 1e-300)
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


# (n, m, s): many coincident draws for small m, both transpose paths (segmented
# for N <= 96 m, radix otherwise), s = m, s up to 64
CASES = [(1, 1, 1), (50, 2, 2), (1000, 3, 3), (777, 16, 3), (5000, 64, 8), (3000, 100, 64), (20000, 300, 2),
         (70000, 300, 5), (4096, 256, 2), (100000, 7, 4)]


@pytest.mark.parametrize("n,m,s", CASES)
def test_variant_hash_bitexact(n, m, s):
    from oracle import variant
    bl = skh().hash_gen(5, m, s, n, want_cols=True, variant=True)
    rows, signs = variant.draw_columns(5, np.arange(n), m, s)
    assert np.array_equal(np_(bl.col_rows)[: n * s].reshape(n, s), rows)
    assert np.array_equal(np_(bl.col_signs)[: n * s].reshape(n, s), signs)
    ptr, brow, bsg = variant.bucket_lists(5, np.arange(n), m, s)
    assert np.array_equal(np_(bl.ptr), ptr)
    assert np.array_equal(np_(bl.rows)[: n * s], brow)
    assert np.array_equal(np_(bl.signs)[: n * s], bsg)
    assert skh().hash_status(bl) == 0


def test_variant_s1_equals_hashing():
    a = skh().hash_gen(8, 50, 1, 3000, want_cols=True, variant=True)
    b = skh().hash_gen(8, 50, 1, 3000, want_cols=True)
    for x, y in [(a.ptr, b.ptr), (a.rows, b.rows), (a.signs, b.signs), (a.col_rows, b.col_rows)]:
        assert torch.equal(x, y)


@pytest.mark.parametrize("n,d,m,s", [(200, 7, 3, 3), (3000, 33, 40, 4), (5000, 64, 256, 2), (20000, 5, 9, 8)])
def test_variant_sketch_dense(n, d, m, s):
    from oracle import variant
    r = np.random.default_rng(n + d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    bl = skh().hash_gen(31, m, s, n, variant=True)
    SA, Sb = skh().sketch_dense(bl, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda())
    TA, Tb = variant.sketch_dense(31, A, b, m, s)
    assert_bits(np_(SA), TA)
    assert_bits(np_(Sb), Tb)


def test_variant_hrht():
    """T H D A (Thm thm::HRHT_variant's sketch): rht_stages then the
    variant lists, vs the oracle's H D A hashed with T."""
    from oracle import sketch, variant
    n, d, m, s = 4096, 16, 64, 3
    A = np.random.default_rng(4).standard_normal((n, d))
    Y = skh().rht_stages(12, torch.from_numpy(A).cuda(), 0, 12, apply_diag=True, alpha=1.0)
    bl = skh().hash_gen(12, m, s, n, variant=True)
    SA, _ = skh().sketch_dense(bl, Y, alpha=skh().c_ns(n, s))
    X = sketch.hadamard.hd(12, A)
    ptr, rows, signs = variant.bucket_lists(12, np.arange(n), m, s)
    assert_bits(np_(SA), sketch.bucket_sum(X, ptr, rows, signs, sketch.c_ns(n, s)))


def test_variant_csr():
    from oracle import sketch, variant
    from synth import configs, gen
    cfg = configs.C4.scaled(n=3000, d=300, m=50)
    rp, ci, v = gen.csr(cfg)
    A = sketch.csr_to_dense(rp, ci, v, cfg.d)
    bl = skh().hash_gen(cfg.seed, cfg.m, cfg.s, cfg.n, variant=True)
    SA, _ = skh().sketch_csr(bl, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(v).cuda(),
                             cfg.d)
    TA, _ = variant.sketch_dense(cfg.seed, A, None, cfg.m, cfg.s)
    assert_bits(np_(SA), TA)
