"""CUDA path (through the C ABI) vs the CPU oracle, element by element.

Indices and bucket lists: bit-exact.  Floating point: the kernels keep the
oracle's summation order (R9/R10), so SA, Sb and H D A are compared
BIT-EXACTLY as well, and additionally against the BASELINE.json tolerance
(relative Frobenius error <= 1e-12) so a future reordered kernel has a stated
bar.  Full-size configs are checked on sampled columns/buckets the oracle can
compute exactly (columns are independent under both H and S).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = 1e-12  # BASELINE.json north_star: relative Frobenius error in fp64


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


def assert_same(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    den = max(np.linalg.norm(want), 1e-300)
    assert np.linalg.norm(got - want) / den <= TOL
    assert np.array_equal(got.view(np.int64), want.view(np.int64)), "not bit-identical to the oracle"


# ------------------------------------------------------------------ R1 + R2
HASH_CASES = [(1, 1, 1), (2, 1, 1), (3, 2, 2), (63, 7, 3), (64, 256, 1), (65, 2, 2), (1000, 16, 16), (777, 64, 64),
              (4096, 256, 2), (5000, 1, 1), (3000, 100000, 3), (70000, 300, 5), (20000, 70000, 2)]


@pytest.mark.parametrize("n,m,s", HASH_CASES)
def test_hash_bitexact(n, m, s):
    from oracle import hashing
    bl = skh().hash_gen(1234, m, s, n, want_cols=True)
    rows, signs = hashing.draw_columns(1234, np.arange(n), m, s)
    assert np.array_equal(np_(bl.col_rows)[: n * s].reshape(n, s), rows)
    assert np.array_equal(np_(bl.col_signs)[: n * s].reshape(n, s), signs)
    ptr, brow, bsg = hashing.bucket_lists(1234, np.arange(n), m, s)
    assert np.array_equal(np_(bl.ptr), ptr)
    assert np.array_equal(np_(bl.rows)[: n * s], brow)
    assert np.array_equal(np_(bl.signs)[: n * s], bsg)
    assert skh().hash_status(bl) == 0


@pytest.mark.parametrize("row0,blk,stride", [(5, 0, 0), (1 << 20, 0, 0), (3, 16, 64), (0, 100, 1000)])
def test_hash_row_maps(row0, blk, stride):
    from oracle import hashing
    n, m, s = 800, 37, 2
    k = np.arange(n)
    gid = row0 + k if blk <= 0 else row0 + (k // blk) * stride + (k % blk)
    bl = skh().hash_gen(99, m, s, n, row0=row0, blk=blk, stride=stride)
    ptr, brow, bsg = hashing.bucket_lists(99, gid, m, s)
    assert np.array_equal(np_(bl.ptr), ptr)
    assert np.array_equal(np_(bl.rows), brow)
    assert np.array_equal(np_(bl.signs), bsg)


def test_hash_empty():
    bl = skh().hash_gen(1, 5, 2, 0)
    assert (np_(bl.ptr) == 0).all()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_hash_full_size(name):
    """Bucket lists at every BASELINE.json size (n_pad columns for the H D configs)."""
    from oracle import hadamard, hashing
    from synth import configs
    cfg = configs.ALL[name]
    n = hadamard.next_pow2(cfg.n) if cfg.hd else cfg.n
    bl = skh().hash_gen(cfg.seed, cfg.m, cfg.s, n)
    ptr, brow, bsg = hashing.bucket_lists(cfg.seed, np.arange(n), cfg.m, cfg.s)
    assert np.array_equal(np_(bl.ptr), ptr)
    assert np.array_equal(np_(bl.rows), brow)
    assert np.array_equal(np_(bl.signs), bsg)


# ------------------------------------------------------------------ R5 dense
@pytest.mark.parametrize("n,d,m,s,pad", [(1, 1, 1, 1, 0), (3, 2, 2, 1, 0), (65, 3, 7, 3, 1), (200, 16, 9, 2, 0),
                                         (300, 17, 40, 2, 3), (1000, 64, 300, 1, 0), (4096, 64, 256, 2, 0),
                                         (513, 130, 50, 4, 2), (2000, 1, 64, 3, 0)])
def test_sketch_dense_small(n, d, m, s, pad):
    from oracle import sketch
    r = np.random.default_rng(n * 7 + d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    At = torch.zeros(n, d + pad, dtype=torch.float64, device="cuda")
    At[:, :d] = torch.from_numpy(A)
    bl = skh().hash_gen(42, m, s, n)
    SA, Sb = skh().sketch_dense(bl, At[:, :d], torch.from_numpy(b).cuda())
    SAo, Sbo = sketch.sketch_dense(42, A, b, m, s)
    assert_same(np_(SA), SAo)
    assert_same(np_(Sb), Sbo)


def test_sketch_dense_C1_and_no_b():
    from oracle import sketch
    from synth import configs, gen
    cfg = configs.C1
    A, b = gen.dense(cfg), gen.rhs(cfg)
    bl = skh().hash_gen(cfg.seed, cfg.m, cfg.s, cfg.n)
    SA, Sb = skh().sketch_dense(bl, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda())
    SAo, Sbo = sketch.sketch_dense(cfg.seed, A, b, cfg.m, cfg.s)
    assert_same(np_(SA), SAo)
    assert_same(np_(Sb), Sbo)
    SA2, Sb2 = skh().sketch_dense(bl, torch.from_numpy(A).cuda())
    assert Sb2 is None
    assert_same(np_(SA2), SAo)
    # unscaled partials (alpha = 1) times c_s reproduce the scaled result for integer A
    Ai = gen.small_int_dense(3, cfg.n, cfg.d)
    U, _ = skh().sketch_dense(bl, torch.from_numpy(Ai).cuda(), alpha=1.0)
    SAi, _ = sketch.sketch_dense(cfg.seed, Ai, None, cfg.m, cfg.s)
    assert_same(skh().c_s(cfg.s) * np_(U), SAi)


def test_sketch_dense_C3_full_sampled_columns():
    """C3 at full size (4 GiB A, s=2): SA[:, cols] vs the oracle on A[:, cols]."""
    from oracle import sketch
    from synth import configs, device, gen
    cfg = configs.C3
    A = device.dense(cfg)
    b = device.rhs(cfg)
    bl = skh().hash_gen(cfg.seed, cfg.m, cfg.s, cfg.n)
    SA, Sb = skh().sketch_dense(bl, A, b)
    cols = [0, 1, 2047, 4095]
    SAo, Sbo = sketch.sketch_dense(cfg.seed, gen.dense_block(cfg, 0, cfg.n, cols), gen.rhs(cfg), cfg.m, cfg.s)
    assert_same(np_(SA[:, cols]), SAo)
    assert_same(np_(Sb), Sbo)
    del A


# ------------------------------------------------------------------ R5 CSR
@pytest.mark.parametrize("n,d,m,s,k", [(1, 1, 1, 1, 1), (50, 9, 5, 2, 3), (3000, 300, 64, 3, 8), (500, 9000, 40, 2, 8),
                                       (20000, 64, 1000, 3, 8)])
def test_sketch_csr(n, d, m, s, k):
    from oracle import sketch
    from synth import configs, gen
    cfg = configs.C4.scaled(n=n, d=d, m=m)
    cfg = type(cfg)(cfg.name, "csr", n, d, m, s, 11, False, nnz_row=k)
    rp, ci, v = gen.csr(cfg)
    b = gen.rhs(cfg)
    bl = skh().hash_gen(cfg.seed, m, s, n)
    SA, Sb = skh().sketch_csr(bl, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                              torch.from_numpy(v).cuda(), d, torch.from_numpy(b).cuda())
    SAo, Sbo = sketch.sketch_csr(cfg.seed, rp, ci, v, d, b, m, s)
    assert_same(np_(SA), SAo)
    assert_same(np_(Sb), Sbo)


def test_sketch_csr_C4_full_sampled_buckets():
    from oracle import sketch
    from synth import configs, device, gen
    cfg = configs.C4
    rp, ci, v = device.csr(cfg)
    b = device.rhs(cfg)
    bl = skh().hash_gen(cfg.seed, cfg.m, cfg.s, cfg.n)
    SA, Sb = skh().sketch_csr(bl, rp, ci, v, cfg.d, b)
    hrp, hci, hv = gen.csr(cfg)
    assert np.array_equal(np_(ci), hci) and np.array_equal(np_(v), hv)
    buckets = [0, 1, 8191, 16383]
    SAo, Sbo = sketch.sketch_csr(cfg.seed, hrp, hci, hv, cfg.d, gen.rhs(cfg), cfg.m, cfg.s, buckets=buckets)
    assert_same(np_(SA[buckets]), SAo)
    assert_same(np_(Sb[buckets]), Sbo)


# ------------------------------------------------------------------ R3 + R4
@pytest.mark.parametrize("nrows,nvalid,d,lo,hi,diag,row0", [
    (1, 1, 1, 0, 0, True, 0), (2, 2, 1, 0, 1, True, 0), (8, 5, 3, 0, 3, True, 7), (256, 256, 64, 0, 8, True, 0),
    (4096, 4096, 64, 0, 12, True, 0), (4096, 3000, 64, 0, 12, True, 100), (1024, 1024, 32, 3, 9, False, 0),
    (2048, 2048, 18, 0, 11, True, 64), (1 << 16, 1 << 16, 16, 0, 16, True, 0), (512, 512, 130, 0, 9, True, 0),
    (8192, 8192, 2, 0, 13, True, 5),
    # single wide tile passes (K = 9, 10, 11), ragged column tiles, lo > 0, padding
    (512, 512, 64, 0, 9, True, 0), (1024, 1024, 70, 0, 10, True, 3), (2048, 2000, 64, 0, 11, True, 0),
    (4096, 4096, 96, 1, 11, False, 0), (8192, 8192, 32, 2, 13, True, 1 << 20), (1 << 12, 3333, 200, 0, 11, True, 64)])
def test_rht_stages(nrows, nvalid, d, lo, hi, diag, row0):
    from oracle import hadamard
    r = np.random.default_rng(nrows + d)
    X = r.standard_normal((nvalid, d))
    Y = skh().rht_stages(77, torch.from_numpy(X).cuda(), lo, hi, nrows=nrows, row0=row0, apply_diag=diag, alpha=1.0)
    Z = np.zeros((nrows, d))
    Z[:nvalid] = X
    if diag:
        Z[:nvalid] *= hadamard.diag_signs(77, np.arange(row0, row0 + nvalid))[:, None].astype(float)
    hadamard.fwht_stages(Z, lo, hi)
    assert_same(np_(Y), Z)


def test_rht_stages_normalised_in_place():
    from oracle import sketch
    n, d = 1024, 64
    X = np.random.default_rng(5).standard_normal((n, d))
    Xt = torch.from_numpy(X).cuda()
    skh().rht_stages(3, Xt, 0, 10, apply_diag=True, alpha=skh().c_n(n), Y=Xt)
    assert_same(np_(Xt), sketch.hda(3, X))


# ------------------------------------------------------------------ R1-R5 HRHT
@pytest.mark.parametrize("n,d,m,s", [(1, 1, 1, 1), (5, 3, 4, 1), (100, 7, 16, 2), (1000, 64, 112, 1),
                                     (8192, 128, 224, 1), (4096, 64, 256, 2), (3000, 33, 50, 3)])
def test_rht_dense(n, d, m, s):
    from oracle import sketch
    r = np.random.default_rng(n + 3 * d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    SA, Sb = skh().rht_dense(21, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), m, s)
    SAo, Sbo = sketch.rht_sketch(21, A, b, m, s)
    assert_same(np_(SA), SAo)
    assert_same(np_(Sb), Sbo)


def test_rht_dense_C2_full_sampled_columns():
    from oracle import sketch
    from synth import configs, device, gen
    cfg = configs.C2
    A = device.dense(cfg)
    b = device.rhs(cfg)
    SA, Sb = skh().rht_dense(cfg.seed, A, b, cfg.m, cfg.s)
    cols = [0, 511, 1023]
    SAo = sketch.rht_sketch_columns(cfg.seed, lambda c: gen.dense_block(cfg, 0, cfg.n, c), cfg.n, cfg.m, cfg.s, cols)
    assert_same(np_(SA[:, cols]), SAo)
    _, Sbo = sketch.rht_sketch(cfg.seed, np.zeros((cfg.n, 1)), gen.rhs(cfg), cfg.m, cfg.s)
    assert_same(np_(Sb), Sbo)


def test_rht_dense_C3HD_full_sampled_columns():
    from oracle import sketch
    from synth import configs, device, gen
    cfg = configs.C3HD
    A = device.dense(cfg)
    SA, _ = skh().rht_dense(cfg.seed, A, None, cfg.m, cfg.s)
    cols = [0, 4095]
    SAo = sketch.rht_sketch_columns(cfg.seed, lambda c: gen.dense_block(cfg, 0, cfg.n, c), cfg.n, cfg.m, cfg.s, cols)
    assert_same(np_(SA[:, cols]), SAo)


def test_rht_dense_C5_full_sampled_columns():
    """C5 at full size (64 GiB A on one GPU) in the launch configuration bench.py
    times (RhtDense workspace), checked on sampled columns."""
    from oracle import sketch
    from synth import configs, device, gen
    cfg = configs.C5
    A = device.dense(cfg)
    b = device.rhs(cfg)
    op = skh().RhtDense(cfg.n, cfg.m, cfg.s, cfg.d)
    SA, Sb = op(cfg.seed, A, b)
    cols = [0, 4095]
    SAo = sketch.rht_sketch_columns(cfg.seed, lambda c: gen.dense_block(cfg, 0, cfg.n, c), cfg.n, cfg.m, cfg.s, cols)
    assert_same(np_(SA[:, cols]), SAo)
    _, Sbo = sketch.rht_sketch(cfg.seed, np.zeros((cfg.n, 1)), gen.rhs(cfg), cfg.m, cfg.s)
    assert_same(np_(Sb), Sbo)
    del A, op
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ host-buffer entry points
def test_host_variants_match_device():
    from synth import configs, gen
    cfg = configs.C2.scaled(n=5000, d=96, m=168)
    A = torch.from_numpy(gen.dense(cfg)).pin_memory()
    b = torch.from_numpy(gen.rhs(cfg)).pin_memory()
    op = skh().RhtDense(cfg.n, cfg.m, cfg.s, cfg.d)
    SAd, Sbd = op(cfg.seed, A.cuda(), b.cuda())
    SAh, Sbh = op.from_host(cfg.seed, A, b)
    assert np.array_equal(np_(SAd), SAh.numpy()) and np.array_equal(np_(Sbd), Sbh.numpy())
    cfg1 = configs.C1
    A1 = torch.from_numpy(gen.dense(cfg1)).pin_memory()
    b1 = torch.from_numpy(gen.rhs(cfg1)).pin_memory()
    bl = skh().hash_gen(cfg1.seed, cfg1.m, cfg1.s, cfg1.n)
    SAd, Sbd = skh().sketch_dense(bl, A1.cuda(), b1.cuda())
    SAh, Sbh = skh().SketchDenseHost(cfg1.n, cfg1.m, cfg1.s, cfg1.d)(cfg1.seed, A1, b1)
    assert np.array_equal(np_(SAd), SAh.numpy()) and np.array_equal(np_(Sbd), Sbh.numpy())


def test_integer_mode_order_independent():
    """Integer inputs: SA == fl(c * exact integer sum) for every path."""
    import math
    from oracle import hadamard, hashing
    from synth import gen
    n, d, m, s = 2048, 24, 60, 2
    A = gen.small_int_dense(8, n, d)
    SA, _ = skh().rht_dense(4, torch.from_numpy(A).cuda(), None, m, s)
    Sint = np.rint(hashing.dense_S(4, n, m, s) * math.sqrt(s)).astype(np.int64)
    X = hadamard.fwht(hadamard.diag_signs(4, np.arange(n))[:, None].astype(float) * A).astype(np.int64)
    T = Sint @ X
    assert np.array_equal(np_(SA), (1.0 / math.sqrt(n * s)) * T.astype(np.float64))


def test_deterministic_rerun():
    from synth import configs, device
    cfg = configs.C2.scaled(n=16384, d=256, m=448)
    A = device.dense(cfg)
    op = skh().RhtDense(cfg.n, cfg.m, cfg.s, cfg.d)
    S1, _ = op(cfg.seed, A)
    S2, _ = op(cfg.seed, A)
    assert torch.equal(S1, S2)


def test_synth_device_matches_host():
    from synth import configs, device, gen
    for name in ("C1", "C3"):
        cfg = configs.ALL[name].scaled(n=5000, d=300)
        assert np.array_equal(np_(device.dense(cfg)), gen.dense(cfg))
        assert np.array_equal(np_(device.rhs(cfg)), gen.rhs(cfg))
    cfg = configs.C4.scaled(n=3000, d=500)
    rp, ci, v = device.csr(cfg, 100, 2100)
    hrp, hci, hv = gen.csr_rows(cfg, 100, 2100)
    assert np.array_equal(np_(rp), hrp) and np.array_equal(np_(ci), hci) and np.array_equal(np_(v), hv)
    assert np.array_equal(np_(device.small_int(5, 70, 9)), gen.small_int_dense(5, 70, 9))
