"""Column-major path (include/skh.h "Column-major A") through the C ABI vs the
CPU oracle, element by element.

* skh_rht_colmajor (H D A alone): stages low bit to high bit as the oracle ->
  bit-exact.
* skh_sketch_dense_colmajor: tiles are consecutive row blocks, so every bucket
  sums in ascending row order -> bit-exact.
* skh_rht_dense_colmajor: the gather is fused into the last transform pass and
  a bucket receives its rows tile by tile (R17), so SA is compared
  against the BASELINE.json tolerance (relative Frobenius <= 1e-12), bit-exactly
  on integer inputs (every partial sum is an exact integer), and bitwise
  against itself run to run.
The oracle works on plain (n, d) arrays: layout is storage only.
"""
import math

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


def rel(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    return np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)


def assert_bitexact(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    assert rel(got, want) <= TOL
    assert np.array_equal(got.view(np.int64), want.view(np.int64)), "not bit-identical to the oracle"


def cm(A, pad=0):
    """Column-major device copy of the (n, d) array A: a (d, n + pad) tensor."""
    n, d = A.shape
    At = torch.zeros(d, n + pad, dtype=torch.float64, device="cuda")
    At[:, :n] = torch.from_numpy(np.ascontiguousarray(A.T))
    return At[:, :n] if pad == 0 else At[:, :n]


# ------------------------------------------------------------------ R3 + R4
@pytest.mark.parametrize("nrows,nvalid,d,diag,row0", [
    (1, 1, 1, True, 0), (2, 2, 3, True, 0), (8, 5, 2, True, 7), (4096, 4096, 3, True, 0), (4096, 3001, 2, True, 64),
    (8192, 8192, 3, True, 0), (8192, 8000, 1, True, 5), (16384, 16384, 3, True, 0), (1 << 15, 30000, 2, False, 0),
    (1 << 17, 1 << 17, 2, True, 1 << 20), (1 << 21, 1 << 21, 1, True, 0), (1 << 22, (1 << 22) - 5, 1, True, 0)])
def test_rht_colmajor_bitexact(nrows, nvalid, d, diag, row0):
    """Pass 1 (13 contiguous bits, D fused), in-place mid passes and the last
    pass, at L = 0 .. 22 with ragged nvalid and global row offsets."""
    from oracle import hadamard
    r = np.random.default_rng(nrows + d)
    X = r.standard_normal((nvalid, d))
    Yt = skh().rht_colmajor(77, cm(X), nrows=nrows, row0=row0, apply_diag=diag)
    Z = np.zeros((nrows, d))
    Z[:nvalid] = X
    if diag:
        Z[:nvalid] *= hadamard.diag_signs(77, np.arange(row0, row0 + nvalid))[:, None].astype(float)
    hadamard.fwht_stages(Z, 0, nrows.bit_length() - 1)
    assert_bitexact(np_(Yt).T, Z)


def test_rht_colmajor_in_place_odd_ld():
    from oracle import hadamard
    n, d = 1 << 14, 3
    X = np.random.default_rng(1).standard_normal((n, d))
    buf = torch.zeros(d, n + 1, dtype=torch.float64, device="cuda")  # odd leading dimension: scalar path
    buf[:, :n] = torch.from_numpy(np.ascontiguousarray(X.T))
    Xt = buf[:, :n]
    skh().rht_colmajor(5, Xt, Yt=Xt)
    Z = X * hadamard.diag_signs(5, np.arange(n))[:, None].astype(float)
    hadamard.fwht_stages(Z, 0, 14)
    assert_bitexact(np_(Xt).T, Z)


# ------------------------------------------------------------------ plain s-hashing, column-major
@pytest.mark.parametrize("n,d,m,s", [(1, 1, 1, 1), (3, 2, 2, 1), (65, 3, 7, 3), (4096, 64, 256, 2), (4097, 5, 40, 2),
                                     (10000, 17, 300, 1), (20000, 4, 10000, 1), (9000, 3, 9000, 2), (3000, 2, 64, 8)])
def test_sketch_dense_colmajor_bitexact(n, d, m, s):
    from oracle import sketch
    r = np.random.default_rng(n * 7 + d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    SAt, Sb = skh().sketch_dense_colmajor(42, cm(A), torch.from_numpy(b).cuda(), m, s)
    SAo, Sbo = sketch.sketch_dense(42, A, b, m, s)
    assert_bitexact(np_(SAt).T, SAo)
    assert_bitexact(np_(Sb), Sbo)


def test_sketch_dense_colmajor_no_b_and_ld():
    from oracle import sketch
    n, d, m, s = 5000, 6, 100, 2
    A = np.random.default_rng(2).standard_normal((n, d))
    buf = torch.zeros(d, n + 3, dtype=torch.float64, device="cuda")
    buf[:, :n] = torch.from_numpy(np.ascontiguousarray(A.T))
    SAbuf = torch.full((d, m + 5), 7.0, dtype=torch.float64, device="cuda")
    SAt, Sb = skh().sketch_dense_colmajor(9, buf[:, :n], None, m, s, SAt=SAbuf[:, :m])
    assert Sb is None
    SAo, _ = sketch.sketch_dense(9, A, None, m, s)
    assert_bitexact(np_(SAt).T, SAo)
    assert (np_(SAbuf[:, m:]) == 7.0).all()


def test_sketch_dense_colmajor_C3_full_sampled_columns():
    """C3 at full size (4 GiB, s = 2) stored column-major: bit-exact on sampled columns."""
    from oracle import sketch
    from synth import configs, device, gen
    cfg = configs.C3
    At = device.dense_colmajor(cfg)
    b = device.rhs(cfg)
    SAt, Sb = skh().sketch_dense_colmajor(cfg.seed, At, b, cfg.m, cfg.s)
    cols = [0, 1, 2047, 4095]
    SAo, Sbo = sketch.sketch_dense(cfg.seed, gen.dense_block(cfg, 0, cfg.n, cols), gen.rhs(cfg), cfg.m, cfg.s)
    assert_bitexact(np_(SAt[cols]).T, SAo)
    assert_bitexact(np_(Sb), Sbo)
    del At
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ HRHT, column-major
@pytest.mark.parametrize("n,d,m,s", [(1, 1, 1, 1), (5, 3, 4, 1), (100, 7, 16, 2), (1000, 64, 112, 1),
                                     (4096, 64, 256, 2), (8192, 9, 224, 1), (8193, 3, 300, 2), (16384, 16, 500, 1),
                                     (40000, 5, 700, 3), (1 << 17, 4, 7168, 2), (1 << 18, 3, 12000, 1),
                                     (1 << 21, 2, 7168, 1), ((1 << 22) - 3, 1, 400, 1), (20000, 3, 64, 8)])
def test_rht_dense_colmajor_tolerance(n, d, m, s):
    """Every pass plan: L <= 12 (one small pass), 13 (no fused stages), 14..21
    (K2 = 1..8 fused stages), 22 (an in-place mid pass); m above the on-chip
    bucket range (several gather launches); s up to 8."""
    from oracle import sketch
    r = np.random.default_rng(n + 3 * d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    SAt, Sb = skh().rht_dense_colmajor(21, cm(A), torch.from_numpy(b).cuda(), m, s)
    SAo, Sbo = sketch.rht_sketch(21, A, b, m, s)
    assert rel(np_(SAt).T, SAo) <= TOL
    assert rel(np_(Sb), Sbo) <= TOL


@pytest.mark.parametrize("n,d,m,s", [(2048, 24, 60, 2), (1 << 17, 3, 1000, 1), (1 << 21, 1, 7168, 1),
                                     (50000, 4, 500, 3),
                                     # >= 2 x 148 columns and a small sketch: two columns per CTA in the
                                     # fused pass (the odd count leaves the last CTA a dummy column)
                                     (1 << 14, 300, 500, 1), (1 << 16, 301, 1792, 2)])
def test_rht_dense_colmajor_integer_exact(n, d, m, s):
    """Integer inputs: every butterfly and partial sum is an exact integer, so the
    fused path equals fl(c_ns * exact integer sum) bit for bit."""
    from oracle import hadamard, hashing, sketch
    from synth import gen
    A = gen.small_int_dense(8, n, d)
    b = gen.small_int_dense(9, n, 1)[:, 0]
    SAt, Sb = skh().rht_dense_colmajor(4, cm(A), torch.from_numpy(b).cuda(), m, s)
    n_pad = hadamard.next_pow2(n)
    Z = np.zeros((n_pad, d + 1))
    Z[:n, :d] = A
    Z[:n, d] = b
    Z[:n] *= hadamard.diag_signs(4, np.arange(n))[:, None].astype(float)
    X = hadamard.fwht(Z)
    assert np.abs(X).max() < 2 ** 40
    ptr, rows, signs = hashing.bucket_lists(4, np.arange(n_pad), m, s)
    T = sketch.bucket_sum(X, ptr, rows, signs, 1.0)  # exact: integers < 2^53
    c = 1.0 / math.sqrt(float(n_pad) * float(s))
    assert np.array_equal(np_(SAt).T, c * T[:, :d])
    assert np.array_equal(np_(Sb), c * T[:, d])


def test_rht_dense_colmajor_deterministic_and_host():
    from synth import configs, device
    cfg = configs.C2.scaled(n=1 << 16, d=64, m=448)
    At = device.dense_colmajor(cfg)
    b = device.rhs(cfg)
    op = skh().RhtDenseColMajor(cfg.n, cfg.m, cfg.s, cfg.d)
    S1, b1 = op(cfg.seed, At, b)
    S1, b1 = S1.clone(), b1.clone()
    S2, b2 = op(cfg.seed, At, b)
    assert torch.equal(S1, S2) and torch.equal(b1, b2)
    SAh, Sbh = op.from_host(cfg.seed, At.cpu().pin_memory(), b.cpu().pin_memory())
    assert np.array_equal(np_(S1), SAh.numpy()) and np.array_equal(np_(b1), Sbh.numpy())


@pytest.mark.parametrize("name,cols", [("C2", [0, 511, 1023]), ("C3HD", [0, 4095])])
def test_rht_dense_colmajor_full_sampled_columns(name, cols):
    from oracle import sketch
    from synth import configs, device, gen
    cfg = configs.ALL[name]
    At = device.dense_colmajor(cfg)
    b = device.rhs(cfg)
    SAt, Sb = skh().rht_dense_colmajor(cfg.seed, At, b, cfg.m, cfg.s)
    SAo = sketch.rht_sketch_columns(cfg.seed, lambda c: gen.dense_block(cfg, 0, cfg.n, c), cfg.n, cfg.m, cfg.s, cols)
    assert rel(np_(SAt[cols]).T, SAo) <= TOL
    _, Sbo = sketch.rht_sketch(cfg.seed, np.zeros((cfg.n, 1)), gen.rhs(cfg), cfg.m, cfg.s)
    assert rel(np_(Sb), Sbo) <= TOL
    del At
    torch.cuda.empty_cache()


def test_rht_dense_colmajor_C5_full_sampled_columns():
    """C5 at full size (64 GiB A, column-major, one GPU) in the launch
    configuration bench.py times (RhtDenseColMajor workspace)."""
    from oracle import sketch
    from synth import configs, device, gen
    cfg = configs.C5
    At = device.dense_colmajor(cfg)
    b = device.rhs(cfg)
    op = skh().RhtDenseColMajor(cfg.n, cfg.m, cfg.s, cfg.d)
    SAt, Sb = op(cfg.seed, At, b)
    cols = [0, 4095]
    SAo = sketch.rht_sketch_columns(cfg.seed, lambda c: gen.dense_block(cfg, 0, cfg.n, c), cfg.n, cfg.m, cfg.s, cols)
    assert rel(np_(SAt[cols]).T, SAo) <= TOL
    _, Sbo = sketch.rht_sketch(cfg.seed, np.zeros((cfg.n, 1)), gen.rhs(cfg), cfg.m, cfg.s)
    assert rel(np_(Sb), Sbo) <= TOL
    del At, op
    torch.cuda.empty_cache()


def test_trace_stage_events():
    from synth import configs, device
    cfg = configs.C2.scaled(n=1 << 15, d=32, m=112)
    At = device.dense_colmajor(cfg)
    op = skh().RhtDenseColMajor(cfg.n, cfg.m, cfg.s, cfg.d)
    with skh().api.Trace(8) as tr:
        op(cfg.seed, At)
    torch.cuda.synchronize()
    # hash + tile lists run on the library's side stream beside pass 1
    assert tr.names == ["begin", "side:hash_gen", "side:tile_lists", "pass1", "side_wait", "pass2_gather"]
    ms = tr.durations_ms()
    assert all(v >= 0 for v in ms.values())
    assert set(ms) == {"hash_gen (overlapped)", "tile_lists (overlapped)", "pass1", "side_wait", "pass2_gather"}


def test_determinism_stress_shared_memory_paths():
    """compute-sanitizer is not available on this pool (SURVEY §5 asks for
    racecheck); the kernels use no floating-point atomics, so a shared-memory
    race would show up as run-to-run differences: five reruns of every
    scatter-style path must be bitwise equal."""
    from synth import configs, device, gen
    cfg = configs.C2.scaled(n=1 << 15, d=33, m=300)
    At = device.dense_colmajor(cfg)
    b = device.rhs(cfg)
    runs = [skh().rht_dense_colmajor(cfg.seed, At, b, cfg.m, 2) for _ in range(5)]
    runs2 = [skh().sketch_dense_colmajor(cfg.seed, At, b, cfg.m, 3) for _ in range(5)]
    c4 = configs.C4.scaled(n=20000, d=500, m=100)
    rp, ci, v = (torch.from_numpy(x).cuda() for x in gen.csr(c4))
    bl = skh().hash_gen(c4.seed, c4.m, c4.s, c4.n)
    runs3 = [skh().sketch_csr(bl, rp, ci, v, c4.d) for _ in range(5)]
    # the count-based CSR reduce (every bucket's run fits in registers)
    bl2 = skh().hash_gen(c4.seed, 2000, c4.s, c4.n)
    runs4 = [skh().sketch_csr(bl2, rp, ci, v, c4.d) for _ in range(5)]
    # the on-chip walk of the plain column-major sketch (small workspace)
    runs5 = [skh().sketch_dense_colmajor(cfg.seed, At, b, cfg.m, 3, fast=False) for _ in range(5)]
    # K2 = 8 (two-CTA pass 2) and K2 = 4 (warp-specialised) column-major transforms
    c8 = configs.C5.scaled(n=1 << 21, d=2, m=700)
    At8 = device.dense_colmajor(c8)
    runs6 = [skh().rht_dense_colmajor(c8.seed, At8, None, c8.m, 1) for _ in range(5)]
    c4b = configs.C5.scaled(n=1 << 17, d=5, m=700)
    At4 = device.dense_colmajor(c4b)
    runs7 = [skh().rht_dense_colmajor(c4b.seed, At4, None, c4b.m, 2) for _ in range(5)]
    # the HR-DHT passes (shared-memory FFT rounds)
    A2 = device.dense(configs.C2.scaled(n=1 << 14, d=40, m=100))
    runs8 = [skh().hrdht_dense(3, A2, None, 100, 2) for _ in range(5)]
    # the 16-lane row gather (s > 1, 64-column slices) and the M3 rank step with
    # folded lists (two-team pass 1 + fused pass 2 with s_eff = 2 draws per row)
    c3 = configs.C3.scaled(n=20000, d=256, m=300)
    A3 = device.dense(c3)
    bl3 = skh().hash_gen(c3.seed, c3.m, c3.s, c3.n)
    runs9 = [skh().sketch_dense(bl3, A3, device.rhs(c3)) for _ in range(5)]
    api = skh().api
    cm3 = configs.C5.scaled(n=1 << 18, d=3, m=700)
    L = cm3.n // 2
    Atm = device.dense_colmajor(cm3, L, cm3.n)
    blc = api.hash_gen(cm3.seed, cm3.m, 1, cm3.n, want_cols=True)
    f = api.fold_cols(blc.col_rows, blc.col_signs, L, 2, 1, 1)
    opm = api.RhtColMajorLists(L, cm3.m, 2, cm3.d)
    runs10 = [tuple(t.clone() for t in opm(cm3.seed, Atm, None, L, f[0], f[1])[:1]) + (None,) for _ in range(5)]
    for rr in (runs, runs2, runs3, runs4, runs5, runs6, runs7, runs8, runs9, runs10):
        for SA, Sb in rr[1:]:
            assert torch.equal(SA, rr[0][0])
            if Sb is not None:
                assert torch.equal(Sb, rr[0][1])


@pytest.mark.parametrize("n,d,m,s", [(5000, 3, 300, 2), (4096 * 3 + 17, 70, 1000, 1), (9000, 129, 64, 8)])
def test_plain_colmajor_fast_and_walk_bit_identical(n, d, m, s):
    """skh_sketch_dense_colmajor's two paths (transpose + row gather when the
    workspace has room for a row-major copy, else the on-chip walk) are both
    bit-identical to the oracle."""
    import numpy as np
    from oracle import sketch
    r = np.random.default_rng(n + d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    bd = torch.from_numpy(b).cuda()
    SAo, Sbo = sketch.sketch_dense(5, A, b, m, s)
    for fast in (True, False):
        SAt, Sb = skh().sketch_dense_colmajor(5, At, bd, m, s, fast=fast)
        assert np.array_equal(SAt.cpu().numpy().T.view(np.int64), SAo.view(np.int64))
        assert np.array_equal(Sb.cpu().numpy().view(np.int64), Sbo.view(np.int64))


@pytest.mark.parametrize("n,d,m,s", [(1 << 15, 33, 300, 1), (40000, 5, 700, 3), (1 << 14, 64, 112, 8)])
def test_rht_colmajor_lists_equals_composite(n, d, m, s):
    """skh_rht_colmajor_lists fed the hash's own column lists (row0 = 0, alpha =
    c_ns) is the composite skh_rht_dense_colmajor, bit for bit; and a folded
    pair of half-size calls (M3 with G = 2 on one GPU) sums to the oracle."""
    from oracle import sketch
    from synth import configs, device, gen
    api = skh().api
    cfg = configs.C2.scaled(n=n, d=d, m=m)
    At = device.dense_colmajor(cfg)
    b = device.rhs(cfg)
    SAt, Sb = skh().RhtDenseColMajor(n, m, s, d)(cfg.seed, At, b)
    n_pad = 1 << (n - 1).bit_length()
    bl = api.hash_gen(cfg.seed, m, s, n_pad, want_cols=True)  # lists of every row of the padded transform
    op = api.RhtColMajorLists(n, m, s, d)
    SAt2, Sb2 = op(cfg.seed, At, b, 0, bl.col_rows, bl.col_signs, alpha=api.c_ns(n_pad, s))
    assert torch.equal(SAt, SAt2) and torch.equal(Sb, Sb2)
    if s <= 4 and n == n_pad:
        L = n // 2
        opL = api.RhtColMajorLists(L, m, 2 * s, d)
        parts = []
        for r in range(2):
            f = api.fold_cols(bl.col_rows, bl.col_signs, L, 2, s, r)
            parts.append(opL(cfg.seed, At[:, r * L:(r + 1) * L].contiguous(), b[r * L:(r + 1) * L].contiguous(),
                             r * L, f[0], f[1], alpha=1.0))
        c = api.c_ns(n, s)
        SA3 = (c * (parts[0][0] + parts[1][0])).cpu().numpy().T
        Sb3 = (c * (parts[0][1] + parts[1][1])).cpu().numpy()
        A = gen.dense(cfg)
        want, wantb = sketch.rht_sketch(cfg.seed, A, gen.rhs(cfg), m, s)
        assert np.linalg.norm(SA3 - want) / np.linalg.norm(want) <= 1e-12
        assert np.linalg.norm(Sb3 - wantb) / np.linalg.norm(wantb) <= 1e-12
