"""Edge shapes across the entry points (one bucket, one column, s = m, wide m,
n just above a power of two, empty rows), each against the oracle: bit-exact
where the path keeps the oracle's order, 1e-12 relative otherwise."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-12


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


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def bits(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.int64), np.asarray(b, np.float64).view(np.int64))


@pytest.mark.parametrize("n,d,m,s", [(50000, 3, 1, 1), (3000, 1, 7, 7), (2000, 65, 64, 64), (40000, 2, 60000, 1)])
def test_dense_edges(n, d, m, s):
    """one bucket holding every row (a 50000-entry list), d = 1 with s = m, s = m = 64, m > n."""
    from oracle import sketch
    r = np.random.default_rng(n + d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    bl = skh().hash_gen(3, m, s, n)
    SA, Sb = skh().sketch_dense(bl, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda())
    SAo, Sbo = sketch.sketch_dense(3, A, b, m, s)
    assert bits(np_(SA), SAo) and bits(np_(Sb), Sbo)
    if s <= 8 and m <= 65536:
        SAt, Sbc = skh().sketch_dense_colmajor(3, torch.from_numpy(np.ascontiguousarray(A.T)).cuda(),
                                               torch.from_numpy(b).cuda(), m, s)
        assert bits(np_(SAt).T, SAo) and bits(np_(Sbc), Sbo)


@pytest.mark.parametrize("n,d,m,s", [((1 << 20) + 1, 2, 100, 1), (1 << 12, 1, 1, 1), (5, 200, 3, 2)])
def test_rht_edges(n, d, m, s):
    """n one above a power of two (padded to 2^21), a single bucket, tiny n with wide d."""
    from oracle import sketch
    r = np.random.default_rng(n)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    SA, Sb = skh().rht_dense(8, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), m, s)
    SAo, Sbo = sketch.rht_sketch(8, A, b, m, s)
    assert bits(np_(SA), SAo) and bits(np_(Sb), Sbo)
    SAt, Sbc = skh().rht_dense_colmajor(8, torch.from_numpy(np.ascontiguousarray(A.T)).cuda(),
                                        torch.from_numpy(b).cuda(), m, s)
    assert rel(np_(SAt).T, SAo) <= TOL and rel(np_(Sbc), Sbo) <= TOL


def test_csr_empty_rows_and_one_bucket():
    from oracle import sketch
    n, d, m, s = 3000, 700, 1, 1
    r = np.random.default_rng(5)
    lens = r.integers(0, 4, size=n)          # many empty rows
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    ci = np.concatenate([np.sort(r.choice(d, size=k, replace=False)) for k in lens]).astype(np.int32)
    v = r.standard_normal(rp[-1])
    b = r.standard_normal(n)
    bl = skh().hash_gen(9, m, s, n)
    SA, Sb = skh().sketch_csr(bl, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(v).cuda(),
                              d, torch.from_numpy(b).cuda())
    SAo, Sbo = sketch.sketch_csr(9, rp, ci, v, d, b, m, s)
    assert bits(np_(SA), SAo) and bits(np_(Sb), Sbo)


def test_hrdht_single_row_and_prime_n():
    from oracle import hartley
    for n, d, m in ((1, 3, 2), (7919, 2, 30)):
        A = np.random.default_rng(n).standard_normal((n, d))
        SA, _ = skh().hrdht_dense(1, torch.from_numpy(A).cuda(), None, m, 1)
        SAo, _ = hartley.hrdht_sketch(1, A, None, m, 1)
        assert rel(np_(SA), SAo) <= TOL


def _csr_from_rows(cols_per_row, r):
    n = len(cols_per_row)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum([len(c) for c in cols_per_row], out=rp[1:])
    ci = np.concatenate([np.sort(np.asarray(c, dtype=np.int32)) for c in cols_per_row]).astype(np.int32)
    return rp, ci, r.standard_normal(rp[-1])


@pytest.mark.parametrize("case", ["leader", "heavy", "side_overflow", "two_tiles", "neg_zero"])
def test_csr_reduce_paths(case):
    """csr_reduce_kernel's paths, bit-exact against the oracle: columns of 3..24
    pairs (one thread sums them in list order), a column in every row (over the
    multiplicity cap: claim-round fallback), a side list over capacity, d over one
    4096-column tile, and -0.0 values (0 + v, not v, is stored)."""
    from oracle import sketch
    r = np.random.default_rng(hash(case) & 0xffff)
    if case == "leader":
        n, d, m, s = 2400, 100, 4, 1
        rows = [r.choice(d, size=1, replace=False) for _ in range(n)]
    elif case == "heavy":
        n, d, m, s = 2000, 300, 4, 1
        rows = [np.unique(np.r_[0, r.choice(d, size=1)]) for _ in range(n)]
    elif case == "side_overflow":
        n, d, m, s = 1800, 40, 1, 1
        rows = [r.choice(d, size=1) for _ in range(n)]
    elif case == "two_tiles":
        n, d, m, s = 3000, 9000, 3, 2
        rows = [np.unique(np.r_[r.choice(d, size=3), r.choice(8, size=1), 4096 + r.choice(8, size=1)]) for _ in range(n)]
    else:
        n, d, m, s = 1000, 64, 8, 3
        rows = [r.choice(d, size=4, replace=False) for _ in range(n)]
    rp, ci, v = _csr_from_rows(rows, r)
    if case == "neg_zero":
        v[::3] = -0.0
        v[1::3] = 0.0
    b = r.standard_normal(n)
    bl = skh().hash_gen(17, m, s, n)
    SA, Sb = skh().sketch_csr(bl, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                              torch.from_numpy(v).cuda(), d, torch.from_numpy(b).cuda())
    SAo, Sbo = sketch.sketch_csr(17, rp, ci, v, d, b, m, s)
    assert bits(np_(SA), SAo) and bits(np_(Sb), Sbo)


def test_side_stream_join_orders_sb():
    """skh_sketch_dense / skh_sketch_csr compute Sb on a library side stream;
    the join must order it before later work on the caller's stream (here a
    non-default torch stream that copies Sb right after the call, 20 times)."""
    from oracle import sketch
    n, d, m, s = 20000, 40, 3000, 2
    r = np.random.default_rng(11)
    A = r.standard_normal((n, d))
    bs = [r.standard_normal(n) for _ in range(4)]
    _, Sbo = zip(*[sketch.sketch_dense(6, A[:, :1], bv, m, s) for bv in bs])
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        bl = skh().hash_gen(6, m, s, n)
        Ad = torch.from_numpy(A).cuda()
        outs = []
        for k in range(20):
            bd = torch.from_numpy(bs[k % 4]).cuda()
            SA, Sb = skh().sketch_dense(bl, Ad, bd)
            outs.append(Sb.clone())  # enqueued on st right after the call
    st.synchronize()
    for k, o in enumerate(outs):
        assert bits(np_(o), Sbo[k % 4])


def test_colmajor_paths_without_b():
    """The transposed column-major paths (plain sketch, HR-DHT) with b = None."""
    from oracle import hartley, sketch
    n, d, m, s = 4096, 33, 500, 2
    A = np.random.default_rng(21).standard_normal((n, d))
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    SAt, Sb = skh().sketch_dense_colmajor(3, At, None, m, s)
    assert Sb is None and bits(np_(SAt).T, sketch.sketch_dense(3, A, None, m, s)[0])
    SAt, Sb = skh().hrdht_dense_colmajor(3, At, None, m, s)
    assert Sb is None and rel(np_(SAt).T, hartley.hrdht_sketch(3, A, None, m, s)[0]) <= TOL
