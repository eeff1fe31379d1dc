"""HR-DHT sketch S_h F D (eq. (6.1)) through the C ABI vs
oracle/hartley.py.  The FFT rounds differently from numpy's: SA, Sb compared to
the BASELINE tolerance (relative Frobenius <= 1e-12); integer inputs are not
exact under an FFT, so no bitwise mode here."""
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


CASES = [(1, 1, 1, 1), (2, 3, 2, 1), (7, 2, 5, 2), (100, 17, 16, 2), (1000, 64, 112, 1), (4097, 33, 200, 3),
         (65536, 8, 448, 1), (100003, 3, 1000, 2)]
# n = 2^L, 2 <= L <= 18: the two-pass transforms of csrc/fht.cu (row-major: every
# tile size 2..512, column tiles 8/16 with ragged tails; column-major from n = 256;
# the 2^19 cuFFT fallback)
POW2 = [(4, 1, 2, 1), (8, 15, 4, 2), (16, 16, 8, 1), (32, 17, 8, 3), (512, 33, 64, 2), (1024, 7, 100, 1),
        (4096, 40, 300, 2), (1 << 17, 9, 700, 2), (1 << 18, 5, 800, 1), (1 << 19, 2, 900, 1)]


@pytest.mark.parametrize("n,d,m,s", CASES + POW2)
def test_hrdht_rowmajor(n, d, m, s):
    from oracle import hartley
    r = np.random.default_rng(n + d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    SA, Sb = skh().hrdht_dense(13, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), m, s)
    SAo, Sbo = hartley.hrdht_sketch(13, A, b, m, s)
    assert rel(np_(SA), SAo) <= TOL and rel(np_(Sb), Sbo) <= TOL


@pytest.mark.parametrize("n,d,m,s", CASES + POW2)
def test_hrdht_colmajor(n, d, m, s):
    from oracle import hartley
    r = np.random.default_rng(n + 2 * d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    SAt, Sb = skh().hrdht_dense_colmajor(13, At, torch.from_numpy(b).cuda(), m, s)
    SAo, Sbo = hartley.hrdht_sketch(13, A, b, m, s)
    assert rel(np_(SAt).T, SAo) <= TOL and rel(np_(Sb), Sbo) <= TOL


@pytest.mark.parametrize("n", [3000, 4096])
def test_hrdht_no_b_deterministic_and_padded_ld(n):
    from oracle import hartley
    d, m, s = 5, 64, 2
    A = np.random.default_rng(3).standard_normal((n, d))
    buf = torch.zeros(n, d + 3, dtype=torch.float64, device="cuda")
    buf[:, :d] = torch.from_numpy(A)
    S1, Sb = skh().hrdht_dense(4, buf[:, :d], None, m, s)
    assert Sb is None
    S2, _ = skh().hrdht_dense(4, buf[:, :d], None, m, s)
    assert torch.equal(S1, S2)
    assert rel(np_(S1), hartley.hrdht_sketch(4, A, None, m, s)[0]) <= TOL


def test_hrdht_C2_full_sampled_columns():
    """C2's shape (65536 x 1024, m = 1792, s = 1) with the paper's own transform."""
    from oracle import hartley
    from synth import configs, device, gen
    cfg = configs.C2
    A = device.dense(cfg)
    b = device.rhs(cfg)
    SA, Sb = skh().hrdht_dense(cfg.seed, A, b, cfg.m, cfg.s)
    cols = [0, 777, 1023]
    SAo, _ = hartley.hrdht_sketch(cfg.seed, gen.dense_block(cfg, 0, cfg.n, cols), None, cfg.m, cfg.s)
    assert rel(np_(SA[:, cols]), SAo) <= TOL
    _, Sbo = hartley.hrdht_sketch(cfg.seed, np.zeros((cfg.n, 1)), gen.rhs(cfg), cfg.m, cfg.s)
    assert rel(np_(Sb), Sbo) <= TOL


@pytest.mark.parametrize("n,d,m", [(1, 1, 1), (100, 7, 30), (4000, 40, 700), (4097, 3, 5), (30000, 16, 50),
                                   (8192, 20, 100)])
def test_srdht(n, d, m):
    """SR-DHT (eq. (7.2)) vs oracle/sampling.py."""
    from oracle import sampling
    r = np.random.default_rng(n + d)
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    SA, Sb = skh().srdht_dense(21, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), m)
    SAo, Sbo = sampling.srdht_sketch(21, A, b, m)
    assert rel(np_(SA), SAo) <= TOL and rel(np_(Sb), Sbo) <= TOL


def test_fig1_claim_at_paper_size():
    """Fig. 1 at the paper's size: coherent A = [I; 0] + 1e-8 J
    (eq. (7.4)), n = 4000, d = 400.  With the GPU sketches, kappa(A R^{-1})
    (QR without pivoting) is smaller with hashing (HR-DHT, s = 1) than with
    sampling (SR-DHT) at m/d in {1.5, 2, 3} for the median over seeds, and the
    hashing kappa at m/d = 1.5 is already modest."""
    from oracle import sampling
    n, d = 4000, 400
    A = torch.from_numpy(sampling.coherent_A(n, d)).cuda()

    def kappa(SA):
        R = torch.linalg.qr(SA, mode="r")[1]
        sv = torch.linalg.svdvals(torch.linalg.solve_triangular(R, A, upper=True, left=False))
        return float(sv[0] / sv[-1])

    for ratio in (1.5, 2.0, 3.0):
        m = int(ratio * d)
        kh = [kappa(skh().hrdht_dense(sd, A, None, m, 1)[0]) for sd in range(5)]
        ks = [kappa(skh().srdht_dense(sd, A, None, m)[0]) for sd in range(5)]
        assert np.median(kh) < np.median(ks)
    assert np.median([kappa(skh().hrdht_dense(sd, A, None, 600, 1)[0]) for sd in range(5)]) < 20
