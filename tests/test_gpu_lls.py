"""Algorithm 1 Steps 2-5 through the C ABI (skh_lls_solve) vs the
oracle (oracle/lls.py) on the same SA, Sb (bit-identical to the oracle's by the
sketch parity tests).  LSQR iterates are compared to rounding: the iteration
count within 1 of the oracle's, the least-squares objective ||A x - b|| to 1e-10
relative, Step 3's x_s (a direct solve) to 1e-10.  LSQR without
reorthogonalisation amplifies the rounding differences of two implementations
(cuSOLVER vs LAPACK QR, reduction orders): at exit both iterates are within the
(7.1) tolerance of the solution but not of each other to rounding, so A x is
compared to 10 tau_r relative (P:L1044-1050 bound the A-norm error by tau_r),
and with tau_r -> 0 both must reach the least-squares solution (lstsq) to
1e-9 kappa-scaled."""
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


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def ill_conditioned(n, d, seed, cond=1e4, noise=1.0):
    r = np.random.default_rng(seed)
    U, _ = np.linalg.qr(r.standard_normal((n, d)))
    V, _ = np.linalg.qr(r.standard_normal((d, d)))
    A = (U * np.logspace(0, -np.log10(cond), d)) @ V.T
    b = A @ r.standard_normal(d) + noise * r.standard_normal(n)
    return A, b


def compare(A, b, SA, Sb, cond=10.0, **kw):
    from oracle import lls
    At, bt = torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda()
    xs = torch.empty(A.shape[1], dtype=torch.float64, device="cuda")
    x, info = skh().LlsSolver(A.shape[0], A.shape[1], SA.shape[0])(At, bt, torch.from_numpy(SA).cuda(),
                                                                   torch.from_numpy(Sb).cuda(), x_s=xs, **kw)
    xo, io = lls.solve(A, b, SA, Sb, **kw)
    assert info["step"] == io["step"]
    assert rel(np_(xs), io["x_s"]) <= 1e-10
    assert abs(info["res_s"] - io["res_s"]) <= 1e-10 * io["res_s"] + 1e-13 * np.linalg.norm(b)
    assert abs(info["iters"] - io["iters"]) <= 1
    tau_r = kw.get("tau_r", 1e-6)
    if info["step"] == 4 and info["iters"] < kw.get("it_max", 10000):
        assert rel(A @ np_(x), A @ xo) <= max(10 * tau_r, 1e-9)
    if tau_r <= 1e-13:
        xstar = np.linalg.lstsq(A, b, rcond=None)[0]
        assert rel(np_(x), xstar) <= 1e-9 * max(1.0, cond / 1e3)
    ro = np.linalg.norm(A @ xo - b)
    assert abs(np.linalg.norm(A @ np_(x) - b) - ro) <= 1e-10 * max(ro, 1.0)
    return info, io


@pytest.mark.parametrize("n,d,m,s,cond", [(3000, 40, 120, 2, 1e3), (5000, 64, 109, 1, 1e6), (2000, 7, 14, 3, 10.0),
                                          (4097, 33, 100, 2, 1e2)])
def test_lls_vs_oracle_plain_hashing(n, d, m, s, cond):
    from oracle import sketch
    A, b = ill_conditioned(n, d, n + d, cond)
    SA, Sb = sketch.sketch_dense(5, A, b, m, s)
    info, io = compare(A, b, SA, Sb, cond=cond)
    assert info["step"] == 4 and info["test2"] <= 1e-6


def test_lls_hrht_paper_defaults():
    """Ski-LLS-dense defaults: S_h H D with s = 1, m = 1.7 d."""
    from oracle import sketch
    r = np.random.default_rng(2)
    n, d = 16384, 256
    A = r.standard_normal((n, d))
    b = r.standard_normal(n)
    m = int(1.7 * d)
    SA, Sb = skh().rht_dense(8, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), m, 1)
    SAo, Sbo = sketch.rht_sketch(8, A, b, m, 1)
    assert np.array_equal(np_(SA), SAo) and np.array_equal(np_(Sb), Sbo)
    compare(A, b, SAo, Sbo)


def test_lls_step3_exit_consistent():
    from oracle import sketch
    A, b = ill_conditioned(3000, 20, 1, cond=10.0, noise=0.0)
    SA, Sb = sketch.sketch_dense(3, A, b, 80, 2)
    info, io = compare(A, b, SA, Sb, tau_a=1e-8)
    assert info["step"] == 3 and info["iters"] == 0


def test_lls_it_max_and_tau():
    from oracle import sketch
    A, b = ill_conditioned(2000, 30, 4, cond=1e5)
    SA, Sb = sketch.sketch_dense(6, A, b, 90, 2)
    for it_max in (0, 1, 3):
        info, io = compare(A, b, SA, Sb, cond=1e5, it_max=it_max)
        assert info["iters"] == io["iters"] == it_max
    info, io = compare(A, b, SA, Sb, cond=1e5, tau_r=1e-14)
    assert info["test2"] <= 1e-14


def test_lls_rank_deficient_is_rejected_in_full_rank_mode():
    """The full-rank (DGEQRF) mode refuses a numerically rank-deficient SA -- a
    zero column, and a column that is a linear combination of others (its r_qq
    is ~1e-16 ||SA||, not 0: the relative test catches it)."""
    from oracle import sketch
    for kind in ("zero", "combination"):
        A, b = ill_conditioned(1000, 10, 5)
        if kind == "zero":
            A[:, 3] = 0.0
        else:
            A[:, 6] = 2.0 * A[:, 1] - A[:, 4]
        SA, Sb = sketch.sketch_dense(1, A, b, 40, 2)
        with pytest.raises(Exception, match="rank deficient"):
            skh().lls_solve(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), torch.from_numpy(SA).cuda(),
                            torch.from_numpy(Sb).cuda())


def deficient(n, d, r, seed, scale=1.0):
    """A of exact rank r: r independent columns, d - r combinations, shuffled."""
    g = np.random.default_rng(seed)
    B = scale * g.standard_normal((n, r))
    C = g.standard_normal((r, d - r))
    A = np.ascontiguousarray(np.concatenate([B, B @ C], axis=1)[:, g.permutation(d)])
    return A, g.standard_normal(n)


@pytest.mark.parametrize("n,d,r,m,s", [(2500, 30, 18, 100, 2), (5000, 64, 1, 120, 1), (4096, 200, 150, 350, 2),
                                       (3000, 40, 40, 90, 3), (2000, 12, 0, 30, 1)])
def test_lls_rank_revealing_vs_oracle(n, d, r, m, s):
    """The paper's default Step 2 (R-CPQR, p = max{q : |r_qq| >= 1e-12},
    L1076-1077, L1109-1112) through skh_lls_solve_rr vs oracle/lls.py's
    scipy-dgeqp3 reading: the same rank p; x zero outside the p pivoted
    coordinates; the least-squares objective within 1e-10 of the minimum-norm
    lstsq residual (the objective is unique, x is not); x_s's residual vs the
    oracle's.  r = d: full rank (then also the QR mode's objective); r = 0: A = 0."""
    from oracle import lls, sketch
    A, b = deficient(n, d, r, 7 + d) if r > 0 else (np.zeros((n, d)), np.random.default_rng(1).standard_normal(n))
    SA, Sb = sketch.sketch_dense(3, A, b, m, s)
    At, bt = torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda()
    xs = torch.empty(d, dtype=torch.float64, device="cuda")
    x, info = skh().LlsSolver(n, d, m, rcond=1e-12)(At, bt, torch.from_numpy(SA).cuda(), torch.from_numpy(Sb).cuda(),
                                                    x_s=xs, tau_a=0.0, tau_r=1e-14, it_max=2000)
    xo, io = lls.solve(A, b, SA, Sb, tau_a=0.0, tau_r=1e-14, it_max=2000, rcond=1e-12)
    assert info["rank"] == io["rank"] == np.linalg.matrix_rank(A)
    rmin = np.linalg.norm(A @ np.linalg.lstsq(A, b, rcond=None)[0] - b)
    got = np.linalg.norm(A @ np_(x) - b)
    assert abs(got - rmin) <= 1e-10 * max(rmin, 1.0)
    assert abs(info["res_s"] - io["res_s"]) <= 1e-8 * max(io["res_s"], 1.0)
    p = info["rank"]
    nz = np.nonzero(np_(x))[0]
    assert len(nz) <= p
    if r == d:
        x2, _ = skh().lls_solve(At, bt, torch.from_numpy(SA).cuda(), torch.from_numpy(Sb).cuda(), tau_a=0.0,
                                tau_r=1e-14, it_max=2000)
        assert abs(np.linalg.norm(A @ np_(x2) - b) - got) <= 1e-10 * max(rmin, 1.0)


def test_lls_rank_revealing_rcond_truncation_and_colmajor():
    """rcond between two pivoted diagonals drops exactly the pivots below it
    (same p as the oracle), and the column-major entry point agrees."""
    from oracle import lls, sketch
    A, b = ill_conditioned(3000, 24, 8, cond=1e9)
    SA, Sb = sketch.sketch_dense(2, A, b, 80, 2)
    import scipy.linalg
    R = scipy.linalg.qr(SA, mode="economic", pivoting=True)[1]
    dg = np.abs(np.diag(R))
    rc = float(np.sqrt(dg[-4] * dg[-3]))
    kw = dict(tau_a=0.0, tau_r=1e-12, it_max=3000)
    x, info = skh().LlsSolver(3000, 24, 80, rcond=rc)(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(),
                                                      torch.from_numpy(SA).cuda(), torch.from_numpy(Sb).cuda(), **kw)
    xo, io = lls.solve(A, b, SA, Sb, rcond=rc, **kw)
    assert info["rank"] == io["rank"] == 21
    xc, ic = skh().LlsSolver(3000, 24, 80, rcond=rc)(torch.from_numpy(np.ascontiguousarray(A.T)).cuda(),
                                                     torch.from_numpy(b).cuda(),
                                                     torch.from_numpy(np.ascontiguousarray(SA.T)).cuda(),
                                                     torch.from_numpy(Sb).cuda(), colmajor=True, **kw)
    assert ic["rank"] == 21
    ro = np.linalg.norm(A @ xo - b)
    for xx in (x, xc):
        assert abs(np.linalg.norm(A @ np_(xx) - b) - ro) <= 1e-9 * ro


def test_lls_deterministic_and_C2_full_size():
    """C2 at full size (65536 x 1024, m = 1792, S_h H D, s = 1) vs the oracle;
    two runs bitwise equal."""
    from oracle import lls
    from synth import configs, device
    cfg = configs.C2
    A = device.dense(cfg)
    b = device.rhs(cfg)
    SA, Sb = skh().rht_dense(cfg.seed, A, b, cfg.m, cfg.s)
    solver = skh().LlsSolver(cfg.n, cfg.d, cfg.m)
    x1, i1 = solver(A, b, SA, Sb)
    x1 = x1.clone()
    x2, i2 = solver(A, b, SA, Sb)
    assert torch.equal(x1, x2) and i1 == i2
    xo, io = lls.solve(np_(A), np_(b), np_(SA), np_(Sb))
    assert abs(i1["iters"] - io["iters"]) <= 1
    An, bn = np_(A), np_(b)
    ro = np.linalg.norm(An @ xo - bn)
    assert abs(np.linalg.norm(An @ np_(x1) - bn) - ro) <= 1e-10 * ro


@pytest.mark.parametrize("n,d,m", [(3000, 40, 120), (8193, 17, 60), (20000, 130, 400)])
def test_lls_colmajor_vs_oracle(n, d, m):
    """skh_lls_solve_colmajor on a column-major A and SA (the layout of
    skh_rht_dense_colmajor) against the oracle."""
    from oracle import lls, sketch
    A, b = ill_conditioned(n, d, n, 1e3)
    SA, Sb = sketch.sketch_dense(2, A, b, m, 2)
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    SAt = torch.from_numpy(np.ascontiguousarray(SA.T)).cuda()
    xs = torch.empty(d, dtype=torch.float64, device="cuda")
    x, info = skh().LlsSolver(n, d, m)(At, torch.from_numpy(b).cuda(), SAt, torch.from_numpy(Sb).cuda(), x_s=xs,
                                       colmajor=True)
    xo, io = lls.solve(A, b, SA, Sb)
    assert info["step"] == io["step"] == 4 and abs(info["iters"] - io["iters"]) <= 1
    assert rel(np_(xs), io["x_s"]) <= 1e-10
    assert rel(A @ np_(x), A @ xo) <= 1e-5
    ro = np.linalg.norm(A @ xo - b)
    assert abs(np.linalg.norm(A @ np_(x) - b) - ro) <= 1e-10 * ro


def test_lls_colmajor_pipeline_hrht():
    """The paper's layout end to end: skh_rht_dense_colmajor then the column-major
    solve; the solution matches the row-major pipeline's objective."""
    from synth import configs, device
    cfg = configs.C2.scaled(n=1 << 15, d=128, m=224)
    A = device.dense(cfg)
    b = device.rhs(cfg)
    At = A.t().contiguous()
    SAt, Sb = skh().rht_dense_colmajor(cfg.seed, At, b, cfg.m, cfg.s)
    x, info = skh().LlsSolver(cfg.n, cfg.d, cfg.m)(At, b, SAt, Sb, colmajor=True)
    SA, Sb2 = skh().rht_dense(cfg.seed, A, b, cfg.m, cfg.s)
    x2, info2 = skh().LlsSolver(cfg.n, cfg.d, cfg.m)(A, b, SA, Sb2)
    r1 = torch.linalg.norm(A @ x - b).item()
    r2 = torch.linalg.norm(A @ x2 - b).item()
    assert info["step"] == 4 and abs(info["iters"] - info2["iters"]) <= 1
    assert abs(r1 - r2) <= 1e-10 * r2


@pytest.mark.parametrize("transform", ["dht", "wht"])
def test_ski_lls_dense_composite(transform):
    """Ski-LLS-dense end to end with the paper's defaults (m = 1.7 d, s = 1):
    the objective matches the least-squares optimum to 1e-10 relative
    (tau_r = 1e-6 bounds the A-norm error)."""
    r = np.random.default_rng(11)
    n, d = 10000, 64
    A = r.standard_normal((n, d)) @ np.diag(np.logspace(0, 3, d))
    b = r.standard_normal(n)
    x, info = skh().ski_lls_dense(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), seed=3,
                                  transform=transform)
    xs = np.linalg.lstsq(A, b, rcond=None)[0]
    best = np.linalg.norm(A @ xs - b)
    assert info["step"] == 4 and info["test2"] <= 1e-6
    assert np.linalg.norm(A @ np_(x) - b) <= best * (1 + 1e-10)


@pytest.mark.parametrize("colmajor", [False, True])
def test_lsqr_graph_equals_host_loop(colmajor, monkeypatch):
    """Step 4 runs as one CUDA-graph WHILE loop with the scalar recurrence on the
    device; SKH_LLS_HOSTLOOP=1 selects the host-driven loop.  Same IEEE
    operations in the same order: bit-identical x, same iteration count
    (also with SKH_LLS_RINV=1, where R^{-1} is applied as a GEMV)."""
    from oracle import sketch
    A, b = ill_conditioned(6000, 48, 3, 1e4)
    SA, Sb = sketch.sketch_dense(4, A, b, 150, 2)
    if colmajor:
        args = (torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), torch.from_numpy(b).cuda(),
                torch.from_numpy(np.ascontiguousarray(SA.T)).cuda(), torch.from_numpy(Sb).cuda())
    else:
        args = tuple(torch.from_numpy(x).cuda() for x in (A, b, SA, Sb))
    solver = skh().LlsSolver(6000, 48, 150)
    x1, i1 = solver(*args, colmajor=colmajor)
    x1 = x1.clone()
    monkeypatch.setenv("SKH_LLS_HOSTLOOP", "1")
    x2, i2 = solver(*args, colmajor=colmajor)
    assert i1 == i2 and i1["iters"] > 3
    assert torch.equal(x1, x2)


def test_rinv_mode_same_minimiser():
    """SKH_LLS_RINV=1 (R^{-1} formed once by dtrsm, applied as GEMVs) reaches the
    same least-squares objective as the default back-solves (a subprocess: the
    mode is read once per process)."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, "tests")
import paper_2105_11815_b200 as skh
from oracle import sketch
from test_gpu_lls import ill_conditioned
A, b = ill_conditioned(6000, 48, 3, 1e6)
SA, Sb = sketch.sketch_dense(4, A, b, 150, 2)
x, info = skh.lls_solve(*(torch.from_numpy(v).cuda() for v in (A, b, SA, Sb)))
print(json.dumps({"x": x.cpu().numpy().tolist(), "info": info}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mode in ("0", "1"):
        env = dict(os.environ, SKH_LLS_RINV=mode)
        p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    A, b = ill_conditioned(6000, 48, 3, 1e6)
    r = [np.linalg.norm(A @ np.array(o["x"]) - b) for o in outs]
    best = np.linalg.norm(A @ np.linalg.lstsq(A, b, rcond=None)[0] - b)
    assert all(o["info"]["step"] == 4 for o in outs)
    assert abs(outs[0]["info"]["iters"] - outs[1]["info"]["iters"]) <= 2
    assert max(r) <= best * (1 + 1e-10)


def test_lls_colmajor_tall_two_row_product():
    """Column-major A with n >= 2^19 takes cm_av2_kernel (two rows per thread,
    16-byte column segments; odd n leaves one row for the tail path): the solve
    reaches the least-squares minimiser like the row-major path."""
    from oracle import sketch
    n, d, m = (1 << 19) + 1, 6, 60
    A, b = ill_conditioned(n, d, 7, 1e3)
    SA, Sb = sketch.sketch_dense(3, A, b, m, 2)
    solver = skh().LlsSolver(n, d, m)
    x, info = solver(torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), torch.from_numpy(b).cuda(),
                     torch.from_numpy(np.ascontiguousarray(SA.T)).cuda(), torch.from_numpy(Sb).cuda(), colmajor=True)
    xs = np.linalg.lstsq(A, b, rcond=None)[0]
    best = np.linalg.norm(A @ xs - b)
    assert info["step"] in (3, 4)
    assert np.linalg.norm(A @ np_(x) - b) <= best * (1 + 1e-10)
