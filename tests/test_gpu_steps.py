"""The exact objects bench.py times (bench.build_step -> pipeline.HrhtStep with
its side-stream fork/join, PlainStep, CsrStep, ColStep), run as bench runs them
(warm-up, then timed steps with stage events) on replicas of the BASELINE
workloads, and compared with the oracle (SA, Sb of every column;
L790-801: S_h H D A):
  * row-major paths: bit-identical (kernels keep the oracle's order, R10);
  * column-major fused path (R17 order): 1e-12 relative, bit-identical on
    integer-valued inputs.
"""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2105_11815_b200.build as b
    b.build()


def run_like_bench(step, steps=3):
    for _ in range(2):
        step.run()
    timers = [step.new_timer() for _ in range(steps)]
    out = None
    for k in range(steps):
        out = step.run(timers[k])
    torch.cuda.synchronize()
    for t in timers:
        assert all(v >= 0 for v in t.durations_ms().values())
    return out


REPLICAS = {
    "C2": dict(n=1 << 14, d=96, m=168),      # HrhtStep: [7,7] passes, side stream for hash + H D b
    "C3HD": dict(n=1 << 15, d=130, m=224),   # s = 2, ragged column tile (d = 130)
    "C5": dict(n=1 << 17, d=32, m=112),      # three passes
    "C1": dict(n=4096, d=64, m=256),         # PlainStep s = 2
    "C3": dict(n=20000, d=70, m=224),        # PlainStep, coherent structure, s = 2
    "C4": dict(n=30000, d=500, m=200),       # CsrStep s = 3
}


@pytest.mark.parametrize("name", list(REPLICAS))
def test_bench_step_row_major_bitexact(name):
    import bench
    from oracle import sketch
    from synth import configs, gen
    cfg = configs.ALL[name].scaled(**REPLICAS[name])
    step, inputs = bench.build_step(cfg, torch, "row")
    SA, Sb = run_like_bench(step)
    if cfg.kind == "csr":
        rp, ci, v = gen.csr(cfg)
        want, wantb = sketch.sketch_csr(cfg.seed, rp, ci, v, cfg.d, gen.rhs(cfg), cfg.m, cfg.s)
    elif cfg.hd:
        want, wantb = sketch.rht_sketch(cfg.seed, gen.dense(cfg), gen.rhs(cfg), cfg.m, cfg.s)
    else:
        want, wantb = sketch.sketch_dense(cfg.seed, gen.dense(cfg), gen.rhs(cfg), cfg.m, cfg.s)
    got, gotb = SA.cpu().numpy(), Sb.cpu().numpy()
    assert np.linalg.norm(got - want) <= TOL * np.linalg.norm(want)
    assert np.array_equal(got, want) and np.array_equal(gotb, wantb)


@pytest.mark.parametrize("name", ["C2", "C3HD", "C5", "C3"])
def test_bench_step_column_major(name):
    import bench
    from oracle import sketch
    from synth import configs, gen
    cfg = configs.ALL[name].scaled(**REPLICAS[name])
    step, inputs = bench.build_step(cfg, torch, "col")
    SAt, Sb = run_like_bench(step)
    A, b = gen.dense(cfg), gen.rhs(cfg)
    want, wantb = (sketch.rht_sketch if cfg.hd else sketch.sketch_dense)(cfg.seed, A, b, cfg.m, cfg.s)
    got = SAt.cpu().numpy().T
    assert np.linalg.norm(got - want) <= TOL * np.linalg.norm(want)
    assert np.linalg.norm(Sb.cpu().numpy() - wantb) <= TOL * np.linalg.norm(wantb)
    if not cfg.hd:  # plain column-major sketch keeps the ascending order: bit-identical
        assert np.array_equal(got, want)


def test_bench_col_step_integer_exact():
    """The fused column-major order (R17) is exact on integer inputs."""
    from oracle import sketch
    from paper_2105_11815_b200 import pipeline
    from synth import gen
    n, d, m, s, seed = 1 << 17, 12, 112, 1, 5
    A = gen.small_int_dense(seed, n, d)
    b = gen.small_int_dense(seed + 1, n, 1)[:, 0]
    step = pipeline.ColStep(seed, torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), torch.from_numpy(b).cuda(), m,
                            s, True, record=True)
    SAt, Sb = run_like_bench(step)
    want, wantb = sketch.rht_sketch(seed, A, b, m, s)
    assert np.array_equal(SAt.cpu().numpy().T, want) and np.array_equal(Sb.cpu().numpy(), wantb)


@pytest.mark.parametrize("name,layout", [("C1", "row"), ("C3", "row"), ("C4", "row"), ("C3HD", "row"),
                                         ("C2", "col"), ("C5", "col")])
def test_bench_step_graph_replay(name, layout):
    """bench.py times short steps as replays of the step captured in a CUDA
    graph (bench.capture_step): every replay redraws S and recomputes SA, Sb.
    Replays after the inputs change must give the oracle's sketch of the NEW
    inputs (nothing cached), bit-identical for the row-major paths and to
    1e-12 for the fused column-major one (R17)."""
    import bench
    from oracle import sketch
    from synth import configs, gen
    cfg = configs.ALL[name].scaled(**REPLICAS[name])
    step, inputs = bench.build_step(cfg, torch, layout)
    g, per_step = bench.capture_step(step, torch)
    assert per_step > 0
    if cfg.kind == "csr":
        rp, ci, v = gen.csr(cfg)
        inputs[2].mul_(-2.0)  # new values in place; the captured pointers stay valid
        want, wantb = sketch.sketch_csr(cfg.seed, rp, ci, -2.0 * v, cfg.d, gen.rhs(cfg), cfg.m, cfg.s)
    else:
        inputs[0].mul_(-2.0)
        A = -2.0 * gen.dense(cfg)
        want, wantb = (sketch.rht_sketch if cfg.hd else sketch.sketch_dense)(cfg.seed, A, gen.rhs(cfg), cfg.m, cfg.s)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    out = step.SAt if layout == "col" else step.SA
    got, gotb = out.cpu().numpy(), step.Sb.cpu().numpy()
    if layout == "col":
        got = got.T
        assert np.linalg.norm(got - want) <= TOL * np.linalg.norm(want)
        assert np.linalg.norm(gotb - wantb) <= TOL * np.linalg.norm(wantb)
    else:
        assert np.array_equal(got, want) and np.array_equal(gotb, wantb)
