"""The sharded path (sharded.py) with the CUDA ops, two ranks sharing the one
GPU of the test box, collectives over gloo (host-staged; the ranks' kernels
never wait on each other).  Checks the CUDA kernels under the sharded row maps
(global D ids, blocked hash row map, rank-order reduction) against the
unsharded oracle: 1e-12 relative, bit-exact on integer inputs."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, G, port, kind, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    try:
        from oracle import sketch
        from paper_2105_11815_b200 import sharded
        from synth import gen
        n, d, m, s, seed = 8192, 64, 112, 1, 9
        A = gen.small_int_dense(seed, n, d) if kind == "int" else np.random.default_rng(seed).standard_normal((n, d))
        b = A[:, 0].copy()
        L = n // G
        At = torch.from_numpy(A[rank * L:(rank + 1) * L].copy()).cuda()
        bt = torch.from_numpy(b[rank * L:(rank + 1) * L].copy()).cuda()
        hr = sharded.ShardedHrht(seed, At, bt, n, m, s, chunk_cols=16)  # 4 column chunks through the pipeline
        strip, sb, lohi = hr.run()
        SA = sharded.gather_strips(strip, lohi, m).cpu().numpy()
        Sb = sharded.gather_strips(sb, lohi, m).cpu().numpy()
        want, wantb = sketch.rht_sketch(seed, A, b, m, s)
        ok = True
        for got, ref in ((SA, want), (Sb, wantb)):
            ok &= np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
            if kind == "int":
                ok &= np.array_equal(got, ref)
        m3 = sharded.ShardedHrhtM3(seed, At, bt, n, m, s)  # exchange-free: skh_fold_lists + one gather
        strip, sb, lohi = m3.run()
        SA = sharded.gather_strips(strip, lohi, m).cpu().numpy()
        Sb = sharded.gather_strips(sb, lohi, m).cpu().numpy()
        for got, ref in ((SA, want), (Sb, wantb)):
            ok &= np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
            if kind == "int":
                ok &= np.array_equal(got, ref)
        # column-major local blocks: skh_fold_cols + skh_rht_colmajor_lists (on-chip fan-out of G s draws)
        m3c = sharded.ShardedHrhtM3Col(seed, At.t().contiguous(), bt, n, m, s)
        sat, dlohi, sb, lohi = m3c.run()
        SA = sharded.gather_strips(sat, dlohi, d).cpu().numpy().T
        Sb = sharded.gather_strips(sb, lohi, m).cpu().numpy()
        for got, ref in ((SA, want), (Sb, wantb)):
            ok &= np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
            if kind == "int":
                ok &= np.array_equal(got, ref)
        pl = sharded.ShardedPlain(seed, At, bt, n, m, 2)
        strip, sb, lohi = pl.run()
        SA = sharded.gather_strips(strip, lohi, m).cpu().numpy()
        want, _ = sketch.sketch_dense(seed, A, b, m, 2)
        ok &= np.linalg.norm(SA - want) / np.linalg.norm(want) <= 1e-12
        if kind == "int":
            ok &= np.array_equal(SA, want)
        # CSR A replicated, bucket strips through the offset view of bucket_ptr (M4)
        from synth import configs
        cfg = configs.C4.scaled(n=5000, d=300, m=97)
        rp, ci, v = gen.csr(cfg)
        bc = np.random.default_rng(3).standard_normal(cfg.n)
        cs = sharded.ShardedCsr(cfg.seed, torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                                torch.from_numpy(v).cuda(), cfg.d, torch.from_numpy(bc).cuda(), cfg.m, cfg.s)
        strip, sb, lohi = cs.run()
        SA = sharded.gather_strips(strip, lohi, cfg.m).cpu().numpy()
        Sb = sharded.gather_strips(sb, lohi, cfg.m).cpu().numpy()
        want, wantb = sketch.sketch_csr(cfg.seed, rp, ci, v, cfg.d, bc, cfg.m, cfg.s)
        ok &= np.array_equal(SA, want) and np.array_equal(Sb, wantb)
        with open(os.path.join(out_dir, f"r{rank}"), "w") as f:
            f.write("ok" if ok else "bad")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["real", "int"])
def test_sharded_cuda_two_ranks(kind, tmp_path):
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2105_11815_b200.build as b
    b.build()
    mp.spawn(_worker, args=(2, _free_port(), kind, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert (tmp_path / f"r{r}").read_text() == "ok"
