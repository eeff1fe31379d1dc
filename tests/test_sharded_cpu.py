"""The multi-GPU sequencing (paper_2105_11815_b200/sharded.py) on CPU with the
gloo backend, world sizes 2 and 4.  The per-rank compute is the oracle (an
ops object defined here, in tests/), so these tests check the index algebra
of the butterfly all-to-all (R7), the row maps handed to hash_gen, and the
deterministic strip reduction (R6) against the unsharded oracle:
  * real inputs: relative Frobenius error <= 1e-12 (BASELINE.json);
  * integer inputs: bit-identical (every partial sum is an exact integer).
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hadamard, hashing, sketch
from synth import configs, gen


class OracleOps:
    """The oracle behind sharded.py's ops interface (CPU tensors)."""

    class BL:
        def __init__(self, m, s, ptr, rows, signs):
            self.m, self.s, self.ptr, self.rows, self.signs = m, s, ptr, rows, signs

    def hash_gen(self, seed, m, s, nrows, row0, blk, stride, out=None):
        k = np.arange(nrows)
        gid = row0 + k if blk <= 0 else row0 + (k // blk) * stride + (k % blk)
        ptr, rows, signs = hashing.bucket_lists(seed, gid, m, s)
        return self.BL(m, s, ptr, rows, signs)

    def rht_stages(self, seed, X, bit_lo, bit_hi, nrows, row0, apply_diag, Y, ws=None):
        Xn = X.numpy()
        Z = np.zeros((nrows, Xn.shape[1]))
        Z[: Xn.shape[0]] = Xn
        if apply_diag:
            Z[: Xn.shape[0]] *= hadamard.diag_signs(seed, np.arange(row0, row0 + Xn.shape[0]))[:, None]
        hadamard.fwht_stages(Z, bit_lo, bit_hi)
        Y.copy_(torch.from_numpy(Z))
        return Y

    def sketch_dense(self, bl, X, b, alpha, SA=None, Sb=None):
        SA.copy_(torch.from_numpy(sketch.bucket_sum(X.numpy(), bl.ptr, bl.rows, bl.signs, alpha)))
        if b is not None:
            Sb.copy_(torch.from_numpy(sketch.bucket_sum(b.numpy(), bl.ptr, bl.rows, bl.signs, alpha)))
        return SA, Sb

    def strip(self, bl, lo, hi):
        # the offset view the CUDA ops hand to skh_sketch_csr: ptr[lo..hi], absolute offsets into rows
        return self.BL(hi - lo, bl.s, np.asarray(bl.ptr)[lo:hi + 1], bl.rows, bl.signs)

    def sketch_csr(self, bl, row_ptr, col_idx, val, d, b, SA=None, Sb=None, ws=None):
        rp, ci, v = row_ptr.numpy(), col_idx.numpy(), val.numpy()
        c = hashing.c_s(bl.s)
        for j in range(len(bl.ptr) - 1):
            acc = np.zeros(d)
            for t in range(int(bl.ptr[j]), int(bl.ptr[j + 1])):
                acc += float(bl.signs[t]) * sketch.csr_row(rp, ci, v, int(bl.rows[t]), d)
            SA[j] = torch.from_numpy(c * acc)
        if b is not None:
            Sb.copy_(torch.from_numpy(sketch.bucket_sum(b.numpy(), np.asarray(bl.ptr) - int(bl.ptr[0]),
                                                        np.asarray(bl.rows)[int(bl.ptr[0]):],
                                                        np.asarray(bl.signs)[int(bl.ptr[0]):], c)))
        return SA, Sb

    def ordered_sum(self, parts, alpha, out=None):
        acc = parts[0].clone()
        for g in range(1, parts.shape[0]):
            acc = acc + parts[g]
        out.copy_(alpha * acc)
        return out

    def fold_lists(self, bl, L, rank):
        j = np.asarray(bl.rows, dtype=np.int64)
        par = np.array([bin(int(g) & rank).count("1") & 1 for g in (j // L)], dtype=np.int64)
        bl.rows = (j % L).astype(bl.rows.dtype)
        bl.signs = np.where(par == 1, -np.asarray(bl.signs), np.asarray(bl.signs)).astype(np.asarray(bl.signs).dtype)
        return bl

    def hash_cols(self, seed, m, s, n, out=None):
        rows, signs = hashing.draw_columns(seed, np.arange(n), m, s)
        bl = self.BL(m, s, None, None, None)
        bl.col_rows, bl.col_signs = rows.reshape(-1), signs.reshape(-1)
        return bl

    def fold_cols(self, bl, L, G, s, rank, out=None):
        # T_r's column lists over local rows: entry (l, g, q) <- global row g L + l, sign x (-1)^popcount(g & r)
        rows = np.asarray(bl.col_rows).reshape(G, L, s)
        signs = np.asarray(bl.col_signs).reshape(G, L, s).astype(np.int64)
        par = np.array([(-1) ** (bin(g & rank).count("1") & 1) for g in range(G)])
        return (rows.transpose(1, 0, 2).reshape(-1),
                (signs * par[:, None, None]).transpose(1, 0, 2).reshape(-1).astype(np.int8))

    def rht_cm_lists_op(self, L, m, s_eff, d, device):
        return (L, m, s_eff, d)

    def rht_cm_lists(self, op, seed, At, b, row0, lists, SAt, Sb):
        # unscaled T_r H_L D A_r from the folded column lists (bucket order: local row, then entry)
        L, m, s_eff, d = op
        lg = L.bit_length() - 1
        D = hadamard.diag_signs(seed, np.arange(row0, row0 + L))
        Z = np.ascontiguousarray(At.numpy().T) * D[:, None]
        hadamard.fwht_stages(Z, 0, lg)
        k = np.asarray(lists[0], dtype=np.int64)
        sg = np.asarray(lists[1])
        local = np.repeat(np.arange(L), s_eff)
        perm = np.argsort(k, kind="stable")
        ptr = np.zeros(m + 1, dtype=np.int64)
        np.cumsum(np.bincount(k, minlength=m), out=ptr[1:])
        SAt.copy_(torch.from_numpy(sketch.bucket_sum(Z, ptr, local[perm], sg[perm], 1.0).T.copy()))
        if b is not None:
            zb = b.numpy() * D
            hadamard.fwht_stages(zb[:, None], 0, lg)
            Sb.copy_(torch.from_numpy(sketch.bucket_sum(zb, ptr, local[perm], sg[perm], 1.0)))
        return SAt, Sb

    def c_ns(self, n_pad, s):
        return sketch.c_ns(n_pad, s)

    def c_s(self, s):
        return hashing.c_s(s)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, G, port, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    try:
        from paper_2105_11815_b200 import sharded
        n, d, m, s, seed, kind = case[:6]
        chunk = case[6] if len(case) > 6 else None
        A = gen.small_int_dense(seed, n, d) if kind == "int" else np.random.default_rng(seed).standard_normal((n, d))
        b = np.random.default_rng(seed + 1).standard_normal(n) if kind != "int" else gen.small_int_dense(seed + 1, n, 1)[:, 0]
        ops = OracleOps()
        L = n // G
        At = torch.from_numpy(A[rank * L:(rank + 1) * L].copy())
        bt = torch.from_numpy(b[rank * L:(rank + 1) * L].copy())
        hr = sharded.ShardedHrht(seed, At, bt, n, m, s, ops=ops, chunk_cols=chunk)
        strip, sb, (lo, hi) = hr.run()
        SA = sharded.gather_strips(strip, (lo, hi), m).numpy()
        Sb = sharded.gather_strips(sb, (lo, hi), m).numpy()
        want, wantb = sketch.rht_sketch(seed, A, b, m, s)
        for got, ref in ((SA, want), (Sb, wantb)):
            assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
            if kind == "int":
                assert np.array_equal(got, ref)
        # the exchange-free variant (M3): H_G folded into the sketch
        m3 = sharded.ShardedHrhtM3(seed, At, bt, n, m, s, ops=ops)
        strip, sb, (lo, hi) = m3.run()
        SA = sharded.gather_strips(strip, (lo, hi), m).numpy()
        Sb = sharded.gather_strips(sb, (lo, hi), m).numpy()
        for got, ref in ((SA, want), (Sb, wantb)):
            assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
            if kind == "int":
                assert np.array_equal(got, ref)
        # the exchange-free variant on column-major local blocks (on-chip fan-out of G s folded draws)
        if G * s <= 8:
            m3c = sharded.ShardedHrhtM3Col(seed, torch.from_numpy(A[rank * L:(rank + 1) * L].T.copy()), bt, n, m, s,
                                           ops=ops)
            sat, dlohi, sb, lohi = m3c.run()
            SA = sharded.gather_strips(sat, dlohi, d).numpy().T
            Sb = sharded.gather_strips(sb, lohi, m).numpy()
            for got, ref in ((SA, want), (Sb, wantb)):
                assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
                if kind == "int":
                    assert np.array_equal(got, ref)
        # plain s-hashing with uneven row blocks
        per = (n + G - 1) // G
        r0, r1 = min(n, rank * per), min(n, (rank + 1) * per)
        pl = sharded.ShardedPlain(seed, torch.from_numpy(A[r0:r1].copy()), torch.from_numpy(b[r0:r1].copy()), n, m,
                                  s, ops=ops)
        strip, sb, (lo, hi) = pl.run()
        SA = sharded.gather_strips(strip, (lo, hi), m).numpy()
        Sb = sharded.gather_strips(sb, (lo, hi), m).numpy()
        want, wantb = sketch.sketch_dense(seed, A, b, m, s)
        for got, ref in ((SA, want), (Sb, wantb)):
            assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
            if kind == "int":
                assert np.array_equal(got, ref)
        # CSR A replicated, bucket strips (M4): every rank's strip through the
        # offset view of bucket_ptr; together they are the oracle's SA, bit for bit
        rp, ci, v = gen.csr(configs.C4.scaled(n=n, d=3 * d + 1, m=m))
        cs = sharded.ShardedCsr(seed, torch.from_numpy(rp), torch.from_numpy(ci), torch.from_numpy(v), 3 * d + 1,
                                torch.from_numpy(b.copy()), m, s, ops=ops)
        strip, sb, (lo, hi) = cs.run()
        SA = sharded.gather_strips(strip, (lo, hi), m).numpy()
        Sb = sharded.gather_strips(sb, (lo, hi), m).numpy()
        want, wantb = sketch.sketch_csr(seed, rp, ci, v, 3 * d + 1, b, m, s)
        assert np.array_equal(SA, want) and np.array_equal(Sb, wantb)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G,case", [(2, (256, 8, 21, 1, 5, "real")), (2, (512, 6, 40, 2, 6, "int")),
                                    (4, (1024, 5, 33, 1, 7, "real")), (4, (256, 4, 17, 3, 8, "int")),
                                    # column-chunk pipeline: 3 chunks (2 + 2 + 1 ragged), both buffers reused
                                    (2, (512, 5, 30, 1, 9, "real", 2)), (4, (256, 7, 19, 2, 10, "int", 3))])
def test_sharded_gloo(G, case):
    mp.spawn(_worker, args=(G, _free_port(), case), nprocs=G, join=True)


def test_strip_rows():
    from paper_2105_11815_b200 import sharded
    mq, st = sharded.strip_rows(7168, 8)
    assert mq == 896 and st[-1] == (6272, 7168)
    mq, st = sharded.strip_rows(10, 4)
    assert mq == 3 and st == [(0, 3), (3, 6), (6, 9), (9, 10)]
    assert math.prod([1]) == 1
