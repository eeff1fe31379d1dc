"""Multi-GPU sequencing of the hot path.

One process per GPU; torch.distributed (NCCL over NVLink/NVSwitch) carries the
two exchange steps the method has when A is row-sharded:

  R7  butterfly exchange (H D A only): H_n = H_G (x) H_{n/G} in the Sylvester
      (natural) order of P:L796, so after the local stages on the low
      log2(n/G) bits of the row index, ONE all-to-all that swaps the rank bits
      with the top log2(G) local bits makes the remaining stages local.
  R6  reduction of the m x d partial sketches: SA = sum_g S_g A_g (linearity of
      Alg. 1 Step 1).  Deterministic (M5): an all-to-all of row strips
      followed by a fixed rank-order sum in our kernel (skh_ordered_sum), so the
      result does not depend on NCCL's reduction order.

The per-rank compute goes through an ``ops`` object.  ``CudaOps`` (the
product) calls libskh; the CPU tests pass an oracle-backed implementation to
check this module's index algebra with the gloo backend.  There is no CPU
fallback in the product path.
"""
import math

import torch
import torch.distributed as dist


class CudaOps:
    """libskh behind the ops interface (device tensors, current stream)."""

    def __init__(self):
        from . import api
        self.api = api

    def hash_gen(self, seed, m, s, nrows, row0, blk, stride, out=None):
        return self.api.hash_gen(seed, m, s, nrows, row0=row0, blk=blk, stride=stride, out=out)

    def rht_stages(self, seed, X, bit_lo, bit_hi, nrows, row0, apply_diag, Y, ws=None):
        return self.api.rht_stages(seed, X, bit_lo, bit_hi, nrows=nrows, row0=row0, apply_diag=apply_diag,
                                   alpha=1.0, Y=Y, ws=ws)

    def sketch_dense(self, bl, X, b, alpha, SA=None, Sb=None):
        return self.api.sketch_dense(bl, X, b, alpha=alpha, SA=SA, Sb=Sb)

    def strip(self, bl, lo, hi):
        """Buckets [lo, hi) of ``bl`` as bucket lists of their own: an offset
        view of bucket_ptr (include/skh.h: ptr[0] need not be 0)."""
        return self.api.BucketLists(hi - lo, bl.s, bl.nrows, bl.ptr[lo:hi + 1], bl.rows, bl.signs)

    def sketch_csr(self, bl, row_ptr, col_idx, val, d, b, SA=None, Sb=None, ws=None):
        return self.api.sketch_csr(bl, row_ptr, col_idx, val, d, b, SA=SA, Sb=Sb, ws=ws)

    def ordered_sum(self, parts, alpha, out=None):
        return self.api.ordered_sum(parts, alpha=alpha, out=out)

    def fold_lists(self, bl, L, rank):
        return self.api.fold_lists(bl, L, rank)

    def hash_cols(self, seed, m, s, n, out=None):
        """Column lists (rows, signs) of all n columns of S, [n][s] (the bucket
        lists are built too and reused through ``out``)."""
        bl = self.api.hash_gen(seed, m, s, n, want_cols=True, out=out)
        return bl

    def fold_cols(self, bl, L, G, s, rank, out=None):
        return self.api.fold_cols(bl.col_rows, bl.col_signs, L, G, s, rank, out=out)

    def rht_cm_lists(self, op, seed, At, b, row0, lists, SAt, Sb):
        """Unscaled S' H_L D A_r for a column-major local block (op: api.RhtColMajorLists)."""
        return op(seed, At, b, row0, lists[0], lists[1], alpha=1.0, SAt=SAt, Sb=Sb)

    def rht_cm_lists_op(self, L, m, s_eff, d, device):
        return self.api.RhtColMajorLists(L, m, s_eff, d, device)

    def c_ns(self, n_pad, s):
        return self.api.c_ns(n_pad, s)

    def c_s(self, s):
        return self.api.c_s(s)


def all_to_all(out, inp, group=None):
    """all_to_all_single with equal splits.  NCCL moves device tensors directly
    (NVLink/NVSwitch); the gloo backend (CPU tests, single-GPU functional runs)
    stages CUDA tensors through host memory."""
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), group=group)
        out.copy_(o)
        return out
    dist.all_to_all_single(out, inp, group=group)
    return out


def all_to_all_async(out, inp, group=None):
    """Asynchronous all_to_all_single (NCCL: the collective runs on NCCL's stream
    after the current stream's prior work; ``handle.wait()`` makes the current
    stream wait for it).  gloo with CUDA tensors stages through host memory and
    is synchronous (returns None)."""
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        all_to_all(out, inp, group=group)
        return None
    return dist.all_to_all_single(out, inp, group=group, async_op=True)


def _log2(x):
    k = int(x).bit_length() - 1
    if (1 << k) != x:
        raise ValueError(f"{x} is not a power of two")
    return k


def strip_rows(m, G):
    """Row strips of the reduce step: rank r owns rows [r*mq, min(m, (r+1)*mq))."""
    mq = (m + G - 1) // G
    return mq, [(r * mq, min(m, (r + 1) * mq)) for r in range(G)]


class ShardedHrht:
    """SA = S_h H D A over G ranks holding contiguous row blocks of A (n = 2^k,
    G = 2^g <= n).  run() returns this rank's strip (rows lo:hi of SA) and of Sb.

    Column-chunk pipeline (SURVEY §8(e) "Overlap: chunk the d axis"): H and S_h
    act on every column independently, so the local transform, the butterfly
    all-to-all (R7), the cross stages and the gather run per chunk of
    ``chunk_cols`` columns, and the all-to-all of chunk k (asynchronous, NCCL's
    stream) overlaps the cross stages + gather of chunk k - 1 and the local
    transform of chunk k + 1 on the compute stream.  Two send and two receive
    buffers of n/G x chunk_cols doubles (contiguous, so every destination's rows
    are one contiguous block); the strip reduction (R6) follows the last chunk."""

    def __init__(self, seed, A_loc, b_loc, n, m, s, ops=None, group=None, chunk_cols=None):
        self.ops = ops or CudaOps()
        self.group = group
        self.G = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.seed, self.n, self.m, self.s = seed, int(n), int(m), int(s)
        self.L = self.n // self.G
        if self.L * self.G != self.n or A_loc.shape[0] != self.L:
            raise ValueError("A_loc must hold n / G rows")
        _log2(self.n)
        self.lg = _log2(self.L)
        self.lq = _log2(self.L // self.G) if self.L >= self.G else None
        if self.lq is None:
            raise ValueError("need n / G >= G")
        self.A, self.b = A_loc, b_loc
        d = A_loc.shape[1]
        self.d = d
        self.W = int(chunk_cols) if chunk_cols else (d if d <= 512 else 512)
        self.K = (d + self.W - 1) // self.W
        kw = dict(dtype=A_loc.dtype, device=A_loc.device)
        nb = min(2, self.K)
        self.send = [torch.empty(self.L * self.W, **kw) for _ in range(nb)]
        self.recv = [torch.empty(self.L * self.W, **kw) for _ in range(nb)]
        self.yb = torch.empty(self.L, 1, **kw) if b_loc is not None else None
        self.yb2 = torch.empty(self.L, 1, **kw) if b_loc is not None else None
        self.mq, self.strips = strip_rows(self.m, self.G)
        self.P = torch.zeros(self.G * self.mq, d, **kw)      # partial, padded to G strips
        self.Pb = torch.zeros(self.G * self.mq, **kw) if b_loc is not None else None
        self.R = torch.empty(self.G, self.mq, d, **kw)       # received strips
        self.Rb = torch.empty(self.G, self.mq, **kw) if b_loc is not None else None
        self.out = torch.empty(self.mq, d, **kw)
        self.outb = torch.empty(self.mq, 1, **kw) if b_loc is not None else None
        self.bl = None
        self.alpha = self.ops.c_ns(self.n, self.s)
        self.ws = None
        if isinstance(self.ops, CudaOps):
            self.ws = self.ops.api.rht_stages_workspace(self.L, self.L, self.r * self.L, max(self.W, 1),
                                                        A_loc.device)

    STAGES = ("hash_gen", "rhs", "pipeline", "reduce")

    def _chunk(self, k):
        c0 = k * self.W
        w = min(self.d, c0 + self.W) - c0
        return c0, w

    def run(self, mark=None):
        """One sharded step; ``mark(name)`` (optional) is called after each of
        STAGES (bench.py records a CUDA event there)."""
        mark = mark or (lambda name: None)
        ops, G, r, L = self.ops, self.G, self.r, self.L
        blk = L // G
        # R1 + R2 for exactly the global rows this rank holds after the exchange:
        # received row k = g*blk + t is global row g*L + r*blk + t (ascending in k)
        self.bl = ops.hash_gen(self.seed, self.m, self.s, L, r * blk, blk, L, out=self.bl)
        mark("hash_gen")
        if self.b is not None:  # the right-hand side: one column, unpipelined
            ops.rht_stages(self.seed, self.b.view(-1, 1), 0, self.lg, L, r * L, True, self.yb, self.ws)
            if G > 1:
                all_to_all(self.yb2, self.yb, group=self.group)
            else:
                self.yb2.copy_(self.yb)
            if self.lq < self.lg:
                ops.rht_stages(self.seed, self.yb2, self.lq, self.lg, L, 0, False, self.yb2, self.ws)
            ops.sketch_dense(self.bl, self.yb2, None, 1.0, SA=self.Pb[: self.m].view(-1, 1))
        mark("rhs")
        handles = [None] * self.K

        def finish(j):
            c0, w = self._chunk(j)
            if handles[j] is not None:
                handles[j].wait()
            Y2 = self.recv[j % len(self.recv)][: L * w].view(L, w)
            # the rank bits g are local bits [log2 blk, log2 L): the remaining
            # global stages, low to high
            if self.lq < self.lg:
                ops.rht_stages(self.seed, Y2, self.lq, self.lg, L, 0, False, Y2, self.ws)
            # R5: unscaled partial sums of this rank's rows, columns c0 .. c0 + w
            ops.sketch_dense(self.bl, Y2, None, 1.0, SA=self.P[: self.m, c0:c0 + w])

        for k in range(self.K):
            c0, w = self._chunk(k)
            Y = self.send[k % len(self.send)][: L * w].view(L, w)
            # R3 + R4 (local): global bits [0, log2 L) = local bits, D with global ids
            ops.rht_stages(self.seed, self.A[:, c0:c0 + w], 0, self.lg, L, r * L, True, Y, self.ws)
            # R7: block q of rows [q*blk, (q+1)*blk) -> rank q (equal splits)
            Y2 = self.recv[k % len(self.recv)][: L * w].view(L, w)
            if G > 1:
                handles[k] = all_to_all_async(Y2, Y, group=self.group)
            else:
                Y2.copy_(Y)
            if k >= 1:
                finish(k - 1)
        finish(self.K - 1)
        mark("pipeline")
        # R6 (M5): strips to their owners, then a rank-order sum scaled once by c_ns
        lo, hi = self.strips[r]
        if G > 1:
            all_to_all(self.R.view(G * self.mq, self.d), self.P, group=self.group)
            if self.b is not None:
                all_to_all(self.Rb.view(-1), self.Pb, group=self.group)
        else:
            self.R[0].copy_(self.P)
            if self.b is not None:
                self.Rb[0].copy_(self.Pb)
        ops.ordered_sum(self.R, self.alpha, out=self.out)
        Sb = None
        if self.b is not None:
            ops.ordered_sum(self.Rb.view(G, self.mq, 1), self.alpha, out=self.outb)
            Sb = self.outb[: hi - lo, 0]
        mark("reduce")
        return self.out[: hi - lo], Sb, (lo, hi)


class ShardedHrhtM3:
    """SA = S_h H D A over G ranks WITHOUT the butterfly all-to-all (SURVEY §8(e)
    M3): H_n = H_G (x) H_L (L = n / G), so with Z_r = H_L D A_r (the local rows,
    every local stage, D with global ids)

        S H D A = sum_r T_r Z_r,   T_r = sum_g (-1)^popcount(g & r) S_g,

    S_g the columns g L .. g L + L - 1 of S.  Each rank draws S for all n
    columns (cheap: n s entries), folds the lists into T_r's (skh_fold_lists:
    row j -> j mod L, sign times (-1)^popcount((j / L) & r)), gathers its local
    Z_r with them (every local row is read by G s list entries) and the partials
    meet in the same deterministic strip reduction as ShardedHrht (R6).  The only
    collective is that reduction: |SA| per rank instead of the (G-1)/G |A_r|
    all-to-all.  Rounding differs from the single-GPU order (the H_G butterflies
    are folded into the sums): 1e-12, bit-identical on integer inputs."""

    STAGES = ("hash_gen", "transform", "gather", "reduce")

    def __init__(self, seed, A_loc, b_loc, n, m, s, ops=None, group=None):
        self.ops = ops or CudaOps()
        self.group = group
        self.G = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.seed, self.n, self.m, self.s = seed, int(n), int(m), int(s)
        self.L = self.n // self.G
        if self.L * self.G != self.n or A_loc.shape[0] != self.L:
            raise ValueError("A_loc must hold n / G rows")
        _log2(self.n)
        self.lg = _log2(self.L)
        if self.n * self.s >= 2 ** 31:
            # every rank draws and sorts the lists of all n columns (int32 entries)
            raise ValueError(f"exchange-free H D needs n * s < 2^31 (n = {self.n}, s = {self.s}): "
                             "use ShardedHrht (its ranks hash only their n / G rows)")
        self.A, self.b = A_loc, b_loc
        d = A_loc.shape[1]
        self.d = d
        kw = dict(dtype=A_loc.dtype, device=A_loc.device)
        self.Z = torch.empty(self.L, d, **kw)
        self.zb = torch.empty(self.L, 1, **kw) if b_loc is not None else None
        self.mq, self.strips = strip_rows(self.m, self.G)
        self.P = torch.zeros(self.G * self.mq, d, **kw)
        self.Pb = torch.zeros(self.G * self.mq, **kw) if b_loc is not None else None
        self.R = torch.empty(self.G, self.mq, d, **kw)
        self.Rb = torch.empty(self.G, self.mq, **kw) if b_loc is not None else None
        self.out = torch.empty(self.mq, d, **kw)
        self.outb = torch.empty(self.mq, 1, **kw) if b_loc is not None else None
        self.bl = None
        self.alpha = self.ops.c_ns(self.n, self.s)
        self.ws = None
        if isinstance(self.ops, CudaOps):
            self.ws = self.ops.api.rht_stages_workspace(self.L, self.L, self.r * self.L, d, A_loc.device)

    def run(self, mark=None):
        mark = mark or (lambda name: None)
        ops, G, r, L = self.ops, self.G, self.r, self.L
        # S for all n columns (global row ids), folded into T_r over local rows
        self.bl = ops.hash_gen(self.seed, self.m, self.s, self.n, 0, 0, 0, out=self.bl)
        ops.fold_lists(self.bl, L, r)
        mark("hash_gen")
        ops.rht_stages(self.seed, self.A, 0, self.lg, L, r * L, True, self.Z, self.ws)
        if self.b is not None:
            ops.rht_stages(self.seed, self.b.view(-1, 1), 0, self.lg, L, r * L, True, self.zb, self.ws)
        mark("transform")
        ops.sketch_dense(self.bl, self.Z, None if self.b is None else self.zb.view(-1), 1.0, SA=self.P[: self.m],
                         Sb=None if self.b is None else self.Pb[: self.m])
        mark("gather")
        lo, hi = self.strips[r]
        if G > 1:
            all_to_all(self.R.view(G * self.mq, self.d), self.P, group=self.group)
            if self.b is not None:
                all_to_all(self.Rb.view(-1), self.Pb, group=self.group)
        else:
            self.R[0].copy_(self.P)
            if self.b is not None:
                self.Rb[0].copy_(self.Pb)
        ops.ordered_sum(self.R, self.alpha, out=self.out)
        Sb = None
        if self.b is not None:
            ops.ordered_sum(self.Rb.view(G, self.mq, 1), self.alpha, out=self.outb)
            Sb = self.outb[: hi - lo, 0]
        mark("reduce")
        return self.out[: hi - lo], Sb, (lo, hi)


class ShardedHrhtM3Col:
    """The exchange-free M3 of ShardedHrhtM3 for a COLUMN-MAJOR local block At
    (d, L) -- the paper's storage -- with the survey's on-chip fan-out
    (SURVEY §8(e) M3): each rank folds the column lists of all n columns of S
    into T_r's (skh_fold_cols: G s entries per local row), then ONE call
    (skh_rht_colmajor_lists) runs pass 1 of H_L D A_r (D over global ids) and
    the fused pass 2, whose owner-planned gather adds every local row, read once
    from HBM, into its G s folded buckets from shared memory.  The unscaled
    partials SA_r^T (d, m) meet in the deterministic rank-order reduction over
    column strips of SA (rank r gets SA[:, dlo:dhi] as SA^T rows, contiguous
    blocks for the all-to-all); Sb over bucket strips as in ShardedHrht.
    Needs G s <= 8 (the fused gather's draws per row).  1e-12 against the
    unsharded oracle, bit-identical on integer inputs.

    run() -> (SAt_strip (dhi - dlo, m), (dlo, dhi), Sb_strip, (lo, hi))."""

    STAGES = ("hash_gen", "sketch", "reduce")

    def __init__(self, seed, At_loc, b_loc, n, m, s, ops=None, group=None):
        self.ops = ops or CudaOps()
        self.group = group
        self.G = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.seed, self.n, self.m, self.s = seed, int(n), int(m), int(s)
        self.L = self.n // self.G
        d, L = At_loc.shape
        if self.L * self.G != self.n or L != self.L:
            raise ValueError("At_loc must be (d, n / G)")
        _log2(self.n)
        if self.G * self.s > 8:
            raise ValueError(f"column-major M3 folds G s = {self.G * self.s} draws per local row; the fused "
                             "gather takes at most 8 (use ShardedHrht)")
        if self.n * self.s >= 2 ** 31:
            raise ValueError(f"exchange-free H D needs n * s < 2^31 (n = {self.n}, s = {self.s})")
        self.At, self.b, self.d = At_loc, b_loc, d
        kw = dict(dtype=At_loc.dtype, device=At_loc.device)
        self.dq, self.dstrips = strip_rows(d, self.G)
        self.mq, self.strips = strip_rows(self.m, self.G)
        self.P = torch.zeros(self.G * self.dq, self.m, **kw)   # partial SA^T, column strips of SA
        self.Pb = torch.zeros(self.G * self.mq, **kw) if b_loc is not None else None
        self.R = torch.empty(self.G, self.dq, self.m, **kw)
        self.Rb = torch.empty(self.G, self.mq, **kw) if b_loc is not None else None
        self.out = torch.empty(self.dq, self.m, **kw)
        self.outb = torch.empty(self.mq, 1, **kw) if b_loc is not None else None
        self.alpha = self.ops.c_ns(self.n, self.s)
        self.bl = None
        self.lists = None
        self.op = self.ops.rht_cm_lists_op(self.L, self.m, self.G * self.s, d, At_loc.device)

    def run(self, mark=None):
        mark = mark or (lambda name: None)
        ops, G, r, L = self.ops, self.G, self.r, self.L
        self.bl = ops.hash_cols(self.seed, self.m, self.s, self.n, out=self.bl)
        self.lists = ops.fold_cols(self.bl, L, G, self.s, r, out=self.lists)
        mark("hash_gen")
        ops.rht_cm_lists(self.op, self.seed, self.At, self.b, r * L, self.lists, self.P[: self.d],
                         None if self.b is None else self.Pb[: self.m])
        mark("sketch")
        dlo, dhi = self.dstrips[r]
        lo, hi = self.strips[r]
        if G > 1:
            all_to_all(self.R.view(G * self.dq, self.m), self.P, group=self.group)
            if self.b is not None:
                all_to_all(self.Rb.view(-1), self.Pb, group=self.group)
        else:
            self.R[0].copy_(self.P)
            if self.b is not None:
                self.Rb[0].copy_(self.Pb)
        ops.ordered_sum(self.R, self.alpha, out=self.out)
        Sb = None
        if self.b is not None:
            ops.ordered_sum(self.Rb.view(G, self.mq, 1), self.alpha, out=self.outb)
            Sb = self.outb[: hi - lo, 0]
        mark("reduce")
        return self.out[: dhi - dlo], (dlo, dhi), Sb, (lo, hi)


class ShardedPlain:
    """SA = S A (s-hashing, no transform) over G ranks with contiguous row blocks."""

    def __init__(self, seed, A_loc, b_loc, n, m, s, ops=None, group=None):
        self.ops = ops or CudaOps()
        self.group = group
        self.G = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.seed, self.n, self.m, self.s = seed, int(n), int(m), int(s)
        per = (self.n + self.G - 1) // self.G
        self.row0 = min(self.n, self.r * per)
        self.nloc = min(self.n, self.row0 + per) - self.row0
        if A_loc.shape[0] != self.nloc:
            raise ValueError(f"rank {self.r} must hold rows [{self.row0}, {self.row0 + self.nloc})")
        self.A, self.b = A_loc, b_loc
        d = A_loc.shape[1]
        self.d = d
        kw = dict(dtype=A_loc.dtype, device=A_loc.device)
        self.mq, self.strips = strip_rows(self.m, self.G)
        self.P = torch.zeros(self.G * self.mq, d, **kw)
        self.Pb = torch.zeros(self.G * self.mq, **kw) if b_loc is not None else None
        self.R = torch.empty(self.G, self.mq, d, **kw)
        self.Rb = torch.empty(self.G, self.mq, **kw) if b_loc is not None else None
        self.out = torch.empty(self.mq, d, **kw)
        self.outb = torch.empty(self.mq, 1, **kw) if b_loc is not None else None
        self.bl = None
        self.alpha = self.ops.c_s(self.s)

    STAGES = ("hash_gen", "gather", "reduce")

    def run(self, mark=None):
        mark = mark or (lambda name: None)
        ops, G, r = self.ops, self.G, self.r
        self.bl = ops.hash_gen(self.seed, self.m, self.s, self.nloc, self.row0, 0, 0, out=self.bl)
        mark("hash_gen")
        ops.sketch_dense(self.bl, self.A, self.b, 1.0, SA=self.P[: self.m],
                         Sb=None if self.b is None else self.Pb[: self.m])
        mark("gather")
        lo, hi = self.strips[r]
        if G > 1:
            all_to_all(self.R.view(G * self.mq, self.d), self.P, group=self.group)
            if self.b is not None:
                all_to_all(self.Rb.view(-1), self.Pb, group=self.group)
        else:
            self.R[0].copy_(self.P)
            if self.b is not None:
                self.Rb[0].copy_(self.Pb)
        ops.ordered_sum(self.R, self.alpha, out=self.out)
        Sb = None
        if self.b is not None:
            ops.ordered_sum(self.Rb.view(G, self.mq, 1), self.alpha, out=self.outb)
            Sb = self.outb[: hi - lo, 0]
        mark("reduce")
        return self.out[: hi - lo], Sb, (lo, hi)


class ShardedCsr:
    """CSR A replicated on every rank (|SA| >> |A| for C4): rank r computes the
    SA rows of its bucket strip, no collective; the strips
    together are SA.  The strip is handed to skh_sketch_csr as an offset view of
    the full bucket_ptr, so every rank hashes all n rows once and reads only its
    buckets' rows of A."""

    def __init__(self, seed, row_ptr, col_idx, val, d, b, m, s, ops=None, group=None):
        self.ops = ops or CudaOps()
        self.G = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.seed, self.m, self.s, self.d = seed, int(m), int(s), int(d)
        self.csr = (row_ptr, col_idx, val)
        self.b = b
        self.mq, self.strips = strip_rows(self.m, self.G)
        lo, hi = self.strips[self.r]
        dev = row_ptr.device
        self.SA = torch.empty(max(hi - lo, 1), self.d, dtype=torch.float64, device=dev)
        self.Sb = torch.empty(max(hi - lo, 1), dtype=torch.float64, device=dev) if b is not None else None
        self.bl = None
        self.ws = None
        if row_ptr.is_cuda:
            from . import api
            self.ws = api.sketch_csr_workspace(row_ptr.numel() - 1, self.s, val.numel(), dev)

    STAGES = ("hash_gen", "gather_csr")

    def run(self, mark=None):
        mark = mark or (lambda name: None)
        ops = self.ops
        n = self.csr[0].numel() - 1
        self.bl = ops.hash_gen(self.seed, self.m, self.s, n, 0, 0, 0, out=self.bl)
        mark("hash_gen")
        lo, hi = self.strips[self.r]
        if hi > lo:
            ops.sketch_csr(ops.strip(self.bl, lo, hi), *self.csr, self.d, self.b, SA=self.SA[: hi - lo],
                           Sb=None if self.b is None else self.Sb[: hi - lo], ws=self.ws)
        mark("gather_csr")
        return self.SA[: hi - lo], None if self.b is None else self.Sb[: hi - lo], (lo, hi)


def gather_strips(strip, lohi, m, group=None):
    """Collect every rank's strip on all ranks (test / user convenience)."""
    G = dist.get_world_size(group)
    mq = math.ceil(m / G)
    buf = torch.zeros(mq, *strip.shape[1:], dtype=strip.dtype, device=strip.device)
    buf[: strip.shape[0]] = strip
    if buf.is_cuda and dist.get_backend(group) == "gloo":
        buf = buf.cpu()
    allb = [torch.empty_like(buf) for _ in range(G)]
    dist.all_gather(allb, buf, group=group)
    return torch.cat(allb, 0)[:m].to(strip.device)
