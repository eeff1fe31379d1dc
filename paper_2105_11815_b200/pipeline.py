"""One step of the hot path (all SURVEY §8(a) rows) with preallocated buffers,
composed from the C-ABI calls so each kernel can be timed live with CUDA
events on the launching stream.  bench.py times these steps and the full-size
parity tests run the same launch configuration.

  HrhtStep  : R1+R2 hash_gen, R3+R4 rht_stages (one call per HBM pass, D fused
              into the first), R5 sketch_dense with alpha = c_ns (C2, C3HD, C5)
  PlainStep : R1+R2, R5 sketch_dense with alpha = c_s (C1, C3)
  CsrStep   : R1+R2, R5 sketch_csr (C4)
  ColStep   : column-major A (the paper's LAPACK layout): one composite call
              (skh_rht_dense_colmajor / skh_sketch_dense_colmajor); its stages
              are timed by the library's stage trace (skh_trace_set)
"""
import torch

from . import api


def _ev():
    return torch.cuda.Event(enable_timing=True)


class _Timed:
    """Records an event after each named stage (stage timing inside the timed
    region).  ``side`` names stages that run on a second stream, overlapped with
    the main-stream stages: they are timed by events on that stream and reported
    with an ``(overlapped)`` suffix, outside the main-stream sum."""

    def __init__(self, names, record, side=()):
        self.names = list(names)
        self.side = list(side)
        self.record = record
        self.events = [_ev() for _ in range(len(self.names) + 1)] if record else None
        self.side_events = [_ev() for _ in range(len(self.side) + 1)] if (record and self.side) else None
        self.i = 0
        self.j = 0

    def side_start(self, stream):
        if self.side_events:
            self.side_events[0].record(stream)
        self.j = 0

    def side_mark(self, stream):
        self.j += 1
        if self.side_events:
            self.side_events[self.j].record(stream)

    def start(self):
        if self.record:
            self.events[0].record()
        self.i = 0

    def mark(self):
        self.i += 1
        if self.record:
            self.events[self.i].record()

    def durations_ms(self):
        """Per-stage durations (call after synchronize)."""
        out = {n: self.events[k].elapsed_time(self.events[k + 1]) for k, n in enumerate(self.names)}
        if self.side_events:
            for k, n in enumerate(self.side):
                out[n + " (overlapped)"] = self.side_events[k].elapsed_time(self.side_events[k + 1])
        return out


class HrhtStep:
    """SA = S_h H D A, Sb = S_h H D b for a row-major A resident on the device
    (variant=True: S_h is the s-hashing variant of Def. 7)."""

    def __init__(self, seed, A, b, m, s, record=False, variant=False):
        self.seed, self.m, self.s = seed, int(m), int(s)
        self.variant = bool(variant)
        self.A, self.b = A, b
        n, d = A.shape
        self.n, self.d = n, d
        n_pad = 1
        while n_pad < n:
            n_pad *= 2
        self.n_pad = n_pad
        self.L = n_pad.bit_length() - 1
        aligned = A.data_ptr() % 16 == 0 and A.stride(0) % 2 == 0
        self.plan = api.rht_pass_plan(self.L, d, aligned)
        dev = A.device
        self.Y = torch.empty(n_pad, d, dtype=torch.float64, device=dev)
        self.yb = torch.empty(n_pad, 1, dtype=torch.float64, device=dev) if b is not None else None
        self.SA = torch.empty(self.m, d, dtype=torch.float64, device=dev)
        self.Sb = torch.empty(self.m, dtype=torch.float64, device=dev) if b is not None else None
        self.bl = None
        self.ws = api.rht_stages_workspace(n_pad, n, 0, d, dev)
        self.alpha = api.c_ns(n_pad, s)
        # the hash and H D b on a side stream beside A's passes (SKH_PIPE_SIDE=0:
        # all on one stream); measured C2 0.511 -> 0.498 ms, C3HD 3.817 -> 3.805 ms
        import os
        self.side = torch.cuda.Stream(device=dev) if os.environ.get("SKH_PIPE_SIDE", "1") != "0" else None
        self.ws_b = api.rht_stages_workspace(n_pad, n, 0, 1, dev) if (self.side is not None and b is not None) else None
        # side-stream mode: the main stream's first stage is only the fork; the
        # hash (and H D b) are timed on the side stream and reported as overlapped
        names = ["fork" if self.side is not None else "hash_gen"] + [f"fwht_pass{p}" for p in range(len(self.plan))]
        if b is not None and self.side is None:
            names.append("fwht_b")
        names.append("gather")
        side = (["hash_gen"] + (["fwht_b"] if b is not None else [])) if self.side is not None else []
        self.timer = _Timed(names, record, side)

    def new_timer(self):
        return _Timed(self.timer.names, True, self.timer.side)

    def run(self, timer=None):
        t = timer or self.timer
        t.start()
        if self.side is not None:
            return self._run_side(t)
        self.bl = api.hash_gen(self.seed, self.m, self.s, self.n_pad, out=self.bl, variant=self.variant)
        t.mark()
        lo = 0
        for p, k in enumerate(self.plan):
            src = self.A if p == 0 else self.Y
            api.rht_stages(self.seed, src, lo, lo + k, nrows=self.n_pad, apply_diag=(p == 0), alpha=1.0, Y=self.Y,
                           ws=self.ws)
            lo += k
            t.mark()
        if self.b is not None:
            api.rht_stages(self.seed, self.b.view(-1, 1), 0, self.L, nrows=self.n_pad, apply_diag=True, alpha=1.0,
                           Y=self.yb, ws=self.ws)
            t.mark()
        api.sketch_dense(self.bl, self.Y, None if self.b is None else self.yb.view(-1), alpha=self.alpha, SA=self.SA,
                         Sb=self.Sb)
        t.mark()
        return self.SA, self.Sb

    def _run_side(self, t):
        main = torch.cuda.current_stream()
        self.side.wait_stream(main)
        with torch.cuda.stream(self.side):
            t.side_start(self.side)
            self.bl = api.hash_gen(self.seed, self.m, self.s, self.n_pad, out=self.bl, variant=self.variant)
            t.side_mark(self.side)
            if self.b is not None:
                api.rht_stages(self.seed, self.b.view(-1, 1), 0, self.L, nrows=self.n_pad, apply_diag=True,
                               alpha=1.0, Y=self.yb, ws=self.ws_b)
                t.side_mark(self.side)
        t.mark()
        lo = 0
        for p, k in enumerate(self.plan):
            src = self.A if p == 0 else self.Y
            api.rht_stages(self.seed, src, lo, lo + k, nrows=self.n_pad, apply_diag=(p == 0), alpha=1.0, Y=self.Y,
                           ws=self.ws)
            lo += k
            t.mark()
        main.wait_stream(self.side)
        api.sketch_dense(self.bl, self.Y, None if self.b is None else self.yb.view(-1), alpha=self.alpha, SA=self.SA,
                         Sb=self.Sb)
        t.mark()
        return self.SA, self.Sb


class PlainStep:
    """SA = S A, Sb = S b (s-hashing, no transform; variant=True: Def. 7)."""

    def __init__(self, seed, A, b, m, s, record=False, variant=False):
        self.seed, self.m, self.s = seed, int(m), int(s)
        self.variant = bool(variant)
        self.A, self.b = A, b
        n, d = A.shape
        dev = A.device
        self.SA = torch.empty(self.m, d, dtype=torch.float64, device=dev)
        self.Sb = torch.empty(self.m, dtype=torch.float64, device=dev) if b is not None else None
        self.bl = None
        self.timer = _Timed(["hash_gen", "gather"], record)

    def new_timer(self):
        return _Timed(self.timer.names, True)

    def run(self, timer=None):
        t = timer or self.timer
        t.start()
        self.bl = api.hash_gen(self.seed, self.m, self.s, self.A.shape[0], out=self.bl, variant=self.variant)
        t.mark()
        api.sketch_dense(self.bl, self.A, self.b, SA=self.SA, Sb=self.Sb)
        t.mark()
        return self.SA, self.Sb


class CsrStep:
    """Dense SA = S A, Sb = S b for CSR A (variant=True: Def. 7)."""

    def __init__(self, seed, row_ptr, col_idx, val, d, b, m, s, record=False, variant=False):
        self.seed, self.m, self.s, self.d = seed, int(m), int(s), int(d)
        self.variant = bool(variant)
        self.csr = (row_ptr, col_idx, val)
        self.b = b
        dev = row_ptr.device
        self.SA = torch.empty(self.m, self.d, dtype=torch.float64, device=dev)
        self.Sb = torch.empty(self.m, dtype=torch.float64, device=dev) if b is not None else None
        self.bl = None
        self.ws = api.sketch_csr_workspace(row_ptr.numel() - 1, s, val.numel(), dev)
        self.timer = _Timed(["hash_gen", "gather_csr"], record)

    def new_timer(self):
        return _Timed(self.timer.names, True)

    def run(self, timer=None):
        t = timer or self.timer
        t.start()
        n = self.csr[0].numel() - 1
        self.bl = api.hash_gen(self.seed, self.m, self.s, n, out=self.bl, variant=self.variant)
        t.mark()
        api.sketch_csr(self.bl, *self.csr, self.d, self.b, SA=self.SA, Sb=self.Sb, ws=self.ws)
        t.mark()
        return self.SA, self.Sb


class ColStep:
    """SA = S_h H D A (hd) or S A for a column-major A given as At (d, n)."""

    def __init__(self, seed, At, b, m, s, hd, record=False):
        self.seed, self.m, self.s, self.hd = seed, int(m), int(s), bool(hd)
        self.At, self.b = At, b
        d, n = At.shape
        self.n, self.d = n, d
        n_pad = 1
        while n_pad < n:
            n_pad *= 2
        self.n_pad = n_pad
        dev = At.device
        self.SAt = torch.empty(d, self.m, dtype=torch.float64, device=dev)
        self.Sb = torch.empty(self.m, dtype=torch.float64, device=dev) if b is not None else None
        if self.hd:
            self.op = api.RhtDenseColMajor(n, m, s, d, dev)
        else:
            lib = api._lib.load()
            self.ws = api._workspace(lib.skh_sketch_dense_colmajor_fast_workspace_bytes(n, m, s, d), dev)
        self.record = record

    def new_timer(self):
        return api.Trace(16)

    def run(self, timer=None):
        if timer is None:
            return self._call()
        with timer:
            return self._call()

    def _call(self):
        if self.hd:
            return self.op(self.seed, self.At, self.b, SAt=self.SAt, Sb=self.Sb)
        return api.sketch_dense_colmajor(self.seed, self.At, self.b, self.m, self.s, SAt=self.SAt, Sb=self.Sb,
                                         ws=self.ws)


class DhtStep:
    """HR-DHT S_h F D (eq. (6.1)) or SR-DHT S_s F D (eq. (7.2)), row-major A: one
    composite call, stages from the library's trace."""

    def __init__(self, seed, A, b, m, s, sampling=False, record=False):
        self.seed, self.m, self.s, self.sampling = seed, int(m), int(s), bool(sampling)
        self.A, self.b = A, b
        n, d = A.shape
        dev = A.device
        lib = api._lib.load()
        nb = (lib.skh_srdht_dense_workspace_bytes(n, self.m, d) if sampling
              else lib.skh_hrdht_dense_workspace_bytes(n, self.m, self.s, d))
        self.ws = api._workspace(nb, dev)
        self.SA = torch.empty(self.m, d, dtype=torch.float64, device=dev)
        self.Sb = torch.empty(self.m, dtype=torch.float64, device=dev) if b is not None else None

    def new_timer(self):
        return api.Trace(16)

    def run(self, timer=None):
        if timer is None:
            return self._call()
        with timer:
            return self._call()

    def _call(self):
        if self.sampling:
            return api.srdht_dense(self.seed, self.A, self.b, self.m, SA=self.SA, Sb=self.Sb, ws=self.ws)
        return api.hrdht_dense(self.seed, self.A, self.b, self.m, self.s, SA=self.SA, Sb=self.Sb, ws=self.ws)
