"""Python binding of libskh (same names as the C ABI in include/skh.h, minus
the ``skh_`` prefix).  Argument marshalling only: every step of the path runs
in the CUDA kernels behind the C ABI; torch supplies device memory and the
current stream.  Raises on a missing library or non-CUDA tensors.

Citations (PAPER.md lines): Alg. 1 Step 1 L871; s-hashing L269-272; HRHT
L790-801.
"""
import math
from dataclasses import dataclass

import torch

from . import _lib


def _stream():
    return ctypes_ptr(torch.cuda.current_stream().cuda_stream)


def ctypes_ptr(x):
    return None if x is None else int(x)


def _ptr(t):
    return None if t is None else t.data_ptr()


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libskh takes CUDA tensors (no CPU fallback)")


def _ld(t):
    # a size-1 dimension's stride is arbitrary in torch/numpy: ignore it
    if t.dim() != 2 or (t.stride(1) != 1 and t.size(1) > 1):
        raise ValueError("expected a row-major 2-D tensor with unit column stride")
    return t.stride(0) if t.size(0) > 1 else max(t.size(1), 1)


def _check_out(t, shape, name):
    """A caller-given output buffer: a CUDA float64 tensor of the output's shape
    (1-D outputs: the right number of elements), since the C ABI only sees a
    pointer and a leading dimension."""
    if not t.is_cuda or t.dtype != torch.float64:
        raise ValueError(f"{name} must be a CUDA float64 tensor")
    ok = t.numel() == shape[0] if len(shape) == 1 else tuple(t.shape) == tuple(shape)
    if not ok:
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def _workspace(nbytes, device):
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def c_s(s):
    return _lib.load().skh_c_s(int(s))


def c_n(n_pad):
    return _lib.load().skh_c_n(int(n_pad))


def c_ns(n_pad, s):
    return _lib.load().skh_c_ns(int(n_pad), int(s))


@dataclass
class BucketLists:
    """CSR form of S_h over this caller's columns (include/skh.h, skh_hash_gen)."""
    m: int
    s: int
    nrows: int
    ptr: torch.Tensor      # int32 [m+1]
    rows: torch.Tensor     # int32 [nrows*s], local column ids
    signs: torch.Tensor    # int8  [nrows*s]
    col_rows: torch.Tensor = None
    col_signs: torch.Tensor = None
    ws: torch.Tensor = None


def hash_gen(seed, m, s, nrows, row0=0, blk=0, stride=0, want_cols=False, device=None, out=None, variant=False):
    """R1+R2: draw the s-hashing columns j(k) and build bucket lists
    (variant=True: the s-hashing variant of Def. 7, draws with replacement)."""
    lib = _lib.load()
    device = device or torch.device("cuda", torch.cuda.current_device())
    N = int(nrows) * int(s)
    if out is None:
        out = BucketLists(m, s, nrows,
                          torch.empty(m + 1, dtype=torch.int32, device=device),
                          torch.empty(max(N, 1), dtype=torch.int32, device=device),
                          torch.empty(max(N, 1), dtype=torch.int8, device=device))
        if want_cols:
            out.col_rows = torch.empty(max(N, 1), dtype=torch.int32, device=device)
            out.col_signs = torch.empty(max(N, 1), dtype=torch.int8, device=device)
        out.ws = _workspace(lib.skh_hash_workspace_bytes(nrows, m, s), device)
    elif (out.ptr.numel() < m + 1 or out.rows.numel() < N or out.signs.numel() < N
          or (out.col_rows is not None and out.col_rows.numel() < N)
          or (out.col_signs is not None and out.col_signs.numel() < N)):
        raise ValueError(f"hash_gen: out holds lists for m={out.m}, s={out.s}, nrows={out.nrows}; "
                         f"asked for m={m}, s={s}, nrows={nrows}")
    else:
        out.m, out.s, out.nrows = int(m), int(s), int(nrows)
    fn = lib.skh_hash_gen_variant if variant else lib.skh_hash_gen
    rc = fn(int(seed) & (2**64 - 1), int(m), int(s), int(nrows), int(row0), int(blk), int(stride),
            _ptr(out.col_rows), _ptr(out.col_signs), _ptr(out.ptr), _ptr(out.rows), _ptr(out.signs),
            _ptr(out.ws), out.ws.numel(), _stream())
    _lib.check(rc, "skh_hash_gen_variant" if variant else "skh_hash_gen")
    return out


def hash_status(bl):
    lib = _lib.load()
    return lib.skh_hash_status(_ptr(bl.ws), _stream())


def sketch_dense(bl, A, b=None, alpha=None, SA=None, Sb=None):
    """R5 dense: SA = alpha * S A (alpha defaults to c_s), Sb likewise."""
    lib = _lib.load()
    _need_cuda(A, b)
    if A.dtype != torch.float64:
        raise ValueError("A must be float64")
    n, d = A.shape
    if SA is None:
        SA = torch.empty(bl.m, d, dtype=torch.float64, device=A.device)
    else:
        _check_out(SA, (bl.m, d), "SA")
    if b is not None and Sb is None:
        Sb = torch.empty(bl.m, dtype=torch.float64, device=A.device)
    elif b is not None:
        _check_out(Sb, (bl.m,), "Sb")
    alpha = c_s(bl.s) if alpha is None else float(alpha)
    rc = lib.skh_sketch_dense(bl.m, bl.s, _ptr(bl.ptr), _ptr(bl.rows), _ptr(bl.signs), n, d, _ptr(A), _ld(A),
                              _ptr(b), _ptr(SA), _ld(SA), _ptr(Sb), alpha, _stream())
    _lib.check(rc, "skh_sketch_dense")
    return SA, Sb


def sketch_csr_workspace(nrows, s, nnz, device=None):
    lib = _lib.load()
    device = device or torch.device("cuda", torch.cuda.current_device())
    return _workspace(lib.skh_sketch_csr_workspace_bytes(int(nrows), int(s), int(nnz)), device)


def sketch_csr(bl, row_ptr, col_idx, val, d, b=None, alpha=None, SA=None, Sb=None, ws=None):
    """R5 sparse (CSR A): dense SA = alpha * S A (nnz = len(val))."""
    lib = _lib.load()
    _need_cuda(row_ptr, col_idx, val, b)
    n = row_ptr.numel() - 1
    nnz = val.numel()
    dev = row_ptr.device
    if SA is None:
        SA = torch.empty(bl.m, d, dtype=torch.float64, device=dev)
    else:
        _check_out(SA, (bl.m, d), "SA")
    if b is not None and Sb is None:
        Sb = torch.empty(bl.m, dtype=torch.float64, device=dev)
    elif b is not None:
        _check_out(Sb, (bl.m,), "Sb")
    if ws is None:
        ws = sketch_csr_workspace(n, bl.s, nnz, dev)
    alpha = c_s(bl.s) if alpha is None else float(alpha)
    rc = lib.skh_sketch_csr(bl.m, bl.s, _ptr(bl.ptr), _ptr(bl.rows), _ptr(bl.signs), n, int(d), nnz, _ptr(row_ptr),
                            _ptr(col_idx), _ptr(val), _ptr(b), _ptr(SA), _ld(SA), _ptr(Sb), alpha, _ptr(ws),
                            ws.numel(), _stream())
    _lib.check(rc, "skh_sketch_csr")
    return SA, Sb


def launch_count():
    """Kernels enqueued through libskh by this process so far."""
    return int(_lib.load().skh_launch_count())


def rht_pass_plan(nbits, d, aligned=True):
    """Stage counts of the HBM passes skh_rht_stages uses (low bits first)."""
    import ctypes
    lib = _lib.load()
    buf = (ctypes.c_int * 64)()
    k = lib.skh_rht_pass_plan(int(nbits), int(d), int(bool(aligned)), buf, 64)
    return [buf[i] for i in range(k)]


def rht_stages_workspace(nrows, nvalid=None, row0=0, d=1, device=None):
    lib = _lib.load()
    device = device or torch.device("cuda", torch.cuda.current_device())
    nvalid = nrows if nvalid is None else nvalid
    return _workspace(lib.skh_rht_stages_workspace_bytes(int(nrows), int(nvalid), int(row0), int(d)), device)


def rht_stages(seed, X, bit_lo, bit_hi, nrows=None, row0=0, apply_diag=True, alpha=1.0, Y=None, ws=None):
    """R3+R4: Y = alpha * Hhat_[bit_lo,bit_hi) D? X along rows (X: nvalid x d)."""
    lib = _lib.load()
    _need_cuda(X)
    if X.dim() == 1:
        X = X.view(-1, 1)
        if Y is not None:
            Y = Y.view(-1, 1)
    nvalid, d = X.shape
    nrows = nvalid if nrows is None else int(nrows)
    if Y is None:
        Y = torch.empty(nrows, d, dtype=torch.float64, device=X.device)
    else:
        _check_out(Y, (nrows, d), "Y")
    if ws is None:
        ws = rht_stages_workspace(nrows, nvalid, row0, d, X.device)
    rc = lib.skh_rht_stages(int(seed) & (2**64 - 1), nrows, nvalid, int(row0), d, _ptr(X), _ld(X), _ptr(Y), _ld(Y),
                            int(bit_lo), int(bit_hi), int(bool(apply_diag)), float(alpha), _ptr(ws),
                            0 if ws is None else ws.numel(), _stream())
    _lib.check(rc, "skh_rht_stages")
    return Y


class RhtDense:
    """Reusable workspace for skh_rht_dense (one allocation per shape)."""

    def __init__(self, n, m, s, d, device=None):
        lib = _lib.load()
        self.n, self.m, self.s, self.d = int(n), int(m), int(s), int(d)
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.ws = _workspace(lib.skh_rht_dense_workspace_bytes(n, m, s, d), device)

    def __call__(self, seed, A, b=None, SA=None, Sb=None):
        lib = _lib.load()
        _need_cuda(A, b)
        if SA is None:
            SA = torch.empty(self.m, self.d, dtype=torch.float64, device=A.device)
        else:
            _check_out(SA, (self.m, self.d), "SA")
        if b is not None and Sb is None:
            Sb = torch.empty(self.m, dtype=torch.float64, device=A.device)
        elif b is not None:
            _check_out(Sb, (self.m,), "Sb")
        rc = lib.skh_rht_dense(int(seed) & (2**64 - 1), self.n, self.m, self.s, self.d, _ptr(A), _ld(A), _ptr(b),
                               _ptr(SA), _ld(SA), _ptr(Sb), _ptr(self.ws), self.ws.numel(), _stream())
        _lib.check(rc, "skh_rht_dense")
        return SA, Sb

    def from_host(self, seed, A_host, b_host=None, SA_host=None, Sb_host=None):
        """Same from host (pinned) tensors; returns host SA, Sb after syncing the stream."""
        lib = _lib.load()
        if A_host.is_cuda:
            raise ValueError("from_host takes CPU tensors")
        if SA_host is None:
            SA_host = torch.empty(self.m, self.d, dtype=torch.float64, pin_memory=True)
        if b_host is not None and Sb_host is None:
            Sb_host = torch.empty(self.m, dtype=torch.float64, pin_memory=True)
        rc = lib.skh_rht_dense_host(int(seed) & (2**64 - 1), self.n, self.m, self.s, self.d, _ptr(A_host),
                                    _ld(A_host), _ptr(b_host), _ptr(SA_host), _ld(SA_host), _ptr(Sb_host),
                                    _ptr(self.ws), self.ws.numel(), _stream())
        _lib.check(rc, "skh_rht_dense_host")
        torch.cuda.current_stream().synchronize()
        return SA_host, Sb_host


def rht_dense(seed, A, b, m, s):
    """R1-R5 on one GPU: SA = S_h H D A, Sb = S_h H D b (HRHT, L790-801)."""
    n, d = A.shape
    return RhtDense(n, m, s, d, A.device)(seed, A, b)


class SketchDenseHost:
    """Workspace + call for skh_sketch_dense_host (plain s-hashing from host buffers)."""

    def __init__(self, n, m, s, d, device=None):
        lib = _lib.load()
        self.n, self.m, self.s, self.d = int(n), int(m), int(s), int(d)
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.ws = _workspace(lib.skh_sketch_dense_workspace_bytes(n, m, s, d), device)

    def __call__(self, seed, A_host, b_host=None, SA_host=None, Sb_host=None):
        lib = _lib.load()
        if SA_host is None:
            SA_host = torch.empty(self.m, self.d, dtype=torch.float64, pin_memory=True)
        if b_host is not None and Sb_host is None:
            Sb_host = torch.empty(self.m, dtype=torch.float64, pin_memory=True)
        rc = lib.skh_sketch_dense_host(int(seed) & (2**64 - 1), self.n, self.m, self.s, self.d, _ptr(A_host),
                                       _ld(A_host), _ptr(b_host), _ptr(SA_host), _ld(SA_host), _ptr(Sb_host),
                                       _ptr(self.ws), self.ws.numel(), _stream())
        _lib.check(rc, "skh_sketch_dense_host")
        torch.cuda.current_stream().synchronize()
        return SA_host, Sb_host


def scale(X, alpha):
    lib = _lib.load()
    _need_cuda(X)
    rows, cols = X.shape
    _lib.check(lib.skh_scale(_ptr(X), rows, cols, _ld(X), float(alpha), _stream()), "skh_scale")
    return X


def fold_lists(bl, L, rank):
    """In place: bucket lists of all n columns of S (global rows) -> the lists of
    T_rank = sum_g (-1)^popcount(g & rank) S_g over local rows j mod L
    (skh_fold_lists; the exchange-free sharded H D A)."""
    lib = _lib.load()
    _need_cuda(bl.rows)
    _lib.check(lib.skh_fold_lists(bl.rows.numel(), _ptr(bl.rows), _ptr(bl.signs), int(L), int(rank), _stream()),
               "skh_fold_lists")
    bl.nrows = int(L)
    return bl


def ordered_sum(parts, alpha=1.0, out=None):
    """parts: [G, rows, cols] contiguous; out = alpha * (((P0 + P1) + P2) + ...)."""
    lib = _lib.load()
    _need_cuda(parts)
    G, rows, cols = parts.shape
    if out is None:
        out = torch.empty(rows, cols, dtype=torch.float64, device=parts.device)
    rc = lib.skh_ordered_sum(_ptr(parts), G, parts.stride(0), rows, cols, parts.stride(1), _ptr(out), _ld(out),
                             float(alpha), _stream())
    _lib.check(rc, "skh_ordered_sum")
    return out


# ---------------------------------------------------------------- column-major A
# The paper's own storage (LAPACK/FFTW, L1073-1081).  A torch tensor ``At`` of
# shape (d, n) with unit last stride IS a column-major n x d matrix with
# lda = At.stride(0); SA comes back the same way, as a (d, m) tensor = SA^T.

def _ld_cm(t, rows):
    if t.dim() == 2 and t.size(0) <= 1 and (t.stride(1) == 1 or t.size(1) <= 1):
        return max(rows, 1)                  # one column: its leading stride is never used
    if t.dim() != 2 or (t.stride(1) != 1 and t.size(1) > 1) or t.stride(0) < rows:
        raise ValueError("expected a (cols, rows) tensor with unit last stride (column-major storage)")
    return t.stride(0)


def fold_cols(col_rows, col_signs, L, G, s, rank, out=None):
    """T_r's column lists over L local rows from the column lists of all n = G L
    columns of S (skh_fold_cols; the column-major exchange-free sharded H D A,
    DESIGN.md §7).  Returns (rows, signs) of L G s entries."""
    lib = _lib.load()
    _need_cuda(col_rows, col_signs)
    N = int(L) * int(G) * int(s)
    if out is None:
        out = (torch.empty(N, dtype=torch.int32, device=col_rows.device),
               torch.empty(N, dtype=torch.int8, device=col_rows.device))
    _lib.check(lib.skh_fold_cols(int(L), int(G), int(s), int(rank), _ptr(col_rows), _ptr(col_signs), _ptr(out[0]),
                                 _ptr(out[1]), _stream()), "skh_fold_cols")
    return out


class RhtColMajorLists:
    """SA^T = alpha * S' H_L D A_r for a column-major local block At (d, L) with
    caller-given column lists (s_eff per row of the transform, next power of two
    >= L rows; skh_rht_colmajor_lists), D over global ids row0 + l.  The M3 rank
    step; returns SA^T (d, m) and Sb."""

    def __init__(self, L, m, s_eff, d, device=None):
        lib = _lib.load()
        self.L, self.m, self.s_eff, self.d = int(L), int(m), int(s_eff), int(d)
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.ws = _workspace(lib.skh_rht_colmajor_lists_workspace_bytes(L, m, s_eff, d), device)

    def __call__(self, seed, At, b, row0, col_rows, col_signs, alpha=1.0, SAt=None, Sb=None):
        lib = _lib.load()
        _need_cuda(At, b, col_rows, col_signs)
        if tuple(At.shape) != (self.d, self.L) or At.dtype != torch.float64:
            raise ValueError(f"At must be float64 of shape (d, L) = ({self.d}, {self.L})")
        if SAt is None:
            SAt = torch.empty(self.d, self.m, dtype=torch.float64, device=At.device)
        else:
            _check_out(SAt, (self.d, self.m), "SAt")
        if b is not None and Sb is None:
            Sb = torch.empty(self.m, dtype=torch.float64, device=At.device)
        elif b is not None:
            _check_out(Sb, (self.m,), "Sb")
        rc = lib.skh_rht_colmajor_lists(int(seed) & (2**64 - 1), self.L, int(row0), self.m, self.s_eff, self.d,
                                        _ptr(At), _ld_cm(At, self.L), _ptr(b), _ptr(col_rows), _ptr(col_signs),
                                        float(alpha), _ptr(SAt), _ld_cm(SAt, self.m), _ptr(Sb), _ptr(self.ws),
                                        self.ws.numel(), _stream())
        _lib.check(rc, "skh_rht_colmajor_lists")
        return SAt, Sb


class RhtDenseColMajor:
    """SA = S_h H D A for column-major A (skh_rht_dense_colmajor): two HBM passes,
    the second fused with the sketch.  Returns SA^T (d, m) and Sb."""

    def __init__(self, n, m, s, d, device=None):
        lib = _lib.load()
        self.n, self.m, self.s, self.d = int(n), int(m), int(s), int(d)
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.ws = _workspace(lib.skh_rht_dense_colmajor_workspace_bytes(n, m, s, d), device)

    def __call__(self, seed, At, b=None, SAt=None, Sb=None):
        lib = _lib.load()
        _need_cuda(At, b)
        if tuple(At.shape) != (self.d, self.n) or At.dtype != torch.float64:
            raise ValueError(f"At must be float64 of shape (d, n) = ({self.d}, {self.n})")
        if SAt is None:
            SAt = torch.empty(self.d, self.m, dtype=torch.float64, device=At.device)
        else:
            _check_out(SAt, (self.d, self.m), "SAt")
        if b is not None and Sb is None:
            Sb = torch.empty(self.m, dtype=torch.float64, device=At.device)
        elif b is not None:
            _check_out(Sb, (self.m,), "Sb")
        rc = lib.skh_rht_dense_colmajor(int(seed) & (2**64 - 1), self.n, self.m, self.s, self.d, _ptr(At),
                                        _ld_cm(At, self.n), _ptr(b), _ptr(SAt), _ld_cm(SAt, self.m), _ptr(Sb),
                                        _ptr(self.ws), self.ws.numel(), _stream())
        _lib.check(rc, "skh_rht_dense_colmajor")
        return SAt, Sb

    def from_host(self, seed, At_host, b_host=None, SAt_host=None, Sb_host=None):
        """Same from host (pinned) tensors; returns host SA^T, Sb after syncing the stream."""
        lib = _lib.load()
        if At_host.is_cuda:
            raise ValueError("from_host takes CPU tensors")
        if SAt_host is None:
            SAt_host = torch.empty(self.d, self.m, dtype=torch.float64, pin_memory=True)
        if b_host is not None and Sb_host is None:
            Sb_host = torch.empty(self.m, dtype=torch.float64, pin_memory=True)
        rc = lib.skh_rht_dense_colmajor_host(int(seed) & (2**64 - 1), self.n, self.m, self.s, self.d,
                                             _ptr(At_host), _ld_cm(At_host, self.n), _ptr(b_host), _ptr(SAt_host),
                                             _ld_cm(SAt_host, self.m), _ptr(Sb_host), _ptr(self.ws),
                                             self.ws.numel(), _stream())
        _lib.check(rc, "skh_rht_dense_colmajor_host")
        torch.cuda.current_stream().synchronize()
        return SAt_host, Sb_host


def rht_dense_colmajor(seed, At, b, m, s):
    """SA^T, Sb for column-major A given as At (d, n)."""
    d, n = At.shape
    return RhtDenseColMajor(n, m, s, d, At.device)(seed, At, b)


def sketch_dense_colmajor(seed, At, b, m, s, SAt=None, Sb=None, ws=None, fast=True):
    """Plain s-hashing SA = S A of column-major A (At: (d, n)); bit-identical to sketch_dense.
    fast=True sizes the workspace for the transposed path (a row-major copy of A),
    fast=False for the on-chip walk (skh.h)."""
    lib = _lib.load()
    _need_cuda(At, b)
    d, n = At.shape
    if SAt is None:
        SAt = torch.empty(d, m, dtype=torch.float64, device=At.device)
    else:
        _check_out(SAt, (d, m), "SAt")
    if b is not None and Sb is None:
        Sb = torch.empty(m, dtype=torch.float64, device=At.device)
    elif b is not None:
        _check_out(Sb, (m,), "Sb")
    if ws is None:
        nb = (lib.skh_sketch_dense_colmajor_fast_workspace_bytes(n, m, s, d) if fast
              else lib.skh_sketch_dense_colmajor_workspace_bytes(n, m, s))
        ws = _workspace(nb, At.device)
    rc = lib.skh_sketch_dense_colmajor(int(seed) & (2**64 - 1), n, int(m), int(s), d, _ptr(At), _ld_cm(At, n),
                                       _ptr(b), _ptr(SAt), _ld_cm(SAt, m), _ptr(Sb), _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "skh_sketch_dense_colmajor")
    return SAt, Sb


def rht_colmajor(seed, Xt, nrows=None, row0=0, apply_diag=True, Yt=None):
    """Yt = (Hhat D? X)^T for column-major X given as Xt (ncols, nvalid): unnormalised, all stages."""
    lib = _lib.load()
    _need_cuda(Xt)
    if Xt.dim() == 1:
        Xt = Xt.view(1, -1)
    ncols, nvalid = Xt.shape
    nrows = nvalid if nrows is None else int(nrows)
    if Yt is None:
        Yt = torch.empty(ncols, nrows, dtype=torch.float64, device=Xt.device)
    ldx = _ld_cm(Xt, nvalid) if ncols > 1 else max(Xt.stride(0), nvalid)
    ldy = _ld_cm(Yt, nrows) if ncols > 1 else max(Yt.stride(0), nrows)
    if Xt.stride(-1) != 1 or Yt.stride(-1) != 1:
        raise ValueError("rht_colmajor: columns must be contiguous (unit last stride)")
    rc = lib.skh_rht_colmajor(int(seed) & (2**64 - 1), nrows, nvalid, int(row0), ncols, _ptr(Xt), ldx, _ptr(Yt),
                              ldy, int(bool(apply_diag)), _stream())
    _lib.check(rc, "skh_rht_colmajor")
    return Yt


class Trace:
    """Per-stage CUDA events recorded by the library's composite calls (skh_trace_set)."""

    def __init__(self, n=16):
        import ctypes
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        for e in self.events:  # torch creates the CUDA event lazily
            e.record()
        torch.cuda.synchronize()
        self._arr = (ctypes.c_void_p * n)(*[e.cuda_event for e in self.events])

    def __enter__(self):
        _lib.check(_lib.load().skh_trace_set(self._arr, len(self.events)), "skh_trace_set")
        return self

    def __exit__(self, *exc):
        lib = _lib.load()
        self.count = lib.skh_trace_count()
        self.names = [lib.skh_trace_name(i).decode() for i in range(self.count)]
        lib.skh_trace_set(None, 0)
        return False

    def durations_ms(self):
        """{stage: ms} of the last traced call (synchronize first).  Stages the
        library ran on its side stream (trace names "side:...") form their own
        chain from the first event and are reported as "<stage> (overlapped)",
        outside the main-stream sum."""
        out = {}
        prev = {False: 0, True: 0}
        for i in range(1, self.count):
            side = self.names[i].startswith("side:")
            name = self.names[i][5:] + " (overlapped)" if side else self.names[i]
            out[name] = out.get(name, 0.0) + self.events[prev[side]].elapsed_time(self.events[i])
            prev[side] = i
        return out


# ---------------------------------------------------------------- Algorithm 1 Steps 2-5
class LlsSolver:
    """x ~ argmin ||A x - b|| from Step 1's SA, Sb (skh_lls_solve; row-major A).

    Defaults are the paper's.  rcond=None: the full-rank QR mode
    (DGEQRF, L1077); rcond=1e-12: the paper's default rank-revealing Step 2
    (column-pivoted QR, p = max{q : |r_qq| >= rcond}, L1109-1112;
    skh_lls_solve_rr)."""

    def __init__(self, n, d, m, device=None, rcond=None):
        lib = _lib.load()
        self.n, self.d, self.m = int(n), int(d), int(m)
        self.rcond = rcond
        device = device or torch.device("cuda", torch.cuda.current_device())
        q = lib.skh_lls_workspace_bytes if rcond is None else lib.skh_lls_rr_workspace_bytes
        nb = q(self.n, self.d, self.m)
        if nb == 0:
            raise ValueError("lls workspace query failed: " + lib.skh_last_error().decode())
        self.ws = _workspace(nb, device)

    def __call__(self, A, b, SA, Sb, tau_a=1e-8, tau_r=1e-6, it_max=10000, x=None, x_s=None, colmajor=False):
        """colmajor=True: A given as At (d, n) and SA as SAt (d, m) (skh_lls_solve_colmajor)."""
        import ctypes
        lib = _lib.load()
        _need_cuda(A, b, SA, Sb)
        if x is None:
            x = torch.empty(self.d, dtype=torch.float64, device=A.device)
        info = (ctypes.c_int64 * 3)()
        stats = (ctypes.c_double * 3)()
        if self.rcond is not None:
            f = lib.skh_lls_solve_rr_colmajor if colmajor else lib.skh_lls_solve_rr
            lda = _ld_cm(A, self.n) if colmajor else _ld(A)
            ldsa = _ld_cm(SA, self.m) if colmajor else _ld(SA)
            rc = f(self.n, self.d, _ptr(A), lda, _ptr(b), self.m, _ptr(SA), ldsa, _ptr(Sb), float(self.rcond),
                   float(tau_a), float(tau_r), int(it_max), _ptr(x), _ptr(x_s), info, stats, _ptr(self.ws),
                   self.ws.numel(), _stream())
            _lib.check(rc, "skh_lls_solve_rr")
            return x, {"step": int(info[0]), "iters": int(info[1]), "rank": int(info[2]), "test2": stats[0],
                       "rnorm": stats[1], "res_s": stats[2]}
        if colmajor:
            rc = lib.skh_lls_solve_colmajor(self.n, self.d, _ptr(A), _ld_cm(A, self.n), _ptr(b), self.m, _ptr(SA),
                                            _ld_cm(SA, self.m), _ptr(Sb), float(tau_a), float(tau_r), int(it_max),
                                            _ptr(x), _ptr(x_s), info, stats, _ptr(self.ws), self.ws.numel(),
                                            _stream())
        else:
            rc = lib.skh_lls_solve(self.n, self.d, _ptr(A), _ld(A), _ptr(b), self.m, _ptr(SA), _ld(SA), _ptr(Sb),
                                   float(tau_a), float(tau_r), int(it_max), _ptr(x), _ptr(x_s), info, stats,
                                   _ptr(self.ws), self.ws.numel(), _stream())
        _lib.check(rc, "skh_lls_solve_colmajor" if colmajor else "skh_lls_solve")
        return x, {"step": int(info[0]), "iters": int(info[1]), "test2": stats[0], "rnorm": stats[1],
                   "res_s": stats[2]}


def lls_solve(A, b, SA, Sb, rcond=None, **kw):
    n, d = A.shape
    return LlsSolver(n, d, SA.shape[0], A.device, rcond=rcond)(A, b, SA, Sb, **kw)


# ---------------------------------------------------------------- HR-DHT (eq. (6.1))
def hrdht_dense(seed, A, b, m, s, SA=None, Sb=None, ws=None):
    """SA = S_h F D A, Sb = S_h F D b with F the normalised DHT (any n); row-major A."""
    lib = _lib.load()
    _need_cuda(A, b)
    n, d = A.shape
    if SA is None:
        SA = torch.empty(m, d, dtype=torch.float64, device=A.device)
    else:
        _check_out(SA, (m, d), "SA")
    if b is not None and Sb is None:
        Sb = torch.empty(m, dtype=torch.float64, device=A.device)
    elif b is not None:
        _check_out(Sb, (m,), "Sb")
    if ws is None:
        nb = lib.skh_hrdht_dense_workspace_bytes(n, int(m), int(s), d)
        if nb == 0:
            raise ValueError("skh_hrdht_dense_workspace_bytes failed: " + lib.skh_last_error().decode())
        ws = _workspace(nb, A.device)
    rc = lib.skh_hrdht_dense(int(seed) & (2**64 - 1), n, int(m), int(s), d, _ptr(A), _ld(A), _ptr(b), _ptr(SA),
                             _ld(SA), _ptr(Sb), _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "skh_hrdht_dense")
    return SA, Sb


def hrdht_dense_colmajor(seed, At, b, m, s, SAt=None, Sb=None, ws=None):
    """Same for column-major A given as At (d, n); returns SA^T (d, m), Sb."""
    lib = _lib.load()
    _need_cuda(At, b)
    d, n = At.shape
    if SAt is None:
        SAt = torch.empty(d, m, dtype=torch.float64, device=At.device)
    else:
        _check_out(SAt, (d, m), "SAt")
    if b is not None and Sb is None:
        Sb = torch.empty(m, dtype=torch.float64, device=At.device)
    elif b is not None:
        _check_out(Sb, (m,), "Sb")
    if ws is None:
        nb = lib.skh_hrdht_dense_colmajor_workspace_bytes(n, int(m), int(s), d)
        if nb == 0:
            raise ValueError("skh_hrdht_dense_colmajor_workspace_bytes failed: " + lib.skh_last_error().decode())
        ws = _workspace(nb, At.device)
    rc = lib.skh_hrdht_dense_colmajor(int(seed) & (2**64 - 1), n, int(m), int(s), d, _ptr(At), _ld_cm(At, n),
                                      _ptr(b), _ptr(SAt), _ld_cm(SAt, m), _ptr(Sb), _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "skh_hrdht_dense_colmajor")
    return SAt, Sb


def srdht_dense(seed, A, b, m, SA=None, Sb=None, ws=None):
    """SR-DHT (Blendenpik, eq. (7.2)): SA = S_s F D A with uniform row sampling."""
    lib = _lib.load()
    _need_cuda(A, b)
    n, d = A.shape
    if SA is None:
        SA = torch.empty(m, d, dtype=torch.float64, device=A.device)
    else:
        _check_out(SA, (m, d), "SA")
    if b is not None and Sb is None:
        Sb = torch.empty(m, dtype=torch.float64, device=A.device)
    elif b is not None:
        _check_out(Sb, (m,), "Sb")
    if ws is None:
        nb = lib.skh_srdht_dense_workspace_bytes(n, int(m), d)
        if nb == 0:
            raise ValueError("skh_srdht_dense_workspace_bytes failed: " + lib.skh_last_error().decode())
        ws = _workspace(nb, A.device)
    rc = lib.skh_srdht_dense(int(seed) & (2**64 - 1), n, int(m), d, _ptr(A), _ld(A), _ptr(b), _ptr(SA), _ld(SA),
                             _ptr(Sb), _ptr(ws), ws.numel(), _stream())
    _lib.check(rc, "skh_srdht_dense")
    return SA, Sb


def ski_lls_dense(A, b, m=None, s=1, seed=0, transform="dht", tau_a=1e-8, tau_r=1e-6, it_max=10000):
    """Ski-LLS-dense: Step 1 with the paper's dense sketch
    S = S_h F D (transform="dht", eq. (6.1)) or the HRHT S_h H D (transform="wht",
    Def. def::HRHT), then Steps 2-5 (skh_lls_solve).  Defaults are the paper's:
    m = 1.7 d, s = 1, tau_a = 1e-8, tau_r = 1e-6, it_max = 1e4.
    Row-major A.  Returns (x, info)."""
    n, d = A.shape
    m = int(m) if m is not None else max(d, int(math.ceil(1.7 * d)))
    if transform == "dht":
        SA, Sb = hrdht_dense(seed, A, b, m, s)
    elif transform == "wht":
        SA, Sb = rht_dense(seed, A, b, m, s)
    else:
        raise ValueError("transform must be 'dht' or 'wht'")
    return LlsSolver(n, d, m, A.device)(A, b, SA, Sb, tau_a=tau_a, tau_r=tau_r, it_max=it_max)
