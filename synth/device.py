"""Device-side synthetic inputs (libsynth.so): same values as synth/gen.py."""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

KIND = {"dense_gauss": 0, "dense_coherent": 1}


def load():
    global _lib
    if _lib is None:
        p = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(p):
            raise RuntimeError(f"{p} missing: run python -m paper_2105_11815_b200.build")
        lib = ctypes.CDLL(p)
        i64, u64, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        lib.synth_dense.argtypes = [ctypes.c_int, u64, i64, i64, i64, i64, vp, i64, vp]
        lib.synth_dense_cm.argtypes = [ctypes.c_int, u64, i64, i64, i64, i64, vp, i64, vp]
        lib.synth_rhs.argtypes = [u64, i64, i64, vp, vp]
        lib.synth_csr.argtypes = [u64, i64, ctypes.c_int, i64, i64, vp, vp, vp, vp, vp]
        lib.synth_small_int.argtypes = [u64, i64, i64, ctypes.c_int, ctypes.c_int, vp, vp]
        _lib = lib
    return _lib


def _st():
    return torch.cuda.current_stream().cuda_stream


def dense(cfg, r0=0, r1=None, out=None, device="cuda"):
    """Rows [r0, r1) of the config's dense A, generated on the device."""
    r1 = cfg.n if r1 is None else r1
    if out is None:
        out = torch.empty(r1 - r0, cfg.d, dtype=torch.float64, device=device)
    rc = load().synth_dense(KIND[cfg.kind], cfg.seed, cfg.n, cfg.d, r0, r1 - r0, out.data_ptr(), out.stride(0), _st())
    if rc:
        raise RuntimeError("synth_dense failed")
    return out


def dense_colmajor(cfg, r0=0, r1=None, out=None, device="cuda"):
    """Rows [r0, r1) of the config's dense A stored column-major: a (d, r1 - r0)
    tensor At with At[c, i] = A[r0 + i, c] (same values as dense())."""
    r1 = cfg.n if r1 is None else r1
    if out is None:
        out = torch.empty(cfg.d, r1 - r0, dtype=torch.float64, device=device)
    rc = load().synth_dense_cm(KIND[cfg.kind], cfg.seed, cfg.n, cfg.d, r0, r1 - r0, out.data_ptr(), out.stride(0),
                               _st())
    if rc:
        raise RuntimeError("synth_dense_cm failed")
    return out


def rhs(cfg, r0=0, r1=None, device="cuda"):
    r1 = cfg.n if r1 is None else r1
    out = torch.empty(r1 - r0, dtype=torch.float64, device=device)
    if load().synth_rhs(cfg.seed, r0, r1 - r0, out.data_ptr(), _st()):
        raise RuntimeError("synth_rhs failed")
    return out


def csr(cfg, r0=0, r1=None, device="cuda"):
    r1 = cfg.n if r1 is None else r1
    nr = r1 - r0
    rp = torch.empty(nr + 1, dtype=torch.int64, device=device)
    ci = torch.empty(nr * cfg.nnz_row, dtype=torch.int32, device=device)
    v = torch.empty(nr * cfg.nnz_row, dtype=torch.float64, device=device)
    fail = torch.zeros(1, dtype=torch.int32, device=device)
    if load().synth_csr(cfg.seed, cfg.d, cfg.nnz_row, r0, nr, rp.data_ptr(), ci.data_ptr(), v.data_ptr(),
                        fail.data_ptr(), _st()):
        raise RuntimeError("synth_csr failed")
    return rp, ci, v


def small_int(seed, n, d, lo=-3, hi=3, device="cuda"):
    out = torch.empty(n, d, dtype=torch.float64, device=device)
    if load().synth_small_int(seed, n, d, lo, hi, out.data_ptr(), _st()):
        raise RuntimeError("synth_small_int failed")
    return out
