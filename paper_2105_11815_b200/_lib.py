"""ctypes loader for libskh.so (the C ABI declared in include/skh.h).

Argument marshalling only.  There is no fallback: if the library or a CUDA
device is missing, the calls raise.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libskh.so")

c_i32, c_i64, c_u64, c_sz, c_d, c_p = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t,
                                       ctypes.c_double, ctypes.c_void_p)

# name -> (restype, argtypes); mirrors include/skh.h
SIGNATURES = {
    "skh_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "skh_last_error": (ctypes.c_char_p, []),
    "skh_abi_version": (ctypes.c_int, []),
    "skh_launch_count": (c_u64, []),
    "skh_c_s": (c_d, [c_i32]),
    "skh_c_n": (c_d, [c_i64]),
    "skh_c_ns": (c_d, [c_i64, c_i32]),
    "skh_hash_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32]),
    "skh_hash_gen": (ctypes.c_int, [c_u64, c_i64, c_i32, c_i64, c_i64, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p, c_p,
                                    c_sz, c_p]),
    "skh_hash_gen_variant": (ctypes.c_int, [c_u64, c_i64, c_i32, c_i64, c_i64, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p,
                                            c_p, c_sz, c_p]),
    "skh_hash_status": (ctypes.c_int, [c_p, c_p]),
    "skh_sketch_dense": (ctypes.c_int, [c_i64, c_i32, c_p, c_p, c_p, c_i64, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p,
                                        c_d, c_p]),
    "skh_sketch_csr_workspace_bytes": (c_sz, [c_i64, c_i32, c_i64]),
    "skh_sketch_csr": (ctypes.c_int, [c_i64, c_i32, c_p, c_p, c_p, c_i64, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p, c_i64,
                                      c_p, c_d, c_p, c_sz, c_p]),
    "skh_rht_stages_workspace_bytes": (c_sz, [c_i64, c_i64, c_i64, c_i64]),
    "skh_rht_pass_plan": (ctypes.c_int, [ctypes.c_int, c_i64, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                         ctypes.c_int]),
    "skh_rht_stages": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i64, c_i64, c_p, c_i64, c_p, c_i64, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, c_d, c_p, c_sz, c_p]),
    "skh_rht_dense_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32, c_i64]),
    "skh_rht_dense": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p, c_p, c_sz,
                                     c_p]),
    "skh_rht_dense_host": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p, c_p,
                                          c_sz, c_p]),
    "skh_sketch_dense_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32, c_i64]),
    "skh_sketch_dense_host": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p, c_p,
                                             c_sz, c_p]),
    "skh_scale": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_d, c_p]),
    "skh_ordered_sum": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_i64, c_i64, c_p, c_i64, c_d, c_p]),
    "skh_fold_lists": (ctypes.c_int, [c_i64, c_p, c_p, c_i64, c_i64, c_p]),
    "skh_fold_cols": (ctypes.c_int, [c_i64, c_i64, c_i32, c_i64, c_p, c_p, c_p, c_p, c_p]),
    "skh_rht_colmajor_lists_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32, c_i64]),
    "skh_rht_colmajor_lists": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_p, c_p,
                                              c_d, c_p, c_i64, c_p, c_p, c_sz, c_p]),
    "skh_rht_dense_colmajor_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32, c_i64]),
    "skh_rht_dense_colmajor": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p,
                                              c_p, c_sz, c_p]),
    "skh_rht_dense_colmajor_host": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_p, c_i64,
                                                   c_p, c_p, c_sz, c_p]),
    "skh_sketch_dense_colmajor_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32]),
    "skh_sketch_dense_colmajor_fast_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32, c_i64]),
    "skh_sketch_dense_colmajor": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p,
                                                 c_p, c_sz, c_p]),
    "skh_rht_colmajor": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i64, c_i64, c_p, c_i64, c_p, c_i64, ctypes.c_int,
                                        c_p]),
    "skh_hrdht_dense_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32, c_i64]),
    "skh_hrdht_dense": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p, c_p, c_sz,
                                       c_p]),
    "skh_hrdht_dense_colmajor_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32, c_i64]),
    "skh_hrdht_dense_colmajor": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p,
                                                c_p, c_sz, c_p]),
    "skh_srdht_dense_workspace_bytes": (c_sz, [c_i64, c_i64, c_i64]),
    "skh_srdht_dense": (ctypes.c_int, [c_u64, c_i64, c_i64, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p, c_p, c_sz, c_p]),
    "skh_lls_workspace_bytes": (c_sz, [c_i64, c_i64, c_i64]),
    "skh_lls_solve": (ctypes.c_int, [c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_d, c_d, c_i64, c_p,
                                     c_p, ctypes.POINTER(c_i64), ctypes.POINTER(c_d), c_p, c_sz, c_p]),
    "skh_lls_solve_colmajor": (ctypes.c_int, [c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_d, c_d, c_i64,
                                              c_p, c_p, ctypes.POINTER(c_i64), ctypes.POINTER(c_d), c_p, c_sz, c_p]),
    "skh_lls_rr_workspace_bytes": (c_sz, [c_i64, c_i64, c_i64]),
    "skh_lls_solve_rr": (ctypes.c_int, [c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_d, c_d, c_d, c_i64,
                                        c_p, c_p, ctypes.POINTER(c_i64), ctypes.POINTER(c_d), c_p, c_sz, c_p]),
    "skh_lls_solve_rr_colmajor": (ctypes.c_int, [c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_d, c_d, c_d,
                                                 c_i64, c_p, c_p, ctypes.POINTER(c_i64), ctypes.POINTER(c_d), c_p, c_sz,
                                                 c_p]),
    "skh_trace_set": (ctypes.c_int, [ctypes.POINTER(c_p), ctypes.c_int]),
    "skh_trace_count": (ctypes.c_int, []),
    "skh_trace_name": (ctypes.c_char_p, [ctypes.c_int]),
}

_lib = None


class SkhError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        lib = _lib
        msg = lib.skh_strerror(code).decode() if lib else str(code)
        detail = lib.skh_last_error().decode() if lib else ""
        super().__init__(f"{where}: {msg} ({detail})")


def load():
    """Load libskh.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2105_11815_b200.build`"
                           " (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(code, where):
    if code != 0:
        raise SkhError(code, where)
