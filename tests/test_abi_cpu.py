"""CPU checks of the C ABI: libskh.so loads, exports every function declared in
include/skh.h, and rejects bad arguments with the documented codes before any
CUDA work (validation paths only; no compute without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2105_11815_b200 import _lib, build
    build.build()
    return _lib.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "skh.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(skh_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    from paper_2105_11815_b200 import _lib
    names = header_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), "binding table out of sync with include/skh.h"
    assert lib.skh_abi_version() == 1


def test_constants(lib):
    # DESIGN.md R5/R9/R10: one IEEE sqrt, one IEEE divide
    assert lib.skh_c_s(2) == 0.7071067811865475
    assert lib.skh_c_s(3) == 0.5773502691896258
    assert lib.skh_c_n(2 ** 16) == 2.0 ** -8
    assert lib.skh_c_n(2 ** 17) == 0.002762135864009951
    assert lib.skh_c_ns(2 ** 21, 1) == 0.0006905339660024878
    assert lib.skh_c_ns(2 ** 17, 2) == 2.0 ** -9


def test_error_codes(lib):
    EINVAL, ENOTPOW2, EDIM, EOVERFLOW, EWS = 1, 2, 3, 5, 6
    p = ctypes.c_void_p(8)  # never dereferenced: validation fails first
    # s > m, s < 1, m < 1, s > 64
    for m, s in [(4, 5), (4, 0), (0, 1), (100, 65)]:
        assert lib.skh_hash_gen(1, m, s, 10, 0, 0, 0, None, None, p, p, p, p, 1 << 20, None) == EINVAL
    assert lib.skh_hash_gen(1, 1 << 31, 1, 10, 0, 0, 0, None, None, p, p, p, p, 1 << 20, None) == EOVERFLOW
    assert lib.skh_hash_gen(1, 8, 2, 1 << 30, 0, 0, 0, None, None, p, p, p, p, 1 << 40, None) == EOVERFLOW
    assert lib.skh_hash_gen(1, 8, 2, 10, 0, 0, 0, None, None, p, p, p, None, 0, None) == EWS
    assert lib.skh_hash_gen(1, 8, 2, 10, 0, 16, 8, None, None, p, p, p, p, 1 << 20, None) == EDIM
    assert lib.skh_hash_gen(1, 8, 2, 10, 0, 0, 0, None, None, None, p, p, p, 1 << 20, None) == EINVAL
    # sketch_dense: lda < d, Sb missing with b
    assert lib.skh_sketch_dense(8, 2, p, p, p, 10, 4, p, 3, None, p, 4, None, 1.0, None) == EDIM
    assert lib.skh_sketch_dense(8, 2, p, p, p, 10, 4, p, 4, p, p, 4, None, 1.0, None) == EDIM
    assert lib.skh_sketch_dense(8, 9, p, p, p, 10, 4, p, 4, None, p, 4, None, 1.0, None) == EINVAL
    assert lib.skh_sketch_csr(8, 2, p, p, p, 10, 4, 80, p, p, p, None, p, 3, None, 1.0, p, 1 << 30, None) == EDIM
    assert lib.skh_sketch_csr(8, 2, p, p, p, 10, 4, 80, p, p, p, None, p, 4, None, 1.0, p, 16, None) == EWS
    assert lib.skh_sketch_csr(8, 2, p, p, p, 10, 4, 1 << 30, p, p, p, None, p, 4, None, 1.0, p, 1 << 40,
                              None) == EOVERFLOW
    # rht_stages: nrows not a multiple of 2^bit_hi; in place with padding
    assert lib.skh_rht_stages(1, 12, 12, 0, 4, p, 4, p, 4, 0, 3, 0, 1.0, None, 0, None) == ENOTPOW2
    assert lib.skh_rht_stages(1, 16, 12, 0, 4, p, 4, p, 4, 0, 4, 0, 1.0, None, 0, None) == EDIM
    assert lib.skh_rht_stages(1, 16, 16, 0, 4, p, 4, p, 4, 0, 4, 1, 1.0, None, 0, None) == EWS
    assert lib.skh_rht_stages(1, 16, 16, 0, 4, p, 4, p, 4, 0, 4, 0, 1.0, p, 8, None) == EWS
    # rht_dense: workspace too small
    assert lib.skh_rht_dense(1, 100, 10, 1, 4, p, 4, None, p, 4, None, p, 16, None) == EWS
    assert b"workspace" in lib.skh_last_error()
    assert lib.skh_rht_dense_host(1, 100, 10, 11, 4, p, 4, None, p, 4, None, p, 1 << 30, None) == EINVAL
    assert lib.skh_strerror(EWS) == b"workspace missing or too small"


def test_workspace_queries(lib):
    n, m, s, d = 1 << 21, 7168, 1, 4096
    ws = lib.skh_rht_dense_workspace_bytes(n, m, s, d)
    assert ws >= n * d * 8 and ws < n * d * 8 * 1.05
    assert lib.skh_hash_workspace_bytes(1000, 10, 3) >= 2 * 8 * 3000
    assert lib.skh_rht_stages_workspace_bytes(256, 130, 60, 8) >= 8 * 3 + 4 * 64


def test_product_has_no_fallback():
    """The binding refuses CPU tensors (there is no CPU path to fall back to)."""
    import torch

    import paper_2105_11815_b200 as p
    with pytest.raises(ValueError):
        p.api._need_cuda(torch.zeros(2))
    src = open(os.path.join(ROOT, "paper_2105_11815_b200", "api.py")).read()
    assert "oracle" not in src.replace("oracle side", "")


def test_error_codes_widened_entry_points(lib):
    """Validation of the column-major, variant, HR-DHT/SR-DHT and solve entry
    points (argument checks run before any CUDA work)."""
    EINVAL, ENOTPOW2, EDIM, EOVERFLOW, EWS = 1, 2, 3, 5, 6
    p = ctypes.c_void_p(8)
    # variant: the same argument rules as skh_hash_gen
    assert lib.skh_hash_gen_variant(1, 4, 5, 10, 0, 0, 0, None, None, p, p, p, p, 1 << 20, None) == EINVAL
    assert lib.skh_hash_gen_variant(1, 8, 2, 10, 0, 0, 0, None, None, p, p, p, None, 0, None) == EWS
    # column-major HRHT: s <= 8, lda >= n, ldsa >= m, Sb with b, workspace (any m: bucket ranges)
    assert lib.skh_rht_dense_colmajor(1, 100, 40, 9, 4, p, 100, None, p, 40, None, p, 1 << 30, None) == EINVAL
    assert lib.skh_rht_dense_colmajor(1, 100, 70000, 1, 4, p, 100, None, p, 70000, None, p, 64, None) == EWS
    assert lib.skh_rht_dense_colmajor(1, 100, 40, 1, 4, p, 99, None, p, 40, None, p, 1 << 30, None) == EDIM
    assert lib.skh_rht_dense_colmajor(1, 100, 40, 1, 4, p, 100, None, p, 39, None, p, 1 << 30, None) == EDIM
    assert lib.skh_rht_dense_colmajor(1, 100, 40, 1, 4, p, 100, p, p, 40, None, p, 1 << 30, None) == EDIM
    assert lib.skh_rht_dense_colmajor(1, 100, 40, 1, 4, p, 100, None, p, 40, None, p, 64, None) == EWS
    assert lib.skh_sketch_dense_colmajor(1, 100, 40, 2, 4, p, 50, None, p, 40, None, p, 1 << 30, None) == EDIM
    assert lib.skh_sketch_dense_colmajor(1, 100, 40, 2, 4, p, 100, None, p, 40, None, p, 16, None) == EWS
    # rht_colmajor: nrows must be a power of two, ld rules
    assert lib.skh_rht_colmajor(1, 12, 12, 0, 2, p, 12, p, 12, 1, None) == ENOTPOW2
    assert lib.skh_rht_colmajor(1, 16, 12, 0, 2, p, 11, p, 16, 1, None) == EDIM
    assert lib.skh_rht_colmajor(1, 16, 17, 0, 2, p, 17, p, 16, 1, None) == EINVAL
    # HR-DHT: s > 64 (row-major) / s > 8 (column-major), n*s overflow
    assert lib.skh_hrdht_dense(1, 100, 70, 65, 4, p, 4, None, p, 4, None, p, 1 << 30, None) == EINVAL
    assert lib.skh_hrdht_dense_colmajor(1, 100, 40, 9, 4, p, 100, None, p, 40, None, p, 1 << 30, None) == EINVAL
    assert lib.skh_hrdht_dense(1, 1 << 30, 70, 3, 4, p, 4, None, p, 4, None, p, 1 << 30, None) == EOVERFLOW
    assert lib.skh_srdht_dense(1, 100, 1 << 31, 4, p, 4, None, p, 4, None, p, 1 << 30, None) == EOVERFLOW
    # solve: m < d, missing outputs, ld rules
    info = (ctypes.c_int64 * 2)()
    stats = (ctypes.c_double * 3)()
    assert lib.skh_lls_solve(100, 10, p, 10, p, 9, p, 10, p, 1e-8, 1e-6, 10, p, None, info, stats, p, 1 << 30,
                             None) == EINVAL
    assert lib.skh_lls_solve(100, 10, p, 9, p, 20, p, 10, p, 1e-8, 1e-6, 10, p, None, info, stats, p, 1 << 30,
                             None) == EDIM
    assert lib.skh_lls_solve_colmajor(100, 10, p, 99, p, 20, p, 20, p, 1e-8, 1e-6, 10, p, None, info, stats, p,
                                      1 << 30, None) == EDIM
    assert lib.skh_lls_solve(100, 10, p, 10, p, 20, p, 10, p, 1e-8, -1.0, 10, p, None, info, stats, p, 1 << 30,
                             None) == EINVAL
    assert lib.skh_trace_set(None, -1) == EINVAL
    assert lib.skh_trace_set(None, 0) == 0 and lib.skh_trace_count() == 0


def test_binding_rejects_mis_sized_outputs():
    """The binding checks caller-given output buffers (the C ABI sees only a
    pointer and a leading dimension): a CPU tensor, a wrong dtype or a wrong
    shape raises before any library call."""
    import torch

    from paper_2105_11815_b200 import api
    with pytest.raises(ValueError, match="CUDA float64"):
        api._check_out(torch.zeros(4, 3, dtype=torch.float64), (4, 3), "SA")
    with pytest.raises(ValueError, match="CUDA float64"):
        api._check_out(torch.zeros(4, 3, dtype=torch.float32), (4, 3), "SA")


@pytest.mark.gpu
def test_binding_rejects_mis_sized_outputs_gpu():
    import torch

    from paper_2105_11815_b200 import api
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    A = torch.zeros(64, 8, dtype=torch.float64, device="cuda")
    bl = api.hash_gen(1, 16, 2, 64)
    with pytest.raises(ValueError, match="shape"):
        api.sketch_dense(bl, A, SA=torch.zeros(16, 7, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="out holds lists"):
        api.hash_gen(1, 16, 2, 65, out=bl)
    SA, _ = api.sketch_dense(bl, A, SA=torch.zeros(16, 8, dtype=torch.float64, device="cuda"))
    assert SA.shape == (16, 8)
