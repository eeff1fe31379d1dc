"""B200-native s-hashing sketch hot path of Ski-LLS (arXiv 2105.11815).

The product is libskh.so (CUDA kernels for sm_100a behind the C ABI in
include/skh.h); this package is its thin Python binding (``api``) plus the
multi-GPU sequencing (``sharded``).  See DESIGN.md.
"""
from .api import (BucketLists, RhtColMajorLists, RhtDense, RhtDenseColMajor, SketchDenseHost, Trace, c_n, c_ns, c_s,  # noqa: F401
                  fold_cols,
                  hash_gen, hash_status, hrdht_dense, hrdht_dense_colmajor, LlsSolver, lls_solve, ordered_sum, rht_colmajor, rht_dense, rht_dense_colmajor, rht_stages,
                  scale, ski_lls_dense, sketch_csr, sketch_dense, sketch_dense_colmajor, srdht_dense)
