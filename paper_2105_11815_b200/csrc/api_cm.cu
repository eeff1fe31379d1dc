// api_cm.cu -- extern "C" entry points of the column-major path (include/skh.h
// "Column-major A"): validation, workspace layout and call sequencing for
// skh_rht_dense_colmajor[_host], skh_sketch_dense_colmajor and
// skh_rht_colmajor; plus the stage-trace hook (skh_trace_*).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace skh {

// cm.cu
int cm_max_buckets(int s);
int launch_cm_pass1(uint64_t seed, const double* X, int64_t ldx, int64_t ncolX, const double* xb, double* Y,
                    int64_t ldy, int64_t nvalid, int L, int apply_diag, int64_t row0, cudaStream_t st,
                    int reserve_sms = 0);
int launch_cm_mid(double* Y, int64_t ldy, int64_t ncols, int64_t nrows, int lo, int K2, cudaStream_t st);
size_t cm_lists_bytes(int64_t ntiles, int s, int64_t m);
int launch_cm_lists(const int32_t* col_rows, const int8_t* col_signs, int s, int64_t m, int K2, int lo,
                    int64_t nvalid, int64_t ntiles, void* lists_ws, cudaStream_t st);
int launch_cm_gather(const double* X, int64_t ldx, int64_t ncolX, const double* xb, int64_t nvalid, int64_t ntiles,
                     int lo, int K2, const void* lists_ws, int s, int64_t m, double* SA, int64_t ldsa,
                     int64_t ncolSA, double* Sb, double alpha, cudaStream_t st);

namespace {

constexpr int kCmP1 = 13;     // bits of pass 1
constexpr int kCmTile = 12;   // log2 positions of a pass-2 tile

// ---- stage trace (thread-local)
struct Trace {
  void* const* ev = nullptr;
  int n = 0;
  int used = 0;
  const char* names[64] = {};
};
thread_local Trace g_trace;

void trace_begin(cudaStream_t st) {
  g_trace.used = 0;
  if (g_trace.ev && g_trace.n > 0) {
    cudaEventRecord(reinterpret_cast<cudaEvent_t>(g_trace.ev[0]), st);
    g_trace.names[0] = "begin";
    g_trace.used = 1;
  }
}

int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}
int log2_of(int64_t p) {
  int k = 0;
  while (((int64_t)1 << k) < p) ++k;
  return k;
}

// Bits of the transform after pass 1: mid passes (<= 8 bits each, balanced) and
// the final fused pass K2 (<= 8).
struct CmPlan {
  int L, K1, nmid, mid[8], K2, lo2;
  int64_t ntiles;
};

CmPlan cm_plan(int64_t n_pad) {
  CmPlan p{};
  p.L = log2_of(n_pad);
  p.K1 = std::min(p.L, kCmP1);
  const int rest = p.L - p.K1;
  const int npass = (rest + 7) / 8;  // passes after pass 1 (the last one fused)
  int lo = p.K1;
  for (int i = 0; i + 1 < npass; ++i) {
    const int k = (rest - (lo - p.K1) + (npass - i) - 1) / (npass - i);
    p.mid[p.nmid++] = k;
    lo += k;
  }
  p.K2 = p.L - lo;
  p.lo2 = p.K2 > 0 ? lo : kCmTile;
  p.ntiles = p.K2 > 0 ? (n_pad >> kCmTile) : (n_pad + (1 << kCmTile) - 1) >> kCmTile;
  return p;
}

int validate(int64_t n, int64_t m, int32_t s, int64_t d, int64_t nrows_hash) {
  if (n < 1 || d < 1 || m < 1 || s < 1 || (int64_t)s > m || s > 8) {
    set_error("colmajor: need n >= 1, d >= 1, 1 <= s <= m, s <= 8 (n=%lld m=%lld s=%d d=%lld)", (long long)n,
              (long long)m, s, (long long)d);
    return SKH_EINVAL;
  }
  if (nrows_hash * (int64_t)s >= (1ll << 31)) {
    set_error("colmajor: n*s exceeds int32 indices");
    return SKH_EOVERFLOW;
  }
  return SKH_OK;
}

struct CmWs {
  double* Y;        // [ncols][n_pad] (rht only)
  double* SA;       // host variants: [d][m]
  double* Sb;
  int32_t* col_rows;
  int8_t* col_signs;
  int32_t* ptr;
  int32_t* rows;
  int8_t* signs;
  void* hws;
  void* lists;
  size_t total;
};

CmWs cm_layout(void* base, int64_t nrows_hash, int64_t ycols, int64_t yrows, int64_t m, int s, int64_t d,
               int64_t ntiles, bool host) {
  CmWs w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align_up(bytes);
    return q;
  };
  w.Y = (double*)take(sizeof(double) * (size_t)ycols * (size_t)yrows);
  w.SA = host ? (double*)take(sizeof(double) * (size_t)m * (size_t)d) : nullptr;
  w.Sb = host ? (double*)take(sizeof(double) * (size_t)m) : nullptr;
  w.col_rows = (int32_t*)take(sizeof(int32_t) * (size_t)nrows_hash * s);
  w.col_signs = (int8_t*)take((size_t)nrows_hash * s);
  w.ptr = (int32_t*)take(sizeof(int32_t) * (size_t)(m + 1));
  w.rows = (int32_t*)take(sizeof(int32_t) * (size_t)nrows_hash * s);
  w.signs = (int8_t*)take((size_t)nrows_hash * s);
  w.hws = take(hash_ws_bytes(nrows_hash, m, s));
  w.lists = take(cm_lists_bytes(ntiles, s, m));
  w.total = off;
  return w;
}

// Hash + tile lists (R1, R2 in tile order).  side: on the side stream (trace
// names "side:...", timed from the fork)
int cm_prepare(uint64_t seed, int64_t nrows_hash, int64_t m, int s, const CmPlan& pl, const CmWs& w,
               cudaStream_t st, bool side = false) {
  int rc = launch_hash(seed, m, s, nrows_hash, 0, 0, 0, w.col_rows, w.col_signs, w.ptr, w.rows, w.signs, w.hws,
                       hash_ws_bytes(nrows_hash, m, s), st);
  if (rc) return rc;
  skh_trace_mark(st, side ? "side:hash_gen" : "hash_gen");
  rc = launch_cm_lists(w.col_rows, w.col_signs, s, m, pl.K2, pl.lo2, nrows_hash, pl.ntiles, w.lists, st);
  if (rc) return rc;
  skh_trace_mark(st, side ? "side:tile_lists" : "tile_lists");
  return SKH_OK;
}

// SMs pass 1 leaves to the side stream's tile-list kernel (one CTA per tile,
// which cannot share an SM with a pass-1 CTA): only where the hash + lists are a
// sizeable share of pass 1, because pass 1 slows in proportion to the SMs it
// loses (measured, C2 / C3HD / C5 total ms: reserve 0: 0.545 / 3.840 / 44.59,
// 8: 0.442 / 3.858 / 45.80, 16: 0.450 / 3.931 / 47.16).  SKH_CM_RESERVE overrides.
int pass1_reserve(const CmPlan& pl, int64_t ncols) {
  static const int env = [] {
    const char* e = getenv("SKH_CM_RESERVE");
    return e ? atoi(e) : -1;
  }();
  if (env >= 0) return env;
  const int64_t chunks = ncols * (((int64_t)1 << pl.L) >> kCmP1);
  return chunks < 32768 ? (int)std::min<int64_t>(pl.ntiles, 8) : 0;
}

// Transform passes after pass 1 (mid passes) then the fused final pass.
int cm_rht_tail(const CmPlan& pl, int64_t n_pad, int64_t ncols, int64_t d, int64_t m, int s, const CmWs& w,
                double* SA, int64_t ldsa, double* Sb, cudaStream_t st, double alpha) {
  int lo = pl.K1;
  for (int i = 0; i < pl.nmid; ++i) {
    int rc = launch_cm_mid(w.Y, n_pad, ncols, n_pad, lo, pl.mid[i], st);
    if (rc) return rc;
    skh_trace_mark(st, "mid_pass");
    lo += pl.mid[i];
  }
  int rc = launch_cm_gather(w.Y, n_pad, ncols, nullptr, n_pad, pl.ntiles, pl.lo2, pl.K2, w.lists, s, m, SA, ldsa, d,
                            Sb, alpha, st);
  if (rc) return rc;
  skh_trace_mark(st, "pass2_gather");
  return SKH_OK;
}

// skh_fold_cols: T_r's column lists over the local rows (M3, include/skh.h)
__global__ void fold_cols_kernel(int64_t L, int64_t G, int s, int64_t rank, const int32_t* __restrict__ col_rows,
                                 const int8_t* __restrict__ col_signs, int32_t* __restrict__ fold_rows,
                                 int8_t* __restrict__ fold_signs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // destination entry
  const int64_t gs = G * s;
  if (t >= L * gs) return;
  const int64_t l = t / gs, g = (t % gs) / s, q = t % s;
  const int64_t src = (g * L + l) * s + q;
  fold_rows[t] = col_rows[src];
  const int neg = __popcll((unsigned long long)(g & rank)) & 1;
  fold_signs[t] = neg ? (int8_t)(-col_signs[src]) : col_signs[src];
}

}  // namespace

void skh_trace_mark(cudaStream_t st, const char* name) {
  if (g_trace.ev && g_trace.used < g_trace.n && g_trace.used < 64) {
    cudaEventRecord(reinterpret_cast<cudaEvent_t>(g_trace.ev[g_trace.used]), st);
    g_trace.names[g_trace.used++] = name;
  }
}
void skh_trace_start(cudaStream_t st) { trace_begin(st); }

}  // namespace skh

using namespace skh;

extern "C" {

int skh_trace_set(void* const* events, int nevents) {
  if (nevents < 0 || (nevents > 0 && !events)) {
    set_error("trace_set: invalid arguments");
    return SKH_EINVAL;
  }
  g_trace.ev = nevents > 0 ? events : nullptr;
  g_trace.n = std::min(nevents, 64);
  g_trace.used = 0;
  return SKH_OK;
}

int skh_trace_count(void) { return g_trace.used; }

const char* skh_trace_name(int i) { return (i >= 0 && i < g_trace.used) ? g_trace.names[i] : ""; }

size_t skh_rht_dense_colmajor_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d) {
  if (n < 1 || m < 1 || s < 1 || d < 1) return 0;
  const int64_t n_pad = next_pow2(n);
  const CmPlan pl = cm_plan(n_pad);
  return cm_layout(nullptr, n_pad, d + 1, n_pad, m, s, d, pl.ntiles, true).total;
}

static int rht_cm_check(int64_t n, int64_t m, int32_t s, int64_t d, int64_t lda, int64_t ldsa, bool has_b,
                        bool has_Sb) {
  const int64_t n_pad = next_pow2(n);
  int rc = validate(n, m, s, d, n_pad);
  if (rc) return rc;
  if (lda < n || ldsa < m || (has_b && !has_Sb)) {
    set_error("colmajor: need lda >= n, ldsa >= m, Sb when b is given");
    return SKH_EDIM;
  }
  return SKH_OK;
}

int skh_rht_dense_colmajor(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d, const double* A, int64_t lda,
                           const double* b, double* SA, int64_t ldsa, double* Sb, void* ws, size_t ws_bytes,
                           void* stream) {
  if (!A || !SA) {
    set_error("rht_dense_colmajor: A and SA required");
    return SKH_EINVAL;
  }
  int rc = rht_cm_check(n, m, s, d, lda, ldsa, b != nullptr, Sb != nullptr);
  if (rc) return rc;
  const int64_t n_pad = next_pow2(n);
  const CmPlan pl = cm_plan(n_pad);
  const int64_t ncols = d + (b ? 1 : 0);
  const CmWs w = cm_layout(ws, n_pad, d + 1, n_pad, m, s, d, pl.ntiles, true);
  if (!ws || ws_bytes < w.total) {
    set_error("rht_dense_colmajor workspace too small: need %zu bytes", w.total);
    return SKH_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  trace_begin(st);
  // hash + tile lists depend only on (seed, n, m, s): on the side stream, beside pass 1
  cudaStream_t ss = skh_side_fork(st);
  rc = cm_prepare(seed, n_pad, m, s, pl, w, ss, ss != st);
  if (!rc) rc = launch_cm_pass1(seed, A, lda, d, b, w.Y, n_pad, n, pl.L, 1, 0, st,
                                ss != st ? pass1_reserve(pl, ncols) : 0);
  if (!rc) skh_trace_mark(st, "pass1");
  const int jc = skh_side_join(st, ss);  // join on every path after the fork
  if (rc) return rc;
  if (jc) return jc;
  skh_trace_mark(st, "side_wait");
  return cm_rht_tail(pl, n_pad, ncols, d, m, s, w, SA, ldsa, Sb, st, skh_c_ns(n_pad, s));
}

int skh_rht_dense_colmajor_host(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d, const double* A_host,
                                int64_t lda, const double* b_host, double* SA_host, int64_t ldsa, double* Sb_host,
                                void* ws, size_t ws_bytes, void* stream) {
  if (!A_host || !SA_host) {
    set_error("rht_dense_colmajor_host: A_host and SA_host required");
    return SKH_EINVAL;
  }
  int rc = rht_cm_check(n, m, s, d, lda, ldsa, b_host != nullptr, Sb_host != nullptr);
  if (rc) return rc;
  const int64_t n_pad = next_pow2(n);
  const CmPlan pl = cm_plan(n_pad);
  const int64_t ncols = d + (b_host ? 1 : 0);
  const CmWs w = cm_layout(ws, n_pad, d + 1, n_pad, m, s, d, pl.ntiles, true);
  if (!ws || ws_bytes < w.total) {
    set_error("rht_dense_colmajor_host workspace too small: need %zu bytes", w.total);
    return SKH_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  cudaStream_t cs = skh_copy_stream();
  if (!cs) {
    set_error("rht_dense_colmajor_host: no copy stream");
    return SKH_ECUDA;
  }
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return check_launch("event");
  cudaEventRecord(ev, st);  // the copies must not overtake earlier users of the workspace
  cudaStreamWaitEvent(cs, ev, 0);
  trace_begin(st);
  rc = cm_prepare(seed, n_pad, m, s, pl, w, st);
  // H2D in groups of columns (~256 MiB), pass 1 in place on each group as it lands
  const int64_t grp = std::max<int64_t>(1, (int64_t)(256ll << 20) / (8 * n));
  for (int64_t c0 = 0; !rc && c0 < d; c0 += grp) {
    const int64_t nc = std::min(grp, d - c0);
    if (cudaMemcpy2DAsync(w.Y + c0 * n_pad, sizeof(double) * n_pad, A_host + c0 * lda, sizeof(double) * lda,
                          sizeof(double) * n, nc, cudaMemcpyHostToDevice, cs) != cudaSuccess) {
      rc = check_launch("H2D A");
      break;
    }
    cudaEventRecord(ev, cs);
    cudaStreamWaitEvent(st, ev, 0);
    rc = launch_cm_pass1(seed, w.Y + c0 * n_pad, n_pad, nc, nullptr, w.Y + c0 * n_pad, n_pad, n, pl.L, 1, 0, st);
  }
  if (!rc && b_host) {
    double* yb = w.Y + d * n_pad;
    if (cudaMemcpyAsync(yb, b_host, sizeof(double) * n, cudaMemcpyHostToDevice, st) != cudaSuccess)
      rc = check_launch("H2D b");
    if (!rc) rc = launch_cm_pass1(seed, yb, n_pad, 1, nullptr, yb, n_pad, n, pl.L, 1, 0, st);
  }
  if (!rc) skh_trace_mark(st, "h2d_pass1");
  if (!rc) rc = cm_rht_tail(pl, n_pad, ncols, d, m, s, w, w.SA, m, w.Sb, st, skh_c_ns(n_pad, s));
  if (!rc && cudaMemcpy2DAsync(SA_host, sizeof(double) * ldsa, w.SA, sizeof(double) * m, sizeof(double) * m, d,
                               cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = check_launch("D2H SA");
  if (!rc && b_host && cudaMemcpyAsync(Sb_host, w.Sb, sizeof(double) * m, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = check_launch("D2H Sb");
  cudaEventDestroy(ev);
  return rc;
}

// Transposed path of skh_sketch_dense_colmajor: bucket lists, A^T into a
// row-major copy, the row gather into a row-major SA, SA transposed out.
struct CmFastWs {
  int32_t* ptr;
  int32_t* rows;
  int8_t* signs;
  void* hws;
  double* Arm;  // [n x d] row-major copy of A
  double* SAt;  // [m x d] row-major SA
  size_t total;
};

CmFastWs cm_fast_layout(void* base, int64_t n, int64_t m, int s, int64_t d) {
  CmFastWs w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align_up(bytes);
    return q;
  };
  w.ptr = (int32_t*)take(sizeof(int32_t) * (size_t)(m + 1));
  w.rows = (int32_t*)take(sizeof(int32_t) * (size_t)n * s);
  w.signs = (int8_t*)take((size_t)n * s);
  w.hws = take(hash_ws_bytes(n, m, s));
  w.Arm = (double*)take(sizeof(double) * (size_t)n * (size_t)d);
  w.SAt = (double*)take(sizeof(double) * (size_t)m * (size_t)d);
  w.total = off;
  return w;
}

size_t skh_sketch_dense_colmajor_workspace_bytes(int64_t n, int64_t m, int32_t s) {
  if (n < 1 || m < 1 || s < 1) return 0;
  const CmPlan pl = cm_plan(n);  // K2 = 0 tiles for any n (only ntiles is used)
  const int64_t ntiles = (n + (1 << kCmTile) - 1) >> kCmTile;
  (void)pl;
  return cm_layout(nullptr, n, 0, 0, m, s, 1, ntiles, false).total;
}

size_t skh_sketch_dense_colmajor_fast_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d) {
  if (n < 1 || m < 1 || s < 1 || d < 1) return 0;
  return std::max(cm_fast_layout(nullptr, n, m, s, d).total, skh_sketch_dense_colmajor_workspace_bytes(n, m, s));
}

int skh_sketch_dense_colmajor(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d, const double* A,
                              int64_t lda, const double* b, double* SA, int64_t ldsa, double* Sb, void* ws,
                              size_t ws_bytes, void* stream) {
  int rc = validate(n, m, s, d, n);
  if (rc) return rc;
  if (!A || !SA) {
    set_error("sketch_dense_colmajor: A and SA required");
    return SKH_EINVAL;
  }
  if (lda < n || ldsa < m || (b && !Sb)) {
    set_error("sketch_dense_colmajor: need lda >= n, ldsa >= m, Sb when b is given");
    return SKH_EDIM;
  }
  if (ws && ws_bytes >= cm_fast_layout(nullptr, n, m, s, d).total) {
    // the workspace holds a row-major copy: transpose, row gather (bit-identical:
    // the same ascending-row sums), transpose SA back
    const CmFastWs f = cm_fast_layout(ws, n, m, s, d);
    cudaStream_t st = as_stream(stream);
    trace_begin(st);
    rc = launch_hash(seed, m, s, n, 0, 0, 0, nullptr, nullptr, f.ptr, f.rows, f.signs, f.hws, hash_ws_bytes(n, m, s),
                     st);
    if (rc) return rc;
    skh_trace_mark(st, "hash_gen");
    transpose_cm_to_rm(n, d, A, lda, f.Arm, d, st);
    if ((rc = check_launch("sketch_dense_colmajor: transpose"))) return rc;
    skh_trace_mark(st, "transpose");
    const double c = skh_c_s(s);
    if ((rc = launch_gather_dense(m, f.ptr, f.rows, f.signs, d, f.Arm, d, f.SAt, d, c, st, s))) return rc;
    if (b && (rc = launch_gather_vec(m, f.ptr, f.rows, f.signs, b, Sb, c, st))) return rc;
    transpose_cm_to_rm(d, m, f.SAt, d, SA, ldsa, st);
    if ((rc = check_launch("sketch_dense_colmajor: SA transpose"))) return rc;
    skh_trace_mark(st, "gather");
    return SKH_OK;
  }
  CmPlan pl{};
  pl.K2 = 0;
  pl.lo2 = kCmTile;
  pl.ntiles = (n + (1 << kCmTile) - 1) >> kCmTile;
  const CmWs w = cm_layout(ws, n, 0, 0, m, s, 1, pl.ntiles, false);
  if (!ws || ws_bytes < w.total) {
    set_error("sketch_dense_colmajor workspace too small: need %zu bytes", w.total);
    return SKH_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  trace_begin(st);
  rc = cm_prepare(seed, n, m, s, pl, w, st);
  if (rc) return rc;
  rc = launch_cm_gather(A, lda, d, b, n, pl.ntiles, pl.lo2, 0, w.lists, s, m, SA, ldsa, d, Sb, skh_c_s(s), st);
  if (rc) return rc;
  skh_trace_mark(st, "gather");
  return SKH_OK;
}

int skh_rht_colmajor(uint64_t seed, int64_t nrows, int64_t nvalid, int64_t row0, int64_t ncols, const double* X,
                     int64_t ldx, double* Y, int64_t ldy, int apply_diag, void* stream) {
  if (nrows < 1 || ncols < 0 || nvalid < 0 || nvalid > nrows || row0 < 0 || (ncols > 0 && (!X || !Y))) {
    set_error("rht_colmajor: invalid arguments");
    return SKH_EINVAL;
  }
  if (next_pow2(nrows) != nrows) {
    set_error("rht_colmajor: nrows = %lld is not a power of two", (long long)nrows);
    return SKH_ENOTPOW2;
  }
  if (ldx < nvalid || ldy < nrows || (X == Y && nvalid != nrows)) {
    set_error("rht_colmajor: need ldx >= nvalid, ldy >= nrows (and nvalid == nrows in place)");
    return SKH_EDIM;
  }
  if (ncols == 0) return SKH_OK;
  cudaStream_t st = as_stream(stream);
  const CmPlan pl = cm_plan(nrows);
  int rc = launch_cm_pass1(seed, X, ldx, ncols, nullptr, Y, ldy, nvalid, pl.L, apply_diag, row0, st);
  if (rc) return rc;
  int lo = pl.K1;
  for (int i = 0; i < pl.nmid; ++i) {
    rc = launch_cm_mid(Y, ldy, ncols, nrows, lo, pl.mid[i], st);
    if (rc) return rc;
    lo += pl.mid[i];
  }
  if (pl.K2 > 0) rc = launch_cm_mid(Y, ldy, ncols, nrows, lo, pl.K2, st);
  return rc;
}

int skh_fold_cols(int64_t L, int64_t G, int32_t s, int64_t rank, const int32_t* col_rows, const int8_t* col_signs,
                  int32_t* fold_rows, int8_t* fold_signs, void* stream) {
  if (L < 1 || G < 1 || s < 1 || rank < 0 || rank >= G || !col_rows || !col_signs || !fold_rows || !fold_signs) {
    set_error("fold_cols: invalid arguments");
    return SKH_EINVAL;
  }
  const int64_t N = L * G * (int64_t)s;
  fold_cols_kernel<<<(unsigned)((N + 255) / 256), 256, 0, as_stream(stream)>>>(L, G, s, rank, col_rows, col_signs,
                                                                               fold_rows, fold_signs);
  note_launch();
  return check_launch("fold_cols");
}

size_t skh_rht_colmajor_lists_workspace_bytes(int64_t L, int64_t m, int32_t s_eff, int64_t d) {
  if (L < 1 || m < 1 || s_eff < 1 || d < 1) return 0;
  const int64_t n_pad = next_pow2(L);
  const CmPlan pl = cm_plan(n_pad);
  return cm_layout(nullptr, n_pad, d + 1, n_pad, m, s_eff, d, pl.ntiles, false).total;
}

int skh_rht_colmajor_lists(uint64_t seed, int64_t L, int64_t row0, int64_t m, int32_t s_eff, int64_t d,
                           const double* A, int64_t lda, const double* b, const int32_t* col_rows,
                           const int8_t* col_signs, double alpha, double* SAt, int64_t ldsa, double* Sb, void* ws,
                           size_t ws_bytes, void* stream) {
  if (!A || !SAt || !col_rows || !col_signs || row0 < 0) {
    set_error("rht_colmajor_lists: A, SAt and the column lists required, row0 >= 0");
    return SKH_EINVAL;
  }
  const int64_t n_pad = next_pow2(std::max<int64_t>(L, 1));
  int rc = validate(L, m, s_eff, d, n_pad);
  if (rc) return rc;
  if (lda < L || ldsa < m || (b && !Sb)) {
    set_error("rht_colmajor_lists: need lda >= L, ldsa >= m, Sb when b is given");
    return SKH_EDIM;
  }
  const CmPlan pl = cm_plan(n_pad);
  const int64_t ncols = d + (b ? 1 : 0);
  const CmWs w = cm_layout(ws, n_pad, d + 1, n_pad, m, s_eff, d, pl.ntiles, false);
  if (!ws || ws_bytes < w.total) {
    set_error("rht_colmajor_lists workspace too small: need %zu bytes", w.total);
    return SKH_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  trace_begin(st);
  // the tile lists depend only on the given column lists: side stream, beside pass 1
  cudaStream_t ss = skh_side_fork(st);
  // the lists cover all n_pad rows of the padded transform (H mixes the zero padding in)
  rc = launch_cm_lists(col_rows, col_signs, s_eff, m, pl.K2, pl.lo2, n_pad, pl.ntiles, w.lists, ss);
  if (!rc) skh_trace_mark(ss, ss != st ? "side:tile_lists" : "tile_lists");
  if (!rc) rc = launch_cm_pass1(seed, A, lda, d, b, w.Y, n_pad, L, pl.L, 1, row0, st,
                                ss != st ? pass1_reserve(pl, ncols) : 0);
  if (!rc) skh_trace_mark(st, "pass1");
  const int jc = skh_side_join(st, ss);
  if (rc) return rc;
  if (jc) return jc;
  skh_trace_mark(st, "side_wait");
  return cm_rht_tail(pl, n_pad, ncols, d, m, s_eff, w, SAt, ldsa, Sb, st, alpha);
}

}  // extern "C"
