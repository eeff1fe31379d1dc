// api.cu -- the extern "C" entry points declared in include/skh.h: argument
// validation, workspace layout, call sequencing, the host-buffer variants, and
// two small elementwise kernels (scale, ordered sum of partials).
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace skh {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SKH_ECUDA;
  }
  return SKH_OK;
}

// fwht.cu
std::vector<int> plan_passes(int L, bool fast);
bool fwht_fast_ok(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t d);
int launch_diag_words(uint64_t seed, int64_t nrows, int64_t nvalid, int64_t row0, int64_t d, void* ws,
                      cudaStream_t st);
int launch_fwht_pass_range(uint64_t seed, int K, bool fast, const double* X, int64_t ldx, double* Y, int64_t ldy,
                           int64_t nrows, int64_t nvalid, int lo, int64_t d, int64_t g_begin, int64_t g_count,
                           void* ws, int64_t row0, int apply_diag, double alpha, cudaStream_t st);

namespace {

__global__ void scale_kernel(double* X, int64_t rows, int64_t cols, int64_t ldx, double alpha) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i / cols, c = i % cols;
  X[r * ldx + c] = alpha * X[r * ldx + c];
}

// M3 fold (exchange-free sharded H D A): global column j of S
// -> local row j mod L, sign times (-1)^popcount((j / L) & rank)
__global__ void fold_lists_kernel(int64_t N, int32_t* __restrict__ rows, int8_t* __restrict__ signs, int64_t L,
                                  int64_t rank) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  const int64_t j = rows[e];
  rows[e] = (int32_t)(j % L);
  if (__popcll((unsigned long long)((j / L) & rank)) & 1) signs[e] = (int8_t)(-signs[e]);
}

__global__ void ordered_sum_kernel(const double* __restrict__ P, int64_t G, int64_t pstride, int64_t rows,
                                   int64_t cols, int64_t ldp, double* __restrict__ out, int64_t ldo, double alpha) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i / cols, c = i % cols;
  double a = P[r * ldp + c];
  for (int64_t g = 1; g < G; ++g) a = a + P[g * pstride + r * ldp + c];
  out[r * ldo + c] = alpha * a;
}

int log2_exact(int64_t n) {
  int k = 0;
  while (((int64_t)1 << k) < n) ++k;
  return ((int64_t)1 << k) == n ? k : -1;
}

int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Library-owned streams, one per calling THREAD and device, so calls from
// several threads on different streams never couple through a shared library
// stream (and a graph capture on one thread cannot pull in another thread's
// work).  Created on first use, never destroyed (a few per thread).
cudaStream_t thread_stream(int which) {
  thread_local cudaStream_t streams[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[dev][which] && cudaStreamCreateWithFlags(&streams[dev][which], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    streams[dev][which] = nullptr;
  }
  return streams[dev][which];
}

// Copy stream (host-buffer variants overlap H2D with compute).
cudaStream_t copy_stream() { return thread_stream(0); }

// Side stream for independent small work (Sb = S b beside S A): fork = the
// side stream waits for everything already on `st`; join = `st` waits for the
// side stream.  Streams and events are per thread and device.
cudaStream_t side_stream() { return thread_stream(1); }

cudaEvent_t side_event(int which) {
  thread_local cudaEvent_t ev[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!ev[dev][which]) cudaEventCreateWithFlags(&ev[dev][which], cudaEventDisableTiming);
  return ev[dev][which];
}

// returns the stream to launch the side work on (st itself if no side stream)
cudaStream_t side_fork(cudaStream_t st) {
  cudaStream_t side = side_stream();
  cudaEvent_t e = side_event(0);
  if (!side || !e || cudaEventRecord(e, st) != cudaSuccess || cudaStreamWaitEvent(side, e, 0) != cudaSuccess) {
    cudaGetLastError();
    return st;
  }
  return side;
}

int side_join(cudaStream_t st, cudaStream_t side) {
  if (side == st) return SKH_OK;
  cudaEvent_t e = side_event(1);
  if (!e || cudaEventRecord(e, side) != cudaSuccess || cudaStreamWaitEvent(st, e, 0) != cudaSuccess)
    return check_launch("side stream join");
  return SKH_OK;
}

int validate_hash_args(int64_t m, int32_t s, int64_t nrows) {
  if (m < 1 || s < 1 || (int64_t)s > m || s > 64 || nrows < 0) {
    set_error("invalid arguments: need 1 <= s <= m, s <= 64, nrows >= 0 (m=%lld s=%d nrows=%lld)", (long long)m, s,
              (long long)nrows);
    return SKH_EINVAL;
  }
  if (m >= (1ll << 31) || nrows * (int64_t)s >= (1ll << 31)) {
    set_error("m or nrows*s exceeds int32 indices");
    return SKH_EOVERFLOW;
  }
  return SKH_OK;
}

struct RhtWs {
  double* Y;
  double* yb;
  double* SA;   // host variants only
  double* Sb;
  double* bin;  // host variants only: b staged on device
  void* dw;  // transform workspace (counters + D bitmap)
  int32_t* ptr;
  int32_t* rows;
  int8_t* signs;
  void* hws;
  size_t total;
};

RhtWs rht_layout(void* base, int64_t n, int64_t n_pad, int64_t m, int s, int64_t d) {
  RhtWs w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align_up(bytes);
    return q;
  };
  w.Y = (double*)take(sizeof(double) * (size_t)n_pad * (size_t)d);
  w.yb = (double*)take(sizeof(double) * (size_t)n_pad);
  w.SA = (double*)take(sizeof(double) * (size_t)m * (size_t)d);
  w.Sb = (double*)take(sizeof(double) * (size_t)m);
  w.bin = (double*)take(sizeof(double) * (size_t)std::max<int64_t>(n, 1));
  w.dw = (void*)take(fwht_ws_bytes(n_pad, n, 0, d));
  w.ptr = (int32_t*)take(sizeof(int32_t) * (size_t)(m + 1));
  w.rows = (int32_t*)take(sizeof(int32_t) * (size_t)n_pad * s);
  w.signs = (int8_t*)take((size_t)n_pad * s);
  w.hws = take(hash_ws_bytes(n_pad, m, s));
  w.total = off;
  return w;
}

struct DenseWs {
  double* X;
  double* SA;
  double* Sb;
  double* bin;
  int32_t* ptr;
  int32_t* rows;
  int8_t* signs;
  void* hws;
  size_t total;
};

DenseWs dense_layout(void* base, int64_t n, int64_t m, int s, int64_t d) {
  DenseWs w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align_up(bytes);
    return q;
  };
  w.X = (double*)take(sizeof(double) * (size_t)n * (size_t)d);
  w.SA = (double*)take(sizeof(double) * (size_t)m * (size_t)d);
  w.Sb = (double*)take(sizeof(double) * (size_t)m);
  w.bin = (double*)take(sizeof(double) * (size_t)std::max<int64_t>(n, 1));
  w.ptr = (int32_t*)take(sizeof(int32_t) * (size_t)(m + 1));
  w.rows = (int32_t*)take(sizeof(int32_t) * (size_t)n * s);
  w.signs = (int8_t*)take((size_t)n * s);
  w.hws = take(hash_ws_bytes(n, m, s));
  w.total = off;
  return w;
}

// The device part of rht_dense after Y (first pass done or not) -- shared by both variants.
int rht_tail(uint64_t seed, int64_t n, int64_t n_pad, int L, int64_t m, int s, int64_t d, const RhtWs& w,
             int first_pass_done, int K0, bool fast, const double* b_dev, double* SA, int64_t ldsa, double* Sb,
             cudaStream_t st) {
  int rc;
  std::vector<int> ks = plan_passes(L, fast);
  int lo = 0;
  for (size_t p = 0; p < ks.size(); ++p) {
    const int K = ks[p];
    if (p == 0 && first_pass_done) {
      lo += K;
      continue;
    }
    rc = launch_fwht_pass_range(seed, K, fast && K >= 4, w.Y, d, w.Y, d, n_pad, n_pad, lo, d, 0, n_pad >> K, w.dw, 0, 0,
                                1.0, st);
    if (rc) return rc;
    lo += K;
  }
  (void)K0;
  const double c = skh_c_ns(n_pad, s);
  rc = launch_gather_dense(m, w.ptr, w.rows, w.signs, d, w.Y, d, SA, ldsa, c, st, s);
  if (rc) return rc;
  if (b_dev) {
    rc = launch_fwht(seed, n_pad, n, 0, 1, b_dev, 1, w.yb, 1, 0, L, 1, 1.0, w.dw, st);
    if (rc) return rc;
    rc = launch_gather_vec(m, w.ptr, w.rows, w.signs, w.yb, Sb, c, st);
    if (rc) return rc;
  }
  return SKH_OK;
}

}  // namespace

cudaStream_t skh_side_fork(cudaStream_t st) { return side_fork(st); }
int skh_side_join(cudaStream_t st, cudaStream_t side) { return side_join(st, side); }

cudaStream_t skh_copy_stream() { return copy_stream(); }

}  // namespace skh

using namespace skh;

extern "C" {

const char* skh_strerror(int code) {
  switch (code) {
    case SKH_OK: return "ok";
    case SKH_EINVAL: return "invalid argument";
    case SKH_ENOTPOW2: return "row count not a multiple of 2^bit_hi";
    case SKH_EDIM: return "dimension mismatch";
    case SKH_ERETRY: return "rejection attempts exhausted";
    case SKH_EOVERFLOW: return "size exceeds 32-bit index range";
    case SKH_EWORKSPACE: return "workspace missing or too small";
    case SKH_ECUDA: return "CUDA error";
    default: return "unknown error";
  }
}

const char* skh_last_error(void) { return g_err; }
int skh_abi_version(void) { return 1; }
uint64_t skh_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

double skh_c_s(int32_t s) { return 1.0 / sqrt((double)s); }
double skh_c_n(int64_t n_pad) { return 1.0 / sqrt((double)n_pad); }
double skh_c_ns(int64_t n_pad, int32_t s) { return 1.0 / sqrt((double)n_pad * (double)s); }

size_t skh_hash_workspace_bytes(int64_t nrows, int64_t m, int32_t s) {
  if (nrows < 0 || s < 1) return 0;
  return hash_ws_bytes(nrows, m, s);
}

static int hash_gen_impl(uint64_t seed, int64_t m, int32_t s, int64_t nrows, int64_t row0, int64_t blk,
                         int64_t stride, int32_t* col_rows, int8_t* col_signs, int32_t* bucket_ptr,
                         int32_t* bucket_rows, int8_t* bucket_signs, void* ws, size_t ws_bytes, int variant,
                         void* stream) {
  int rc = validate_hash_args(m, s, nrows);
  if (rc) return rc;
  if (!bucket_ptr || (nrows > 0 && (!bucket_rows || !bucket_signs))) {
    set_error("bucket_ptr/bucket_rows/bucket_signs must not be NULL");
    return SKH_EINVAL;
  }
  if (row0 < 0 || (blk > 0 && stride < blk)) {
    set_error("bad row map (row0=%lld blk=%lld stride=%lld)", (long long)row0, (long long)blk, (long long)stride);
    return SKH_EDIM;
  }
  if (nrows > 0 && row_map(nrows - 1, row0, blk, stride) >= (1ll << 47)) {
    set_error("global column id exceeds 2^47");
    return SKH_EOVERFLOW;
  }
  if (!ws || ws_bytes < hash_ws_bytes(nrows, m, s)) {
    set_error("hash workspace too small: need %zu bytes", hash_ws_bytes(nrows, m, s));
    return SKH_EWORKSPACE;
  }
  return launch_hash_v(seed, m, s, nrows, row0, blk, stride, col_rows, col_signs, bucket_ptr, bucket_rows,
                       bucket_signs, ws, ws_bytes, variant, as_stream(stream));
}

int skh_hash_gen(uint64_t seed, int64_t m, int32_t s, int64_t nrows, int64_t row0, int64_t blk, int64_t stride,
                 int32_t* col_rows, int8_t* col_signs, int32_t* bucket_ptr, int32_t* bucket_rows,
                 int8_t* bucket_signs, void* ws, size_t ws_bytes, void* stream) {
  return hash_gen_impl(seed, m, s, nrows, row0, blk, stride, col_rows, col_signs, bucket_ptr, bucket_rows,
                       bucket_signs, ws, ws_bytes, 0, stream);
}

int skh_hash_gen_variant(uint64_t seed, int64_t m, int32_t s, int64_t nrows, int64_t row0, int64_t blk,
                         int64_t stride, int32_t* col_rows, int8_t* col_signs, int32_t* bucket_ptr,
                         int32_t* bucket_rows, int8_t* bucket_signs, void* ws, size_t ws_bytes, void* stream) {
  return hash_gen_impl(seed, m, s, nrows, row0, blk, stride, col_rows, col_signs, bucket_ptr, bucket_rows,
                       bucket_signs, ws, ws_bytes, 1, stream);
}

int skh_hash_status(const void* ws, void* stream) {
  if (!ws) return SKH_EINVAL;
  return hash_status(ws, as_stream(stream));
}

int skh_sketch_dense(int64_t m, int32_t s, const int32_t* bucket_ptr, const int32_t* bucket_rows,
                     const int8_t* bucket_signs, int64_t nrows, int64_t d, const double* A, int64_t lda,
                     const double* b, double* SA, int64_t ldsa, double* Sb, double alpha, void* stream) {
  int rc = validate_hash_args(m, s, nrows);
  if (rc) return rc;
  if (d < 1 || !bucket_ptr || !SA || (nrows > 0 && (!A || !bucket_rows || !bucket_signs))) {
    set_error("sketch_dense: d >= 1 and non-NULL bucket lists, A, SA required");
    return SKH_EINVAL;
  }
  if (lda < d || ldsa < d || (b && !Sb)) {
    set_error("sketch_dense: lda/ldsa < d or Sb NULL with b given");
    return SKH_EDIM;
  }
  cudaStream_t st = as_stream(stream);
  // Sb (latency-bound, one warp per bucket) on the side stream beside S A
  cudaStream_t side = b ? side_fork(st) : st;
  if (b) rc = launch_gather_vec(m, bucket_ptr, bucket_rows, bucket_signs, b, Sb, alpha, side);
  if (!rc) rc = launch_gather_dense(m, bucket_ptr, bucket_rows, bucket_signs, d, A, lda, SA, ldsa, alpha, st, s);
  // join on every path after the fork: the caller's stream stays ordered after the side work
  const int jc = b ? side_join(st, side) : SKH_OK;
  return rc ? rc : jc;
}

size_t skh_sketch_csr_workspace_bytes(int64_t nrows, int32_t s, int64_t nnz) {
  if (nrows < 0 || s < 1 || nnz < 0) return 0;
  return csr_ws_bytes(nrows, s, nnz);
}

int skh_sketch_csr(int64_t m, int32_t s, const int32_t* bucket_ptr, const int32_t* bucket_rows,
                   const int8_t* bucket_signs, int64_t nrows, int64_t d, int64_t nnz, const int64_t* row_ptr,
                   const int32_t* col_idx, const double* val, const double* b, double* SA, int64_t ldsa, double* Sb,
                   double alpha, void* ws, size_t ws_bytes, void* stream) {
  int rc = validate_hash_args(m, s, nrows);
  if (rc) return rc;
  if (d < 1 || nnz < 0 || !bucket_ptr || !SA || (nrows > 0 && (!row_ptr || !bucket_rows || !bucket_signs)) ||
      (nnz > 0 && (!col_idx || !val))) {
    set_error("sketch_csr: d >= 1, nnz >= 0 and non-NULL bucket lists, row_ptr, col_idx, val, SA required");
    return SKH_EINVAL;
  }
  if (d >= (1ll << 31) || ldsa < d || (b && !Sb)) {
    set_error("sketch_csr: ldsa < d, d too large, or Sb NULL with b given");
    return SKH_EDIM;
  }
  if (nnz * (int64_t)s >= (1ll << 31)) {
    set_error("sketch_csr: s * nnz exceeds int32 offsets");
    return SKH_EOVERFLOW;
  }
  if (!ws || ws_bytes < csr_ws_bytes(nrows, s, nnz)) {
    set_error("sketch_csr workspace too small: need %zu bytes", csr_ws_bytes(nrows, s, nnz));
    return SKH_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  cudaStream_t side = b ? side_fork(st) : st;  // Sb beside the expand + reduce of S A
  if (b) rc = launch_gather_vec(m, bucket_ptr, bucket_rows, bucket_signs, b, Sb, alpha, side);
  if (!rc)
    rc = launch_gather_csr(m, s, bucket_ptr, bucket_rows, bucket_signs, nrows, d, nnz, row_ptr, col_idx, val, SA,
                           ldsa, alpha, ws, st);
  const int jc = b ? side_join(st, side) : SKH_OK;  // join on every path after the fork
  return rc ? rc : jc;
}

size_t skh_rht_stages_workspace_bytes(int64_t nrows, int64_t nvalid, int64_t row0, int64_t d) {
  if (nrows < 0 || nvalid < 0 || row0 < 0 || d < 1) return 0;
  return fwht_ws_bytes(nrows, nvalid, row0, d);
}

int skh_rht_pass_plan(int nbits, int64_t d, int aligned, int* bits_out, int max_out) {
  if (nbits < 0 || d < 1) return 0;
  const bool fast = aligned && d % 2 == 0 && d >= 16;
  std::vector<int> ks = plan_passes(nbits, fast);
  for (int i = 0; i < (int)ks.size() && i < max_out; ++i) bits_out[i] = ks[i];
  return (int)ks.size();
}

int skh_rht_stages(uint64_t seed, int64_t nrows, int64_t nvalid, int64_t row0, int64_t d, const double* X,
                   int64_t ldx, double* Y, int64_t ldy, int bit_lo, int bit_hi, int apply_diag, double alpha,
                   void* ws, size_t ws_bytes, void* stream) {
  if (nrows < 1 || d < 1 || !X || !Y || bit_lo < 0 || bit_hi < bit_lo || bit_hi > 62 || nvalid < 0 ||
      nvalid > nrows || row0 < 0) {
    set_error("rht_stages: invalid arguments");
    return SKH_EINVAL;
  }
  if (nrows % ((int64_t)1 << bit_hi) != 0) {
    set_error("rht_stages: nrows=%lld not a multiple of 2^%d", (long long)nrows, bit_hi);
    return SKH_ENOTPOW2;
  }
  if (ldx < d || ldy < d || (X == Y && nvalid != nrows)) {
    set_error("rht_stages: ldx/ldy < d, or in place with nvalid != nrows");
    return SKH_EDIM;
  }
  if (!ws || ws_bytes < fwht_ws_bytes(nrows, nvalid, row0, d)) {
    set_error("rht_stages workspace too small: need %zu bytes", fwht_ws_bytes(nrows, nvalid, row0, d));
    return SKH_EWORKSPACE;
  }
  return launch_fwht(seed, nrows, nvalid, row0, d, X, ldx, Y, ldy, bit_lo, bit_hi, apply_diag, alpha, ws,
                     as_stream(stream));
}

size_t skh_rht_dense_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d) {
  if (n < 1 || m < 1 || s < 1 || d < 1) return 0;
  return rht_layout(nullptr, n, next_pow2(n), m, s, d).total;
}

int skh_rht_dense(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d, const double* A, int64_t lda,
                  const double* b, double* SA, int64_t ldsa, double* Sb, void* ws, size_t ws_bytes, void* stream) {
  if (n < 1 || d < 1 || !A || !SA) {
    set_error("rht_dense: n >= 1, d >= 1, A and SA required");
    return SKH_EINVAL;
  }
  const int64_t n_pad = next_pow2(n);
  int rc = validate_hash_args(m, s, n_pad);
  if (rc) return rc;
  if (lda < d || ldsa < d || (b && !Sb)) {
    set_error("rht_dense: lda/ldsa < d or Sb NULL with b given");
    return SKH_EDIM;
  }
  RhtWs w = rht_layout(ws, n, n_pad, m, s, d);
  if (!ws || ws_bytes < w.total) {
    set_error("rht_dense workspace too small: need %zu bytes", w.total);
    return SKH_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  const int L = log2_exact(n_pad);
  rc = launch_hash(seed, m, s, n_pad, 0, 0, 0, nullptr, nullptr, w.ptr, w.rows, w.signs, w.hws,
                   hash_ws_bytes(n_pad, m, s), st);
  if (rc) return rc;
  rc = launch_fwht(seed, n_pad, n, 0, d, A, lda, w.Y, d, 0, L, 1, 1.0, w.dw, st);
  if (rc) return rc;
  const bool fast = fwht_fast_ok(w.Y, d, w.Y, d, d);
  // all passes done by launch_fwht: run only the gather part of the tail
  const double c = skh_c_ns(n_pad, s);
  rc = launch_gather_dense(m, w.ptr, w.rows, w.signs, d, w.Y, d, SA, ldsa, c, st, s);
  if (rc) return rc;
  (void)fast;
  if (b) {
    rc = launch_fwht(seed, n_pad, n, 0, 1, b, 1, w.yb, 1, 0, L, 1, 1.0, w.dw, st);
    if (rc) return rc;
    rc = launch_gather_vec(m, w.ptr, w.rows, w.signs, w.yb, Sb, c, st);
  }
  return rc;
}

int skh_rht_dense_host(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d, const double* A_host, int64_t lda,
                       const double* b_host, double* SA_host, int64_t ldsa, double* Sb_host, void* ws,
                       size_t ws_bytes, void* stream) {
  if (n < 1 || d < 1 || !A_host || !SA_host) {
    set_error("rht_dense_host: n >= 1, d >= 1, A_host and SA_host required");
    return SKH_EINVAL;
  }
  const int64_t n_pad = next_pow2(n);
  int rc = validate_hash_args(m, s, n_pad);
  if (rc) return rc;
  if (lda < d || ldsa < d || (b_host && !Sb_host)) {
    set_error("rht_dense_host: lda/ldsa < d or Sb_host NULL with b_host given");
    return SKH_EDIM;
  }
  RhtWs w = rht_layout(ws, n, n_pad, m, s, d);
  if (!ws || ws_bytes < w.total) {
    set_error("rht_dense_host workspace too small: need %zu bytes", w.total);
    return SKH_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  cudaStream_t cs = copy_stream();
  if (!cs) {
    set_error("rht_dense_host: no copy stream");
    return SKH_ECUDA;
  }
  const int L = log2_exact(n_pad);
  const bool fast = fwht_fast_ok(w.Y, d, w.Y, d, d);
  std::vector<int> ks = plan_passes(L, fast);
  const int K0 = ks[0];
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return check_launch("event");
  // copy stream must not overtake earlier work on st that may still use the workspace
  cudaEventRecord(ev, st);
  cudaStreamWaitEvent(cs, ev, 0);
  rc = launch_hash(seed, m, s, n_pad, 0, 0, 0, nullptr, nullptr, w.ptr, w.rows, w.signs, w.hws,
                   hash_ws_bytes(n_pad, m, s), st);
  if (!rc && !(fast && K0 >= 4)) rc = launch_diag_words(seed, n_pad, n, 0, d, w.dw, st);
  // chunked H2D into Y overlapped with the first pass (its groups are 2^K0 consecutive rows)
  const int64_t grp = (int64_t)1 << K0;
  int64_t chunk = std::max<int64_t>(grp, ((int64_t)(256ll << 20) / (8 * d)) / grp * grp);
  for (int64_t r0 = 0; !rc && r0 < n; r0 += chunk) {
    const int64_t nr = std::min(chunk, n - r0);
    if (cudaMemcpy2DAsync(w.Y + r0 * d, sizeof(double) * d, A_host + r0 * lda, sizeof(double) * lda,
                          sizeof(double) * d, nr, cudaMemcpyHostToDevice, cs) != cudaSuccess) {
      rc = check_launch("H2D A");
      break;
    }
    cudaEventRecord(ev, cs);
    cudaStreamWaitEvent(st, ev, 0);
    const int64_t g0 = r0 / grp, gc = (nr + grp - 1) / grp;
    rc = launch_fwht_pass_range(seed, K0, fast && K0 >= 4, w.Y, d, w.Y, d, n_pad, n, 0, d, g0, gc, w.dw, 0, 1, 1.0, st);
  }
  if (!rc && n < n_pad) {  // groups entirely in the zero padding
    const int64_t g0 = (n + grp - 1) / grp, gc = (n_pad >> K0) - g0;
    if (gc > 0)
      rc = launch_fwht_pass_range(seed, K0, fast && K0 >= 4, w.Y, d, w.Y, d, n_pad, n, 0, d, g0, gc, w.dw, 0, 1, 1.0, st);
  }
  if (!rc && b_host) {
    if (cudaMemcpyAsync(w.bin, b_host, sizeof(double) * n, cudaMemcpyHostToDevice, st) != cudaSuccess)
      rc = check_launch("H2D b");
  }
  if (!rc)
    rc = rht_tail(seed, n, n_pad, L, m, s, d, w, 1, K0, fast, b_host ? w.bin : nullptr, w.SA, d, w.Sb, st);
  if (!rc) {
    if (cudaMemcpy2DAsync(SA_host, sizeof(double) * ldsa, w.SA, sizeof(double) * d, sizeof(double) * d, m,
                          cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = check_launch("D2H SA");
    if (!rc && b_host &&
        cudaMemcpyAsync(Sb_host, w.Sb, sizeof(double) * m, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = check_launch("D2H Sb");
  }
  cudaEventDestroy(ev);
  return rc;
}

size_t skh_sketch_dense_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d) {
  if (n < 0 || m < 1 || s < 1 || d < 1) return 0;
  return dense_layout(nullptr, n, m, s, d).total;
}

int skh_sketch_dense_host(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d, const double* A_host,
                          int64_t lda, const double* b_host, double* SA_host, int64_t ldsa, double* Sb_host, void* ws,
                          size_t ws_bytes, void* stream) {
  int rc = validate_hash_args(m, s, n);
  if (rc) return rc;
  if (d < 1 || !SA_host || (n > 0 && !A_host)) {
    set_error("sketch_dense_host: d >= 1, A_host and SA_host required");
    return SKH_EINVAL;
  }
  if (lda < d || ldsa < d || (b_host && !Sb_host)) {
    set_error("sketch_dense_host: lda/ldsa < d or Sb_host NULL with b_host given");
    return SKH_EDIM;
  }
  DenseWs w = dense_layout(ws, n, m, s, d);
  if (!ws || ws_bytes < w.total) {
    set_error("sketch_dense_host workspace too small: need %zu bytes", w.total);
    return SKH_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  cudaStream_t cs = copy_stream();
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return check_launch("event");
  cudaEventRecord(ev, st);
  cudaStreamWaitEvent(cs, ev, 0);
  if (n > 0 &&
      cudaMemcpy2DAsync(w.X, sizeof(double) * d, A_host, sizeof(double) * lda, sizeof(double) * d, n,
                        cudaMemcpyHostToDevice, cs) != cudaSuccess)
    rc = check_launch("H2D A");
  if (!rc) rc = launch_hash(seed, m, s, n, 0, 0, 0, nullptr, nullptr, w.ptr, w.rows, w.signs, w.hws,
                            hash_ws_bytes(n, m, s), st);
  if (!rc && b_host && n > 0 &&
      cudaMemcpyAsync(w.bin, b_host, sizeof(double) * n, cudaMemcpyHostToDevice, st) != cudaSuccess)
    rc = check_launch("H2D b");
  cudaEventRecord(ev, cs);
  cudaStreamWaitEvent(st, ev, 0);
  const double c = skh_c_s(s);
  if (!rc) rc = launch_gather_dense(m, w.ptr, w.rows, w.signs, d, w.X, d, w.SA, d, c, st, s);
  if (!rc && b_host) rc = launch_gather_vec(m, w.ptr, w.rows, w.signs, w.bin, w.Sb, c, st);
  if (!rc && cudaMemcpy2DAsync(SA_host, sizeof(double) * ldsa, w.SA, sizeof(double) * d, sizeof(double) * d, m,
                               cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = check_launch("D2H SA");
  if (!rc && b_host && cudaMemcpyAsync(Sb_host, w.Sb, sizeof(double) * m, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = check_launch("D2H Sb");
  cudaEventDestroy(ev);
  return rc;
}

int skh_scale(double* X, int64_t rows, int64_t cols, int64_t ldx, double alpha, void* stream) {
  if (rows < 0 || cols < 0 || (rows * cols > 0 && !X) || (rows > 0 && ldx < cols)) {
    set_error("scale: invalid arguments");
    return SKH_EINVAL;
  }
  const int64_t N = rows * cols;
  if (N == 0) return SKH_OK;
  scale_kernel<<<(unsigned)((N + 255) / 256), 256, 0, as_stream(stream)>>>(X, rows, cols, ldx, alpha); note_launch();
  return check_launch("scale");
}

int skh_fold_lists(int64_t nentries, int32_t* bucket_rows, int8_t* bucket_signs, int64_t L, int64_t rank,
                   void* stream) {
  if (nentries < 0 || L < 1 || rank < 0 || (nentries > 0 && (!bucket_rows || !bucket_signs))) {
    set_error("fold_lists: invalid arguments");
    return SKH_EINVAL;
  }
  if (nentries == 0) return SKH_OK;
  fold_lists_kernel<<<(unsigned)((nentries + 255) / 256), 256, 0, as_stream(stream)>>>(nentries, bucket_rows,
                                                                                      bucket_signs, L, rank);
  note_launch();
  return check_launch("fold_lists");
}

int skh_ordered_sum(const double* parts, int64_t G, int64_t part_stride, int64_t rows, int64_t cols, int64_t ldp,
                    double* out, int64_t ldo, double alpha, void* stream) {
  if (G < 1 || rows < 0 || cols < 0 || (rows * cols > 0 && (!parts || !out)) || (rows > 0 && (ldp < cols || ldo < cols))) {
    set_error("ordered_sum: invalid arguments");
    return SKH_EINVAL;
  }
  const int64_t N = rows * cols;
  if (N == 0) return SKH_OK;
  ordered_sum_kernel<<<(unsigned)((N + 255) / 256), 256, 0, as_stream(stream)>>>(parts, G, part_stride, rows, cols,
                                                                                  ldp, out, ldo, alpha); note_launch();
  return check_launch("ordered_sum");
}

}  // extern "C"
