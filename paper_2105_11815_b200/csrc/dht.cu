// dht.cu -- the HR-DHT sketch S = S_h F D (eq. eqn::HR-DHT, "(6.1)", PAPER.md
// L1066-1075): the sketch the paper's dense solver actually uses, with the
// normalised Discrete Hartley Transform F_ij = n^{-1/2} [cos + sin](2 pi ij / n)
// for ANY n (no padding, L1097).  SURVEY §8(f) NEXT-3.
//
//   1. hash the n rows (R1, R2: bucket lists, or tile lists for column-major);
//   2. Y = D [A | b], column-major (a tiled transpose for row-major A), D fused;
//   3. cuFFT D2Z on every column (a library FFT, like the paper's FFTW; its work
//      area comes from the caller's workspace: the library still never
//      allocates): X_k = sum_j y_j e^{-2 pi i jk/n}, k <= n/2;
//   4. Fhat y = Re X - Im X, with X_{n-k} = conj(X_k) for k > n/2
//      (cos t + sin t = Re e^{-it} - Im e^{-it}), written row-major (for the
//      row-major gather) or column-major (for the column-major tile gather);
//   5. SA = c S_h (Fhat D A), c = 1 / sqrt(n s) (R20).
#include <cuda_runtime.h>
#include <cufft.h>
#include <math.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>
#include <map>
#include <tuple>

#include "common.cuh"

namespace skh {

// cm.cu
size_t cm_lists_bytes(int64_t ntiles, int s, int64_t m);
int launch_cm_lists(const int32_t* col_rows, const int8_t* col_signs, int s, int64_t m, int K2, int lo,
                    int64_t nvalid, int64_t ntiles, void* lists_ws, cudaStream_t st);
int launch_cm_gather(const double* X, int64_t ldx, int64_t ncolX, const double* xb, int64_t nvalid, int64_t ntiles,
                     int lo, int K2, const void* lists_ws, int s, int64_t m, double* SA, int64_t ldsa,
                     int64_t ncolSA, double* Sb, double alpha, cudaStream_t st);

// fht.cu (n = 2^L, row-major: our own two-pass Hartley transform)
bool dht_pow2_supported(int64_t n);
size_t dht_pow2_z_elems(int64_t n, int64_t ncol);
int launch_dht_pow2(int64_t n, int64_t d, const double* A, int64_t lda, const double* b, uint64_t dkey,
                    double2* Z, double2* tw, double* H, int64_t ldh, double* hb, cudaStream_t st);

// Y[i * ldy + c] = X[c * ldx + i]: column-major n x d -> row-major, 64 x 64
// tiles, 16-byte accesses on both sides when X, Y and the strides are even
// (512 bytes per warp instruction), 2-way shared-memory conflicts at most.
namespace {
template <bool V2>
__global__ void __launch_bounds__(256) cm_to_rm_kernel(int64_t n, int64_t d, const double* __restrict__ X,
                                                       int64_t ldx, double* __restrict__ Y, int64_t ldy) {
  __shared__ double tile[64][65];  // [c][i]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * 64, c0 = (int64_t)blockIdx.y * 64;
  for (int k = w; k < 64; k += 8) {  // column c0 + k, rows i0 + 2 lane, + 1
    const int64_t c = c0 + k, i = i0 + 2 * lane;
    double2 v = make_double2(0.0, 0.0);
    if (c < d) {
      if (V2 && i + 1 < n) {
        v = __ldg(reinterpret_cast<const double2*>(X + c * ldx + i));
      } else {
        if (i < n) v.x = X[c * ldx + i];
        if (i + 1 < n) v.y = X[c * ldx + i + 1];
      }
    }
    tile[k][2 * lane] = v.x;
    tile[k][2 * lane + 1] = v.y;
  }
  __syncthreads();
  for (int k = w; k < 64; k += 8) {  // row i0 + k, columns c0 + 2 lane, + 1
    const int64_t i = i0 + k, c = c0 + 2 * lane;
    if (i >= n) continue;
    const double2 v = make_double2(tile[2 * lane][k], tile[2 * lane + 1][k]);
    if (V2 && c + 1 < d) {
      *reinterpret_cast<double2*>(Y + i * ldy + c) = v;
    } else {
      if (c < d) Y[i * ldy + c] = v.x;
      if (c + 1 < d) Y[i * ldy + c + 1] = v.y;
    }
  }
}

}  // namespace

void transpose_cm_to_rm(int64_t n, int64_t d, const double* X, int64_t ldx, double* Y, int64_t ldy, cudaStream_t st) {
  const bool v2 = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) % 16 == 0) && ldx % 2 == 0 &&
                  ldy % 2 == 0;
  dim3 g((unsigned)((n + 63) / 64), (unsigned)((d + 63) / 64));
  if (v2) cm_to_rm_kernel<true><<<g, 256, 0, st>>>(n, d, X, ldx, Y, ldy);
  else cm_to_rm_kernel<false><<<g, 256, 0, st>>>(n, d, X, ldx, Y, ldy);
  note_launch();
}

namespace {

// n = 2^L (4 <= n <= 2^18) takes the fht.cu passes -- column-major A through a
// tiled transpose first -- unless SKH_DHT_CUFFT=1 (kept for comparison: D +
// layout change, cuFFT D2Z, Hartley combine).
bool use_pow2(int64_t n, bool rowmajor) {
  static const bool force_cufft = [] {
    const char* e = getenv("SKH_DHT_CUFFT");
    return e && e[0] == '1';
  }();
  return !force_cufft && dht_pow2_supported(n);
}

__device__ __forceinline__ double dsign(uint64_t dkey, int64_t g) {
  return ((stream_u(dkey, (uint64_t)(g >> 6)) >> (g & 63)) & 1ull) ? -1.0 : 1.0;
}

// Y[c * n + i] = D_i A[i, c] (row-major A, lda) for c < d; Y[d * n + i] = D_i b[i]
__global__ void diag_transpose_kernel(int64_t n, int64_t d, const double* __restrict__ A, int64_t lda,
                                      double* __restrict__ Y, uint64_t dkey) {
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < n && c < d) ? A[r * lda + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < n && c < d) Y[c * n + r] = dsign(dkey, r) * tile[threadIdx.x][k];
  }
}

// Y[c * n + i] = D_i X[c * ldx + i] (column-major X) for c < ncol
__global__ void diag_copy_cm_kernel(int64_t n, int64_t ncol, const double* __restrict__ X, int64_t ldx,
                                    double* __restrict__ Y, uint64_t dkey) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * ncol) return;
  const int64_t c = e / n, i = e % n;
  Y[c * n + i] = dsign(dkey, i) * X[c * ldx + i];
}

__device__ __forceinline__ double hartley_at(const cufftDoubleComplex* __restrict__ Z, int64_t nh, int64_t n,
                                             int64_t c, int64_t i) {
  const int64_t k = i <= n / 2 ? i : n - i;
  const cufftDoubleComplex z = Z[c * nh + k];
  return i <= n / 2 ? z.x - z.y : z.x + z.y;
}

// column-major H[c * n + i]
__global__ void hartley_cm_kernel(int64_t n, int64_t ncol, const cufftDoubleComplex* __restrict__ Z,
                                  double* __restrict__ H) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * ncol) return;
  const int64_t c = e / n, i = e % n;
  H[c * n + i] = hartley_at(Z, n / 2 + 1, n, c, i);
}

// row-major H[i * d + c] for c < d (tiled transpose); hb[i] for column d
__global__ void hartley_rm_kernel(int64_t n, int64_t d, const cufftDoubleComplex* __restrict__ Z,
                                  double* __restrict__ H, double* __restrict__ hb) {
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  const int64_t nh = n / 2 + 1;
  const int64_t ncol = d + (hb ? 1 : 0);
  for (int k = threadIdx.y; k < 32; k += 8) {  // read along i (coalesced in Z)
    const int64_t c = c0 + k, i = r0 + threadIdx.x;
    tile[k][threadIdx.x] = (i < n && c < ncol) ? hartley_at(Z, nh, n, c, i) : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {  // write along c
    const int64_t i = r0 + k, c = c0 + threadIdx.x;
    if (i < n && c < ncol) {
      const double v = tile[threadIdx.x][k];
      if (c < d) H[i * d + c] = v;
      else hb[i] = v;
    }
  }
}

// SR-DHT (eq. (7.2)): SA[r, :] = alpha * H[j_r, :], Sb[r] = alpha * hb[j_r],
// j_r = floor(u(mix64(seed ^ "SAMP"), r) * n / 2^64) (R21)
__global__ void sample_rows_kernel(int64_t m, int64_t n, int64_t d, uint64_t skey, const double* __restrict__ H,
                                   const double* __restrict__ hb, double* __restrict__ SA, int64_t ldsa,
                                   double* __restrict__ Sb, double alpha) {
  const int64_t r = blockIdx.x;
  const int64_t j = (int64_t)__umul64hi(stream_u(skey, (uint64_t)r), (uint64_t)n);
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) SA[r * ldsa + c] = alpha * H[j * d + c];
  if (Sb && threadIdx.x == 0) Sb[r] = alpha * hb[j];
}

// ---------------------------------------------------------------- cuFFT plans (per thread, device, n, batch)
struct Plan {
  cufftHandle h = 0;
  size_t work = 0;
};
thread_local std::map<std::tuple<int, int64_t, int64_t>, Plan> g_plans;

int get_plan(int64_t n, int64_t ncol, Plan** out) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto key = std::make_tuple(dev, n, ncol);
  auto it = g_plans.find(key);
  if (it == g_plans.end()) {
    Plan p;
    if (cufftCreate(&p.h) != CUFFT_SUCCESS) {
      set_error("hrdht: cufftCreate failed");
      return SKH_ECUDA;
    }
    cufftSetAutoAllocation(p.h, 0);
    long long nn[1] = {(long long)n};
    long long inem[1] = {(long long)n}, onem[1] = {(long long)(n / 2 + 1)};
    if (cufftMakePlanMany64(p.h, 1, nn, inem, 1, n, onem, 1, n / 2 + 1, CUFFT_D2Z, ncol, &p.work) != CUFFT_SUCCESS) {
      cufftDestroy(p.h);
      set_error("hrdht: cufftMakePlanMany64 failed (n=%lld, batch=%lld)", (long long)n, (long long)ncol);
      return SKH_ECUDA;
    }
    it = g_plans.emplace(key, p).first;
  }
  *out = &it->second;
  return SKH_OK;
}

struct DhtWs {
  double* Y;                 // [ncol][n] D A, then Fhat D A (column-major)
  cufftDoubleComplex* Z;     // [ncol][n/2 + 1] (cuFFT) or fht.cu's four-step buffer
  cufftDoubleComplex* tw;    // fht.cu: W_n^e, e <= n/2
  double* H;                 // row-major Fhat D A [n][d] (row-major path)
  double* hb;                // Fhat D b [n] (row-major path)
  double* SAt;               // column-major power-of-two path: row-major SA before the transpose
  void* fftwork;
  int32_t* col_rows;
  int8_t* col_signs;
  int32_t* ptr;
  int32_t* rows;
  int8_t* signs;
  void* hws;
  void* lists;
  size_t total;
};

DhtWs dht_layout(void* base, int64_t n, int64_t m, int s, int64_t d, bool rowmajor, size_t fftwork) {
  DhtWs w{};
  const bool pow2 = use_pow2(n, rowmajor);
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align_up(bytes);
    return q;
  };
  const int64_t ncol = d + 1;
  if (pow2) {  // column-major input is transposed into H first (row-major kernels, §5d)
    w.Z = (cufftDoubleComplex*)take(sizeof(cufftDoubleComplex) * dht_pow2_z_elems(n, ncol));
    w.tw = (cufftDoubleComplex*)take(sizeof(cufftDoubleComplex) * (size_t)(n / 2 + 1));
    if (!rowmajor) {
      w.H = (double*)take(sizeof(double) * (size_t)n * d);
      w.hb = (double*)take(sizeof(double) * (size_t)n);
      w.SAt = (double*)take(sizeof(double) * (size_t)m * d);
    }
  } else {
    w.Y = (double*)take(sizeof(double) * (size_t)n * ncol);
    w.Z = (cufftDoubleComplex*)take(sizeof(cufftDoubleComplex) * (size_t)(n / 2 + 1) * ncol);
  }
  if (rowmajor) {
    w.H = (double*)take(sizeof(double) * (size_t)n * d);
    w.hb = (double*)take(sizeof(double) * (size_t)n);
  }
  if (!pow2) w.fftwork = take(std::max<size_t>(fftwork, 16));
  w.col_rows = (int32_t*)take(sizeof(int32_t) * (size_t)n * s);
  w.col_signs = (int8_t*)take((size_t)n * s);
  w.ptr = (int32_t*)take(sizeof(int32_t) * (size_t)(m + 1));
  w.rows = (int32_t*)take(sizeof(int32_t) * (size_t)n * s);
  w.signs = (int8_t*)take((size_t)n * s);
  w.hws = take(hash_ws_bytes(n, m, s));
  if (!rowmajor && !pow2) w.lists = take(cm_lists_bytes((n + 4095) / 4096, s, m));
  w.total = off;
  return w;
}

int check_args(int64_t n, int64_t m, int32_t s, int64_t d, bool rowmajor) {
  if (n < 1 || d < 1 || m < 1 || s < 1 || (int64_t)s > m || s > (rowmajor ? 64 : 8)) {
    set_error("hrdht: need n, d >= 1, 1 <= s <= m, s <= %d", rowmajor ? 64 : 8);
    return SKH_EINVAL;
  }
  if (!rowmajor && m > 65536) {
    set_error("hrdht_colmajor: m > 65536");
    return SKH_EINVAL;
  }
  if (n * (int64_t)s >= (1ll << 31) || m >= (1ll << 31)) {
    set_error("hrdht: n*s or m exceeds int32 indices");
    return SKH_EOVERFLOW;
  }
  return SKH_OK;
}

size_t ws_bytes_for(int64_t n, int64_t m, int32_t s, int64_t d, bool rowmajor) {
  if (check_args(n, m, s, d, rowmajor)) return 0;
  if (use_pow2(n, rowmajor)) return dht_layout(nullptr, n, m, s, d, rowmajor, 0).total;
  Plan* p = nullptr;
  if (get_plan(n, d + 1, &p)) return 0;
  return dht_layout(nullptr, n, m, s, d, rowmajor, p->work).total;
}

// row-major H = Fhat D A, hb = Fhat D b in the workspace: S_h (or S_s) applied
int finish_rowmajor(uint64_t seed, int64_t n, int64_t m, int64_t d, const DhtWs& w, const double* b, double* SA,
                    int64_t ldsa, double* Sb, double c, bool sample, cudaStream_t st) {
  int rc;
  if (sample) {
    sample_rows_kernel<<<(unsigned)m, 256, 0, st>>>(m, n, d, mix64(seed ^ 0x53414D50ull), w.H, w.hb, SA, ldsa,
                                                    b ? Sb : nullptr, 1.0 / sqrt((double)n));
    note_launch();
    if ((rc = check_launch("srdht: sample"))) return rc;
  } else {
    if ((rc = launch_gather_dense(m, w.ptr, w.rows, w.signs, d, w.H, d, SA, ldsa, c, st))) return rc;
    if (b && (rc = launch_gather_vec(m, w.ptr, w.rows, w.signs, w.hb, Sb, c, st))) return rc;
  }
  skh_trace_mark(st, "gather");
  return SKH_OK;
}

int hrdht_run(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d, const double* A, int64_t lda,
              const double* b, double* SA, int64_t ldsa, double* Sb, void* ws, size_t ws_bytes, bool rowmajor,
              cudaStream_t st, bool sample = false) {
  int rc = check_args(n, m, s, d, rowmajor);
  if (rc) return rc;
  if (!A || !SA) {
    set_error("hrdht: A and SA required");
    return SKH_EINVAL;
  }
  if ((rowmajor && (lda < d || ldsa < d)) || (!rowmajor && (lda < n || ldsa < m)) || (b && !Sb)) {
    set_error("hrdht: bad leading dimension or Sb missing");
    return SKH_EDIM;
  }
  const int64_t ncol = d + (b ? 1 : 0);
  const bool pow2 = use_pow2(n, rowmajor);
  Plan* plan = nullptr;
  Plan* pmax = nullptr;
  if (!pow2) {
    if ((rc = get_plan(n, ncol, &plan))) return rc;
    // the workspace query sizes the FFT for d + 1 columns, the largest plan
    if ((rc = get_plan(n, d + 1, &pmax))) return rc;
  }
  const DhtWs w = dht_layout(ws, n, m, s, d, rowmajor, pow2 ? 0 : std::max(plan->work, pmax->work));
  if (!ws || ws_bytes < w.total) {
    set_error("hrdht workspace too small: need %zu bytes", w.total);
    return SKH_EWORKSPACE;
  }
  skh_trace_start(st);
  if (!sample) {
    rc = launch_hash(seed, m, s, n, 0, 0, 0, w.col_rows, w.col_signs, w.ptr, w.rows, w.signs, w.hws,
                     hash_ws_bytes(n, m, s), st);
    if (rc) return rc;
  }
  if (!rowmajor && !pow2 &&
      (rc = launch_cm_lists(w.col_rows, w.col_signs, s, m, 0, 12, n, (n + 4095) / 4096, w.lists, st)))
    return rc;
  skh_trace_mark(st, "hash_gen");
  const uint64_t dkey = key_diag(seed);
  const double c = 1.0 / sqrt((double)n * (double)s);
  if (pow2 && rowmajor) {
    if ((rc = launch_dht_pow2(n, d, A, lda, b, dkey, (double2*)w.Z, (double2*)w.tw, w.H, d, w.hb, st))) return rc;
    return finish_rowmajor(seed, n, m, d, w, b, SA, ldsa, Sb, c, sample, st);
  }
  if (pow2) {  // column-major, n = 2^L: transpose A into H, the row-major passes (H in place), gather, transpose SA
    transpose_cm_to_rm(n, d, A, lda, w.H, d, st);
    if ((rc = check_launch("hrdht: transpose"))) return rc;
    skh_trace_mark(st, "transpose");
    if ((rc = launch_dht_pow2(n, d, w.H, d, b, dkey, (double2*)w.Z, (double2*)w.tw, w.H, d, w.hb, st))) return rc;
    if ((rc = launch_gather_dense(m, w.ptr, w.rows, w.signs, d, w.H, d, w.SAt, d, c, st, s))) return rc;
    if (b && (rc = launch_gather_vec(m, w.ptr, w.rows, w.signs, w.hb, Sb, c, st))) return rc;
    transpose_cm_to_rm(d, m, w.SAt, d, SA, ldsa, st);  // SA[c * ldsa + b] = SAt[b * d + c]
    if ((rc = check_launch("hrdht: SA transpose"))) return rc;
    skh_trace_mark(st, "gather");
    return SKH_OK;
  }
  if (rowmajor) {
    dim3 grid((unsigned)((d + 31) / 32), (unsigned)((n + 31) / 32));
    diag_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(n, d, A, lda, w.Y, dkey);
    note_launch();
  } else {
    diag_copy_cm_kernel<<<(unsigned)((n * d + 255) / 256), 256, 0, st>>>(n, d, A, lda, w.Y, dkey);
    note_launch();
  }
  if (b) {
    diag_copy_cm_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, 1, b, n, w.Y + d * n, dkey);
    note_launch();
  }
  if ((rc = check_launch("hrdht: D"))) return rc;
  skh_trace_mark(st, "diag");
  cufftSetStream(plan->h, st);
  cufftSetWorkArea(plan->h, w.fftwork);
  if (cufftExecD2Z(plan->h, w.Y, w.Z) != CUFFT_SUCCESS) {
    set_error("hrdht: cufftExecD2Z failed");
    return SKH_ECUDA;
  }
  skh_trace_mark(st, "fft");
  if (rowmajor) {
    dim3 grid((unsigned)((ncol + 31) / 32), (unsigned)((n + 31) / 32));
    hartley_rm_kernel<<<grid, dim3(32, 8), 0, st>>>(n, d, w.Z, w.H, b ? w.hb : nullptr);
    note_launch();
    if ((rc = check_launch("hrdht: hartley"))) return rc;
    skh_trace_mark(st, "hartley");
    return finish_rowmajor(seed, n, m, d, w, b, SA, ldsa, Sb, c, sample, st);
  } else {
    hartley_cm_kernel<<<(unsigned)((n * ncol + 255) / 256), 256, 0, st>>>(n, ncol, w.Z, w.Y);
    note_launch();
    if ((rc = check_launch("hrdht: hartley"))) return rc;
    skh_trace_mark(st, "hartley");
    if ((rc = launch_cm_gather(w.Y, n, ncol, nullptr, n, (n + 4095) / 4096, 12, 0, w.lists, s, m, SA, ldsa, d, Sb, c,
                               st)))
      return rc;
  }
  skh_trace_mark(st, "gather");
  return SKH_OK;
}

}  // namespace
}  // namespace skh

using namespace skh;

extern "C" {

size_t skh_hrdht_dense_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d) {
  return ws_bytes_for(n, m, s, d, true);
}

int skh_hrdht_dense(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d, const double* A, int64_t lda,
                    const double* b, double* SA, int64_t ldsa, double* Sb, void* ws, size_t ws_bytes, void* stream) {
  return hrdht_run(seed, n, m, s, d, A, lda, b, SA, ldsa, Sb, ws, ws_bytes, true, as_stream(stream));
}

size_t skh_hrdht_dense_colmajor_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d) {
  return ws_bytes_for(n, m, s, d, false);
}

int skh_hrdht_dense_colmajor(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d, const double* A,
                             int64_t lda, const double* b, double* SA, int64_t ldsa, double* Sb, void* ws,
                             size_t ws_bytes, void* stream) {
  return hrdht_run(seed, n, m, s, d, A, lda, b, SA, ldsa, Sb, ws, ws_bytes, false, as_stream(stream));
}

size_t skh_srdht_dense_workspace_bytes(int64_t n, int64_t m, int64_t d) {
  return ws_bytes_for(n, m < 1 ? 1 : m, 1, d, true);
}

int skh_srdht_dense(uint64_t seed, int64_t n, int64_t m, int64_t d, const double* A, int64_t lda, const double* b,
                    double* SA, int64_t ldsa, double* Sb, void* ws, size_t ws_bytes, void* stream) {
  if (m >= (1ll << 31)) {
    set_error("srdht: m too large");
    return SKH_EOVERFLOW;
  }
  return hrdht_run(seed, n, m, 1, d, A, lda, b, SA, ldsa, Sb, ws, ws_bytes, true, as_stream(stream), true);
}

}  // extern "C"
