// fwht.cu -- R3 (D) and R4 (unnormalised Walsh-Hadamard butterflies) along the
// row index of a row-major n x d matrix (Def. def::HRHT, PAPER.md L790-801;
// DESIGN.md R7-R9).
//
// The transform over bits [bit_lo, bit_hi) is split into HBM passes of K <= 8
// bits.  A pass over bits [lo, lo+K) is a set of independent work items
// (group, column tile): the 2^K rows r = hi*2^(lo+K) + mid*2^lo + low
// (mid = 0..2^K-1) restricted to TC = 2^(13-K) columns, i.e. 64 KiB of fp64.
// Each item is loaded once (16-byte loads, 16 rows per thread), transformed in
// registers (mid bits 0..3), exchanged once through shared memory, transformed
// again (mid bits 4..K-1), scaled and stored once.  Stages run low bit to high
// bit everywhere, the oracle's order, so results are bit-identical to it.
// D is fused into the first pass (sign flip from a per-call bitmap of the
// splitmix64 words u(key_DIAG, g >> 6)); zero padding rows are never read.
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ bool diag_neg(const uint64_t* __restrict__ dw, int64_t w0, int64_t grow) {
  return (dw[(grow >> 6) - w0] >> (grow & 63)) & 1ull;
}

__global__ void diag_words_kernel(uint64_t key, int64_t w0, int64_t nw, uint64_t* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nw) out[q] = stream_u(key, (uint64_t)(w0 + q));
}

__device__ __forceinline__ double2 neg2(double2 a) { return make_double2(-a.x, -a.y); }
__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// Fast pass: K in [4, 8], TC = 2^(13-K) columns, 16-byte aligned X/Y, even ld, even d.
template <int K>
__global__ void __launch_bounds__(kThreads) fwht_fast_kernel(
    const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy, int64_t nvalid, int lo,
    int64_t d, int64_t ntc, int64_t g_begin, const uint64_t* __restrict__ dw, int64_t row0, int64_t w0,
    int apply_diag, double alpha) {
  constexpr int TC = 1 << (13 - K);
  constexpr int CP = TC / 2;
  constexpr int RS = kThreads / CP;  // = 2^(K-4)
  constexpr int NB = 16 / RS;        // bsel values per thread in phase 2
  extern __shared__ double2 tile[];  // [2^K][CP]
  const int cp = threadIdx.x % CP, rs = threadIdx.x / CP;
  const int64_t g = g_begin + blockIdx.x / ntc;
  const int64_t tc = blockIdx.x % ntc;
  const int64_t low = g & (((int64_t)1 << lo) - 1);
  const int64_t hi = g >> lo;
  const int64_t rbase = (hi << (lo + K)) + low;
  const int64_t c = tc * TC + 2 * cp;
  const bool cv = c < d;

  double2 v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int64_t r = rbase + ((int64_t)(rs * 16 + j) << lo);
    double2 x = make_double2(0.0, 0.0);
    if (cv && r < nvalid) {
      x = __ldg(reinterpret_cast<const double2*>(X + r * ldx + c));
      if (apply_diag && diag_neg(dw, w0, row0 + r)) x = neg2(x);
    }
    v[j] = x;
  }
#pragma unroll
  for (int bb = 0; bb < 4; ++bb) {
    const int h = 1 << bb;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (!(j & h)) {
        const double2 a = v[j], b = v[j + h];
        v[j] = add2(a, b);
        v[j + h] = sub2(a, b);
      }
    }
  }
  if (K == 4) {
    if (cv) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t r = rbase + ((int64_t)(rs * 16 + j) << lo);
        *reinterpret_cast<double2*>(Y + r * ldy + c) = make_double2(alpha * v[j].x, alpha * v[j].y);
      }
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) tile[(rs * 16 + j) * CP + cp] = v[j];
  __syncthreads();
  // phase 2: thread holds mid = a*16 + (rs*NB + t), a = 0..RS-1, t = 0..NB-1
#pragma unroll
  for (int t = 0; t < NB; ++t)
#pragma unroll
    for (int a = 0; a < RS; ++a) v[t * RS + a] = tile[(a * 16 + rs * NB + t) * CP + cp];
#pragma unroll
  for (int bb = 0; bb < K - 4; ++bb) {
    const int h = 1 << bb;
#pragma unroll
    for (int t = 0; t < NB; ++t)
#pragma unroll
      for (int a = 0; a < RS; ++a) {
        if (!(a & h)) {
          const double2 x = v[t * RS + a], y = v[t * RS + a + h];
          v[t * RS + a] = add2(x, y);
          v[t * RS + a + h] = sub2(x, y);
        }
      }
  }
  if (cv) {
#pragma unroll
    for (int t = 0; t < NB; ++t)
#pragma unroll
      for (int a = 0; a < RS; ++a) {
        const int mid = a * 16 + rs * NB + t;
        const int64_t r = rbase + ((int64_t)mid << lo);
        const double2 x = v[t * RS + a];
        *reinterpret_cast<double2*>(Y + r * ldy + c) = make_double2(alpha * x.x, alpha * x.y);
      }
  }
}

// Generic pass: any d, any alignment, K in [0, 6]; one thread per (group, column).
template <int K>
__global__ void __launch_bounds__(kThreads) fwht_generic_kernel(
    const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy, int64_t nvalid, int lo,
    int64_t d, int64_t g_begin, int64_t ngroups, const uint64_t* __restrict__ dw, int64_t row0, int64_t w0,
    int apply_diag, double alpha) {
  constexpr int R = 1 << K;
  const int64_t idx = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (idx >= ngroups * d) return;
  const int64_t c = idx % d;
  const int64_t g = g_begin + idx / d;
  const int64_t low = g & (((int64_t)1 << lo) - 1);
  const int64_t hi = g >> lo;
  const int64_t rbase = (hi << (lo + K)) + low;
  double v[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int64_t r = rbase + ((int64_t)j << lo);
    double x = 0.0;
    if (r < nvalid) {
      x = X[r * ldx + c];
      if (apply_diag && diag_neg(dw, w0, row0 + r)) x = -x;
    }
    v[j] = x;
  }
#pragma unroll
  for (int bb = 0; bb < K; ++bb) {
    const int h = 1 << bb;
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (!(j & h)) {
        const double a = v[j], b = v[j + h];
        v[j] = a + b;
        v[j + h] = a - b;
      }
  }
#pragma unroll
  for (int j = 0; j < R; ++j) Y[(rbase + ((int64_t)j << lo)) * ldy + c] = alpha * v[j];
}

template <int K>
int launch_fast(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nrows, int64_t nvalid, int lo,
                int64_t d, int64_t g_begin, int64_t g_count, const uint64_t* dw, int64_t row0, int64_t w0,
                int apply_diag, double alpha, cudaStream_t st) {
  constexpr int TC = 1 << (13 - K);
  const size_t smem = (size_t)(1 << K) * TC * sizeof(double);
  cudaFuncSetAttribute(fwht_fast_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntc = (d + TC - 1) / TC;
  (void)nrows;
  // chunk the grid so every launch has < 2^31 CTAs
  const int64_t max_groups = ((1ll << 31) - 1) / ntc;
  for (int64_t g0 = g_begin; g0 < g_begin + g_count; g0 += max_groups) {
    const int64_t gc = min(max_groups, g_begin + g_count - g0);
    fwht_fast_kernel<K><<<(unsigned)(gc * ntc), kThreads, smem, st>>>(X, ldx, Y, ldy, nvalid, lo, d, ntc, g0, dw,
                                                                      row0, w0, apply_diag, alpha); note_launch();
  }
  return check_launch("fwht_fast");
}

template <int K>
int launch_generic(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nvalid, int lo, int64_t d,
                   int64_t g_begin, int64_t g_count, const uint64_t* dw, int64_t row0, int64_t w0, int apply_diag,
                   double alpha, cudaStream_t st) {
  const int64_t per = ((1ll << 31) - 1) * (int64_t)kThreads / d;  // groups per launch (grid < 2^31)
  const int64_t step = per > 0 ? per : 1;
  for (int64_t g0 = g_begin; g0 < g_begin + g_count; g0 += step) {
    const int64_t gc = min(step, g_begin + g_count - g0);
    const int64_t threads = gc * d;
    fwht_generic_kernel<K><<<(unsigned)((threads + kThreads - 1) / kThreads), kThreads, 0, st>>>(
        X, ldx, Y, ldy, nvalid, lo, d, g0, gc, dw, row0, w0, apply_diag, alpha); note_launch();
  }
  return check_launch("fwht_generic");
}

int launch_pass(bool fast, int K, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nrows,
                int64_t nvalid, int lo, int64_t d, int64_t g_begin, int64_t g_count, const uint64_t* dw,
                int64_t row0, int64_t w0, int apply_diag, double alpha, cudaStream_t st) {
  if (fast) {
    switch (K) {
      case 4: return launch_fast<4>(X, ldx, Y, ldy, nrows, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
      case 5: return launch_fast<5>(X, ldx, Y, ldy, nrows, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
      case 6: return launch_fast<6>(X, ldx, Y, ldy, nrows, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
      case 7: return launch_fast<7>(X, ldx, Y, ldy, nrows, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
      case 8: return launch_fast<8>(X, ldx, Y, ldy, nrows, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
      default: break;
    }
  }
  switch (K) {
    case 0: return launch_generic<0>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
    case 1: return launch_generic<1>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
    case 2: return launch_generic<2>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
    case 3: return launch_generic<3>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
    case 4: return launch_generic<4>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
    case 5: return launch_generic<5>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
    case 6: return launch_generic<6>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st);
    default: break;
  }
  set_error("internal: bad pass width %d", K);
  return SKH_EINVAL;
}

}  // namespace

// Split L bits into passes: fast passes hold 4..8 bits, generic passes 0..6.
std::vector<int> plan_passes(int L, bool fast) {
  std::vector<int> ks;
  if (L <= 0) {
    ks.push_back(0);
    return ks;
  }
  const int kmax = fast ? 8 : 6;
  const int P = (L + kmax - 1) / kmax;
  for (int p = 0; p < P; ++p) ks.push_back(L / P + (p < L % P ? 1 : 0));
  return ks;
}

bool fwht_fast_ok(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t d) {
  return ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) % 16 == 0) && ldx % 2 == 0 &&
         ldy % 2 == 0 && d % 2 == 0 && d >= 16;
}

size_t fwht_ws_bytes(int64_t nvalid, int64_t row0) {
  if (nvalid <= 0) return 256;
  const int64_t w0 = row0 >> 6, w1 = (row0 + nvalid - 1) >> 6;
  return align_up(sizeof(uint64_t) * (size_t)(w1 - w0 + 1));
}

// Enqueue the diag bitmap for rows [row0, row0 + nvalid) into ws.
int launch_diag_words(uint64_t seed, int64_t nvalid, int64_t row0, void* ws, cudaStream_t st) {
  if (nvalid <= 0) return SKH_OK;
  const int64_t w0 = row0 >> 6, nw = ((row0 + nvalid - 1) >> 6) - w0 + 1;
  diag_words_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(key_diag(seed), w0, nw, (uint64_t*)ws); note_launch();
  return check_launch("diag_words");
}

// One pass restricted to groups [g_begin, g_begin + g_count) (for chunked host input).
int launch_fwht_pass_range(int K, bool fast, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nrows,
                           int64_t nvalid, int lo, int64_t d, int64_t g_begin, int64_t g_count, const void* dw,
                           int64_t row0, int apply_diag, double alpha, cudaStream_t st) {
  if (fast && (K < 4 || K > 8)) fast = false;
  return launch_pass(fast, K, X, ldx, Y, ldy, nrows, nvalid, lo, d, g_begin, g_count, (const uint64_t*)dw, row0,
                     row0 >> 6, apply_diag, alpha, st);
}

int launch_fwht(uint64_t seed, int64_t nrows, int64_t nvalid, int64_t row0, int64_t d, const double* X,
                int64_t ldx, double* Y, int64_t ldy, int bit_lo, int bit_hi, int apply_diag, double alpha,
                void* ws, cudaStream_t st) {
  const bool fast = fwht_fast_ok(X, ldx, Y, ldy, d);
  int rc;
  if (apply_diag) {
    rc = launch_diag_words(seed, nvalid, row0, ws, st);
    if (rc) return rc;
  }
  std::vector<int> ks = plan_passes(bit_hi - bit_lo, fast);
  int lo = bit_lo;
  for (size_t p = 0; p < ks.size(); ++p) {
    const int K = ks[p];
    const bool first = p == 0, last = p + 1 == ks.size();
    const bool f = fast && K >= 4;
    const int64_t ngroups = nrows >> K;
    rc = launch_pass(f, K, first ? X : Y, first ? ldx : ldy, Y, ldy, nrows, first ? nvalid : nrows, lo, d, 0,
                     ngroups, (const uint64_t*)ws, row0, row0 >> 6, first ? apply_diag : 0, last ? alpha : 1.0, st);
    if (rc) return rc;
    lo += K;
  }
  return SKH_OK;
}

}  // namespace skh
