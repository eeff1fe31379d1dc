// fwht.cu -- R3 (D) and R4 (unnormalised Walsh-Hadamard butterflies) along the
// row index of a row-major n x d matrix (Def. def::HRHT, PAPER.md L790-801;
// DESIGN.md R7-R9).
//
// The transform over bits [bit_lo, bit_hi) is split into HBM passes of K bits.
// A pass over bits [lo, lo+K) is a set of independent tiles (group, column
// tile): the 2^K rows r = hi*2^(lo+K) + mid*2^lo + low (mid = 0..2^K-1)
// restricted to TC columns.  A tile is loaded once with 16-byte loads (16 rows x
// one column pair per thread, so 16 loads in flight per thread), transformed in
// registers 4 bits at a time, re-distributed through shared memory between
// 4-bit phases, scaled and stored once: every element crosses HBM exactly twice
// per pass.  Stages run low bit to high bit everywhere -- the oracle's order --
// so results are bit-identical to it.  D is fused into the first pass as a sign
// flip; its bits come from a per-call bitmap of the splitmix64 words
// u(key_DIAG, g >> 6), loaded before the data so the 16 data loads stay in
// flight together.  Zero padding rows are never read.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kGenThreads = 256;


__global__ void diag_words_kernel(uint64_t key, int64_t w0, int64_t nw, uint64_t* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nw) out[q] = stream_u(key, (uint64_t)(w0 + q));
}

__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// mid index of value v (0..15) of row-slot rs in phase P of a K-bit tile.
template <int K, int P>
__device__ __forceinline__ int mid_of(int rs, int v) {
  constexpr int LB = 4 * P;
  constexpr int BP = (K - LB) < 4 ? (K - LB) : 4;
  constexpr int J = 1 << BP;
  constexpr int NG = 16 / J;
  const int g = v / J, j = v % J;
  const int other = rs * NG + g;
  return (other & ((1 << LB) - 1)) | (j << LB) | ((other >> LB) << (LB + BP));
}

template <int K, int P>
__device__ __forceinline__ void phase_stages(double2 (&x)[16]) {
  constexpr int LB = 4 * P;
  constexpr int BP = (K - LB) < 4 ? (K - LB) : 4;
#pragma unroll
  for (int bb = 0; bb < BP; ++bb) {
    const int h = 1 << bb;
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      if (!(v & h)) {
        const double2 a = x[v], b = x[v + h];
        x[v] = add2(a, b);
        x[v + h] = sub2(a, b);
      }
    }
  }
}

template <int K, int P, int CP>
__device__ __forceinline__ void exchange(double2 (&x)[16], double2* tile, int cp, int rs) {
#pragma unroll
  for (int v = 0; v < 16; ++v) tile[mid_of<K, P>(rs, v) * CP + cp] = x[v];
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = tile[mid_of<K, P + 1>(rs, v) * CP + cp];
  __syncthreads();
}

template <int K>
__host__ __device__ constexpr int tile_cols() {
  return (1 << (13 - K)) > 64 ? 64 : ((1 << (13 - K)) < 8 ? 8 : (1 << (13 - K)));
}
template <int K>
__host__ __device__ constexpr int tile_threads() {
  return (1 << K) * tile_cols<K>() / 32;
}

// Fast pass: K in [4, 11]; X/Y 16-byte aligned, even ld, even d.
template <int K, bool DIAG>
// K = 7..9 are capped at 80 registers so three CTAs fit per SM (same-box A/Bs,
// `profiles/r02/ab_tile9_occupancy.log`, `ab_tile789_occupancy.log`): C3HD pass 0
// 1.47 -> 1.42 ms, pass 1 1.349 -> 1.337; C5 row-major passes -1.3 %
__global__ void __launch_bounds__(tile_threads<K>(), K >= 7 && K <= 9 ? 3 : 1) fwht_tile_kernel(
    const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy, int64_t nvalid, int lo,
    int64_t d, int64_t ntc, int64_t g_begin, uint64_t dkey, int64_t row0, double alpha) {
  constexpr int TC = tile_cols<K>();
  constexpr int CP = TC / 2;
  constexpr int NPH = (K + 3) / 4;
  extern __shared__ double2 tile[];  // [2^K][CP]
  const int cp = threadIdx.x % CP, rs = threadIdx.x / CP;
  const int64_t g = g_begin + blockIdx.x / ntc;
  const int64_t tc = blockIdx.x % ntc;
  const int64_t low = g & (((int64_t)1 << lo) - 1);
  const int64_t hi = g >> lo;
  const int64_t rbase = (hi << (lo + K)) + low;
  const int64_t c = tc * TC + 2 * cp;
  const bool cv = c < d;

  // Phase-0 rows of this thread are r0 + v * 2^lo (v = 0..15): one base pointer
  // and one stride instead of per-row 64-bit index arithmetic; rows >= nvalid
  // (zero padding) are the tail v >= nv.  The 16 loads are issued first; the D
  // signs are computed while they are in flight.
  double2 x[16];
  {
    const int64_t r0 = rbase + ((int64_t)(rs * 16) << lo);
    const int64_t left = nvalid - r0;
    const int nv = left <= 0 ? 0 : (left >= ((int64_t)16 << lo) ? 16 : (int)((left + ((int64_t)1 << lo) - 1) >> lo));
    const double2* p = reinterpret_cast<const double2*>(X + r0 * ldx + c);
    const int64_t step = (ldx << lo) / 2;  // in double2
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      x[v] = make_double2(0.0, 0.0);
      if (cv && v < nv) x[v] = __ldg(p + v * step);
    }
  }
  // D signs from the splitmix64 words, in registers (no memory access).
  uint32_t negmask = 0;
  if (DIAG) {
    if (lo == 0) {
      // 16 consecutive global rows g0..g0+15: their D bits are bits (g0 & 63) ..
      // of the 128-bit word pair (w1:w0), one funnel shift
      const int64_t g0 = row0 + rbase + mid_of<K, 0>(rs, 0);
      const uint64_t wa = stream_u(dkey, (uint64_t)(g0 >> 6));
      const int sh = (int)(g0 & 63);
      uint64_t win = wa >> sh;
      if (sh > 48) win |= stream_u(dkey, (uint64_t)((g0 >> 6) + 1)) << (64 - sh);
      const int64_t left = nvalid - (g0 - row0);
      const uint32_t vmask = left >= 16 ? 0xFFFFu : (left <= 0 ? 0u : ((1u << left) - 1u));
      negmask = (uint32_t)(win & 0xFFFFull) & vmask;
    } else {
#pragma unroll
      for (int v = 0; v < 16; ++v) {
        const int64_t r = rbase + ((int64_t)mid_of<K, 0>(rs, v) << lo);
        const int64_t gr = row0 + r;
        if (r < nvalid) negmask |= (uint32_t)((stream_u(dkey, (uint64_t)(gr >> 6)) >> (gr & 63)) & 1ull) << v;
      }
    }
  }
  if (DIAG) {
#pragma unroll
    for (int v = 0; v < 16; ++v)
      if ((negmask >> v) & 1u) x[v] = make_double2(-x[v].x, -x[v].y);
  }
  phase_stages<K, 0>(x);
  if constexpr (NPH > 1) {
    exchange<K, 0, CP>(x, tile, cp, rs);
    phase_stages<K, 1>(x);
  }
  if constexpr (NPH > 2) {
    exchange<K, 1, CP>(x, tile, cp, rs);
    phase_stages<K, 2>(x);
  }
  if (cv) {
    // last-phase mid = rs*NG + g + j*2^LB for v = g*J + j
    constexpr int LB = 4 * (NPH - 1);
    constexpr int BP = K - LB;
    constexpr int J = 1 << BP;
    constexpr int NG = 16 / J;
    double2* q = reinterpret_cast<double2*>(Y + (rbase + ((int64_t)(rs * NG) << lo)) * ldy + c);
    const int64_t sg = (ldy << lo) / 2, sj = (ldy << (lo + LB)) / 2;
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      const int g2 = v / J, j = v % J;
      q[g2 * sg + j * sj] = make_double2(alpha * x[v].x, alpha * x[v].y);
    }
  }
}


// Generic pass: any d, any alignment, K in [0, 5]; one thread per (group, column).
template <int K>
__global__ void __launch_bounds__(kGenThreads) fwht_generic_kernel(
    const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy, int64_t nvalid, int lo,
    int64_t d, int64_t g_begin, int64_t ngroups, const uint64_t* __restrict__ dw, int64_t row0, int64_t w0,
    int apply_diag, double alpha) {
  constexpr int R = 1 << K;
  const int64_t idx = (int64_t)blockIdx.x * kGenThreads + threadIdx.x;
  if (idx >= ngroups * d) return;
  const int64_t c = idx % d;
  const int64_t g = g_begin + idx / d;
  const int64_t low = g & (((int64_t)1 << lo) - 1);
  const int64_t hi = g >> lo;
  const int64_t rbase = (hi << (lo + K)) + low;
  double v[R];
  uint64_t wv[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int64_t r = rbase + ((int64_t)j << lo);
    wv[j] = (apply_diag && r < nvalid) ? dw[((row0 + r) >> 6) - w0] : 0ull;
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int64_t r = rbase + ((int64_t)j << lo);
    v[j] = r < nvalid ? X[r * ldx + c] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int64_t r = rbase + ((int64_t)j << lo);
    if ((wv[j] >> ((row0 + r) & 63)) & 1ull) v[j] = -v[j];
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

template <int K, bool DIAG>
int launch_tile(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nvalid, int lo, int64_t d,
                int64_t g_begin, int64_t g_count, uint64_t dkey, int64_t row0, double alpha, cudaStream_t st) {
  constexpr int TC = tile_cols<K>();
  constexpr int T = tile_threads<K>();
  const size_t smem = (size_t)(1 << K) * TC * sizeof(double);
  cudaFuncSetAttribute(fwht_tile_kernel<K, DIAG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntc = (d + TC - 1) / TC;
  const int64_t max_groups = ((1ll << 31) - 1) / ntc;  // keep every grid below 2^31 CTAs
  for (int64_t g0 = g_begin; g0 < g_begin + g_count; g0 += max_groups) {
    const int64_t gc = std::min(max_groups, g_begin + g_count - g0);
    fwht_tile_kernel<K, DIAG><<<(unsigned)(gc * ntc), T, smem, st>>>(X, ldx, Y, ldy, nvalid, lo, d, ntc, g0, dkey,
                                                                      row0, alpha);
    note_launch();
  }
  return check_launch("fwht_tile");
}

template <int K>
int launch_generic(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nvalid, int lo, int64_t d,
                   int64_t g_begin, int64_t g_count, const uint64_t* dw, int64_t row0, int64_t w0, int apply_diag,
                   double alpha, cudaStream_t st) {
  const int64_t per = ((1ll << 31) - 1) * (int64_t)kGenThreads / d;  // groups per launch (grid < 2^31)
  const int64_t step = per > 0 ? per : 1;
  for (int64_t g0 = g_begin; g0 < g_begin + g_count; g0 += step) {
    const int64_t gc = std::min(step, g_begin + g_count - g0);
    const int64_t threads = gc * d;
    fwht_generic_kernel<K><<<(unsigned)((threads + kGenThreads - 1) / kGenThreads), kGenThreads, 0, st>>>(
        X, ldx, Y, ldy, nvalid, lo, d, g0, gc, dw, row0, w0, apply_diag, alpha);
    note_launch();
  }
  return check_launch("fwht_generic");
}

template <int K>
int launch_tile_d(bool diag, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nvalid, int lo,
                  int64_t d, int64_t g_begin, int64_t g_count, uint64_t dkey, int64_t row0, double alpha,
                  cudaStream_t st) {
  return diag ? launch_tile<K, true>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dkey, row0, alpha, st)
              : launch_tile<K, false>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dkey, row0, alpha, st);
}

int launch_pass(bool fast, int K, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nvalid, int lo,
                int64_t d, int64_t g_begin, int64_t g_count, const uint64_t* dw, uint64_t dkey,
                int64_t row0, int64_t w0, int apply_diag, double alpha, cudaStream_t st) {
  const bool dg = apply_diag != 0;
  if (fast) {
#define SKH_TILE(KK) \
  case KK: return launch_tile_d<KK>(dg, X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dkey, row0, alpha, st)
    switch (K) {
      SKH_TILE(4);
      SKH_TILE(5);
      SKH_TILE(6);
      SKH_TILE(7);
      SKH_TILE(8);
      SKH_TILE(9);
      SKH_TILE(10);
      SKH_TILE(11);
      default: break;
    }
#undef SKH_TILE
  }
#define SKH_GEN(KK) \
  case KK: return launch_generic<KK>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, dw, row0, w0, apply_diag, alpha, st)
  switch (K) {
    SKH_GEN(0);
    SKH_GEN(1);
    SKH_GEN(2);
    SKH_GEN(3);
    SKH_GEN(4);
    SKH_GEN(5);
    default: break;
  }
#undef SKH_GEN
  set_error("internal: bad pass width %d", K);
  return SKH_EINVAL;
}

int kmax_fast() {
  // Widest pass used by the planner.  Default 8: single-CTA tile
  // passes run at the HBM copy rate, while the 9..11-bit passes (fused through
  // L2 or over DSMEM clusters) measured at ~0.5x of it on B200 because L2 and
  // DSMEM move data no faster than HBM (profiles/r01).  SKH_FWHT_KMAX=9..11
  // enables them for experiments.
  static int v = [] {
    const char* e = getenv("SKH_FWHT_KMAX");
    int k = e ? atoi(e) : 10;
    return k < 4 ? 4 : (k > 11 ? 11 : k);
  }();
  return v;
}

}  // namespace

// Split L bits into passes (low bits first): tile passes hold 4..kmax bits,
// generic passes at most 5.
std::vector<int> plan_passes(int L, bool fast) {
  std::vector<int> ks;
  if (L <= 0) {
    ks.push_back(0);
    return ks;
  }
  const int kmax = fast ? kmax_fast() : 5;
  if (!fast || kmax <= 8) {
    const int P = (L + kmax - 1) / kmax;
    for (int p = 0; p < P; ++p) ks.push_back(L / P + (p < L % P ? 1 : 0));
    return ks;
  }
  // Wider tile passes read/write narrower row segments and run slower; pick the
  // split of L bits minimising the summed relative pass cost (measured on B200,
  // a 4..8-bit pass runs at the copy rate).
  // (the small quadratic term prefers balanced splits among equal-cost ones)
  auto cost = [](int K) {
    return K <= 8 ? 1.0 + 0.001 * (K - 6) * (K - 6) : (K == 9 ? 1.28 : (K == 10 ? 2.2 : 2.4));
  };
  std::vector<double> best(L + 1, 1e30);
  std::vector<int> pick(L + 1, 0);
  best[0] = 0.0;
  for (int l = 1; l <= L; ++l)
    for (int K = 1; K <= std::min(l, kmax); ++K) {
      if (K < 4 && l != K) continue;  // narrow passes only as the whole plan
      const double c = best[l - K] + cost(K);
      if (c < best[l] - 1e-9) {
        best[l] = c;
        pick[l] = K;
      }
    }
  for (int l = L; l > 0; l -= pick[l]) ks.push_back(pick[l]);
  std::sort(ks.begin(), ks.end(), [](int a, int b) { return a > b; });
  return ks;
}

bool fwht_fast_ok(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t d) {
  return ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) % 16 == 0) && ldx % 2 == 0 &&
         ldy % 2 == 0 && d % 2 == 0 && d >= 16;
}

// Workspace of a transform call: [256-byte header][D bitmap for the generic first pass].
size_t fwht_counter_bytes(int64_t, int64_t) { return 256; }

size_t fwht_ws_bytes(int64_t nrows, int64_t nvalid, int64_t row0, int64_t d) {
  size_t b = fwht_counter_bytes(nrows, d);
  if (nvalid > 0) {
    const int64_t w0 = row0 >> 6, w1 = (row0 + nvalid - 1) >> 6;
    b += align_up(sizeof(uint64_t) * (size_t)(w1 - w0 + 1));
  }
  return b;
}

static uint64_t* bitmap_of(void* ws, int64_t nrows, int64_t d) {
  return reinterpret_cast<uint64_t*>(static_cast<char*>(ws) + fwht_counter_bytes(nrows, d));
}

// Enqueue the diag bitmap for rows [row0, row0 + nvalid) (used by generic passes).
int launch_diag_words(uint64_t seed, int64_t nrows, int64_t nvalid, int64_t row0, int64_t d, void* ws,
                      cudaStream_t st) {
  if (nvalid <= 0) return SKH_OK;
  const int64_t w0 = row0 >> 6, nw = ((row0 + nvalid - 1) >> 6) - w0 + 1;
  diag_words_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(key_diag(seed), w0, nw, bitmap_of(ws, nrows, d));
  note_launch();
  return check_launch("diag_words");
}

// One pass restricted to groups [g_begin, g_begin + g_count) (for chunked host input).
int launch_fwht_pass_range(uint64_t seed, int K, bool fast, const double* X, int64_t ldx, double* Y, int64_t ldy,
                           int64_t nrows, int64_t nvalid, int lo, int64_t d, int64_t g_begin, int64_t g_count,
                           void* ws, int64_t row0, int apply_diag, double alpha, cudaStream_t st) {
  if (fast && (K < 4 || K > 11)) fast = false;
  return launch_pass(fast, K, X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, bitmap_of(ws, nrows, d), key_diag(seed), row0, row0 >> 6, apply_diag, alpha, st);
}

int launch_fwht(uint64_t seed, int64_t nrows, int64_t nvalid, int64_t row0, int64_t d, const double* X,
                int64_t ldx, double* Y, int64_t ldy, int bit_lo, int bit_hi, int apply_diag, double alpha,
                void* ws, cudaStream_t st) {
  const bool fast = fwht_fast_ok(X, ldx, Y, ldy, d);
  int rc;
  std::vector<int> ks = plan_passes(bit_hi - bit_lo, fast);
  if (apply_diag && !(fast && ks[0] >= 4)) {  // only the generic first pass reads the bitmap
    rc = launch_diag_words(seed, nrows, nvalid, row0, d, ws, st);
    if (rc) return rc;
  }
  int lo = bit_lo;
  for (size_t p = 0; p < ks.size(); ++p) {
    const int K = ks[p];
    const bool first = p == 0, last = p + 1 == ks.size();
    const int64_t ngroups = nrows >> K;
    rc = launch_pass(fast && K >= 4, K, first ? X : Y, first ? ldx : ldy, Y, ldy, first ? nvalid : nrows, lo, d, 0,
                     ngroups, bitmap_of(ws, nrows, d), key_diag(seed), row0, row0 >> 6,
                     first ? apply_diag : 0, last ? alpha : 1.0, st);
    if (rc) return rc;
    lo += K;
  }
  return SKH_OK;
}

}  // namespace skh
