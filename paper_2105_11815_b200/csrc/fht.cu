// fht.cu -- the Hartley transform of HR-DHT (eq. (6.1))
// for row-major A and n = 2^L (2 <= L <= 18), in two HBM passes of our own
// instead of transpose + cuFFT + transpose.
//
// Fhat y = Re X - Im X with X = DFT(y), X_k = sum_j y_j W^{jk}, W = e^{-2 pi i/n}
// (cos t + sin t = Re e^{-it} - Im e^{-it}).  Four-step split n = n1 n2,
// j = j1 + n1 j2, k = k2 + n2 k1:
//   X[k2 + n2 k1] = sum_j1 W_n1^{j1 k1} [ W_n^{j1 k2} sum_j2 y[j1 + n1 j2] W_n2^{j2 k2} ].
// pass A (one CTA per j1 x column tile): the n2-point DFTs over the strided rows
//   j1 + n1 j2 of D [A | b] (D fused into the load), times W_n^{j1 k2}; y is real,
//   so only k2 <= n2/2 is stored: Z[(k2 n1 + j1)][c], complex;
// pass B (one CTA per k2 <= n2/2 x column tile): the n1-point DFTs over the n1
//   contiguous rows of Z, giving X_k for k = k2 + n2 k1, and
//   H[k] = Re X_k - Im X_k,  H[n - k] = Re X_k + Im X_k  (X_{n-k} = conj X_k),
//   the mirror written only for 0 < k2 < n2/2 (groups 0 and n2/2 hold their own
//   mirrors), so every row of H is written exactly once.
// Each tile DFT is an in-place radix-2 decimation-in-frequency FFT in shared
// memory, three butterfly stages per register round (one barrier per round);
// the output of position i is X[bitrev(i)].  Pass A transforms two real columns
// per complex FFT.  128-thread CTAs, ~36 KB of shared memory: 5-6 CTAs per SM
// in different phases (load / butterflies / store) keep HBM busy.  Traffic: pass A reads |A|, writes
// ~|A|; pass B reads ~|A|, writes |A|: 4|A|, the same as two WHT tile passes.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kThreads = 128;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

__device__ __forceinline__ double dsign_row(uint64_t dkey, int64_t g) {
  return ((stream_u(dkey, (uint64_t)(g >> 6)) >> (g & 63)) & 1ull) ? -1.0 : 1.0;
}

// tw[e] = W_n^e = (cos, -sin)(2 pi e / n), e = 0..n/2
__global__ void twiddle_kernel(int64_t n, double2* __restrict__ tw) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e > n / 2) return;
  double sv, cv;
  sincospi(2.0 * (double)e / (double)n, &sv, &cv);
  tw[e] = make_double2(cv, -sv);
}

__device__ __forceinline__ int bitrev(int i, int K) { return (int)(__brev((unsigned)i) >> (32 - K)); }

// One register round of the DIF FFT over index bits [P - a, P) of an N = 2^K
// point transform, TC columns, z[i * TC + c].  FIRST: the inputs come from
// `ld(u, t, i, c)` (group u of the thread, point t; registers or global memory)
// instead of shared memory; FINAL: P - a == 0, the
// outputs go to `epi(i, c, v)` instead of back to shared memory.  A thread takes
// CH groups at a time (all their loads issued before any butterfly), CH * 2^a
// <= 16 complex values in registers.
template <int K, int TC, int P, int A, bool FIRST, bool FINAL, class Ld, class Epi>
__device__ __forceinline__ void dif_round(double2* __restrict__ z, const double2* __restrict__ wN, Ld&& ld,
                                          Epi&& epi) {
  constexpr int N = 1 << K, R = 1 << A, p = P - A;
  constexpr int G = (N >> A) * TC;
  constexpr int GPT = (G + kThreads - 1) / kThreads;
  constexpr int CH0 = 16 / R < 1 ? 1 : 16 / R;
  constexpr int CH = CH0 < GPT ? CH0 : GPT;
#pragma unroll
  for (int u0 = 0; u0 < GPT; u0 += CH) {
    double2 v[CH][R];
    int bs[CH], los[CH], cs[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int g = threadIdx.x + (u0 + u) * kThreads;
      const int c = g % TC, rest = g / TC;
      los[u] = rest & ((1 << p) - 1);
      bs[u] = los[u] | ((rest >> p) << P);
      cs[u] = c;
      if (g < G && u0 + u < GPT) {
#pragma unroll
        for (int t = 0; t < R; ++t) {
          if constexpr (FIRST) v[u][t] = ld(u0 + u, t, bs[u] + (t << p), c);
          else v[u][t] = z[(bs[u] + (t << p)) * TC + c];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int g = threadIdx.x + (u0 + u) * kThreads;
      if (g >= G || u0 + u >= GPT) continue;
#pragma unroll
      for (int s = 0; s < A; ++s) {
        const int half = R >> (s + 1);
        const int q = P - 1 - s;
#pragma unroll
        for (int t = 0; t < R; ++t) {
          if (t & half) continue;
          const double2 a = v[u][t], w = v[u][t + half];
          v[u][t] = make_double2(a.x + w.x, a.y + w.y);
          const double2 dlt = make_double2(a.x - w.x, a.y - w.y);
          const int e = (los[u] | ((t & (half - 1)) << p)) << (K - 1 - q);
          v[u][t + half] = e ? cmul(dlt, wN[e]) : dlt;
        }
      }
      if constexpr (FINAL) {
#pragma unroll
        for (int t = 0; t < R; ++t) epi(bs[u] + (t << p), cs[u], v[u][t]);
      } else {
#pragma unroll
        for (int t = 0; t < R; ++t) z[(bs[u] + (t << p)) * TC + cs[u]] = v[u][t];
      }
    }
  }
}

// rounds of radix min(16, 2^P) from the top bits down; the first reads `ld`
// (wN: W_N^m, m < N/2, in shared memory)
// (FA: radix exponent of the first round, MAXA: of the others)
template <int K, int TC, int P, int MAXA, int FA, class Ld, class Epi>
__device__ __forceinline__ void dif_rounds(double2* z, const double2* wN, Ld&& ld, Epi&& epi) {
  constexpr bool FIRST = P == K;
  constexpr int A = P < (FIRST ? FA : MAXA) ? P : (FIRST ? FA : MAXA);
  if constexpr (P - A == 0) {
    dif_round<K, TC, P, A, FIRST, true>(z, wN, ld, epi);
  } else {
    dif_round<K, TC, P, A, FIRST, false>(z, wN, ld, epi);
    __syncthreads();
    dif_rounds<K, TC, P - A, MAXA, FA>(z, wN, ld, epi);
  }
}

// complex columns per tile (pass B; pass A packs twice as many real columns):
// 8 x 16 B = 128 B row segments.  For N = 512 the tile is 64 KB (3 CTAs/SM);
// 4 columns (6 CTAs/SM, 64 B segments) measured slower (C3HD pass B 3.30 vs 2.93 ms)
template <int K>
__host__ __device__ constexpr int tile_cols() {
  return 8;
}

// W_N^m = W_n^{m n/N}, m < N/2, into shared memory
template <int K>
__device__ __forceinline__ void load_wN(double2* wN, const double2* __restrict__ tw, int64_t n) {
  constexpr int N = 1 << K;
  const int64_t step = n >> K;
  for (int m = threadIdx.x; m < N / 2; m += kThreads) wN[m] = tw[m * step];
}

// pass A: K = log2 n2.  Two real columns share one complex FFT (z = y_a + i y_b;
// Y_a[k] = (Z[k] + conj Z[N-k]) / 2, Y_b[k] = (Z[k] - conj Z[N-k]) / 2i), so the
// real tile [N][2 TC], stored as is, IS the packed complex tile [N][TC].
template <int K>
__global__ void __launch_bounds__(kThreads, 5)
    dht_passA_kernel(int64_t n1, int64_t d, const double* __restrict__ A, int64_t lda, const double* __restrict__ b,
                     uint64_t dkey, const double2* __restrict__ tw, double2* __restrict__ Z, int64_t ldz,
                     int64_t ctiles) {
  constexpr int N = 1 << K, TC = tile_cols<K>(), TR = 2 * TC;
  extern __shared__ double2 smem[];
  double2* z = smem;
  double2* wN = smem + N * TC;
  double* sg = reinterpret_cast<double*>(wN + N / 2);
  const int64_t j1 = blockIdx.x / ctiles, c0 = (blockIdx.x % ctiles) * TR;
  // load the strided real tile straight into the first round's registers: group
  // u of this thread, point t = packed complex column c (real columns c0 + 2c,
  // c0 + 2c + 1) of row j1 + n1 (base + t 2^p1); every load in flight before
  // the twiddles and D signs are computed
  constexpr int A1 = K < 4 ? K : 4, R1 = 1 << A1, p1 = K - A1;
  constexpr int G1 = (N >> A1) * TC, GPT1 = (G1 + kThreads - 1) / kThreads;
  const bool pairs = ((reinterpret_cast<uintptr_t>(A) | (uintptr_t)(lda * 8)) & 15) == 0;
  double2 pre[GPT1][R1];
#pragma unroll
  for (int u = 0; u < GPT1; ++u) {
    const int g = threadIdx.x + u * kThreads;
    const int c = g % TC, rest = g / TC;
    const int base = (rest & ((1 << p1) - 1)) | ((rest >> p1) << K);
    const int64_t col = c0 + 2 * c;
#pragma unroll
    for (int t = 0; t < R1; ++t) {
      const int64_t row = j1 + n1 * (base + (t << p1));
      const double* a = A + row * lda;
      double2 x = make_double2(0.0, 0.0);
      if (g < G1) {
        if (pairs && col + 1 < d) {
          x = __ldg(reinterpret_cast<const double2*>(a + col));
        } else {
          x.x = col < d ? a[col] : (col == d && b) ? b[row] : 0.0;
          x.y = col + 1 < d ? a[col + 1] : (col + 1 == d && b) ? b[row] : 0.0;
        }
      }
      pre[u][t] = x;
    }
  }
  load_wN<K>(wN, tw, n1 << K);
  for (int j2 = threadIdx.x; j2 < N; j2 += kThreads) sg[j2] = dsign_row(dkey, j1 + n1 * j2);
  __syncthreads();
  dif_rounds<K, TC, K, 4, 4>(
      z, wN,
      [&](int u, int t, int i, int) {
        const double sgn = sg[i];
        return make_double2(sgn * pre[u][t].x, sgn * pre[u][t].y);
      },
      [&](int i, int c, double2 v) { z[i * TC + c] = v; });
  __syncthreads();
  for (int e = threadIdx.x; e < (N / 2 + 1) * TC; e += kThreads) {
    const int k2 = e / TC, c = e % TC;
    const double2 zk = z[bitrev(k2, K) * TC + c], zm = z[bitrev((N - k2) & (N - 1), K) * TC + c];
    double2 ya = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    double2 yb = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
    if (j1 && k2) {
      const double2 w = tw[j1 * k2];  // j1 k2 <= n/2
      ya = cmul(ya, w);
      yb = cmul(yb, w);
    }
    double2* dst = Z + ((int64_t)k2 * n1 + j1) * ldz + c0 + 2 * c;
    dst[0] = ya;
    dst[1] = yb;
  }
}

// pass B: K = log2 n1
template <int K>
__global__ void __launch_bounds__(kThreads, K >= 9 ? 3 : 5)
    dht_passB_kernel(int64_t n2, int64_t d, const double2* __restrict__ Z, int64_t ldz,
                     const double2* __restrict__ tw, double* __restrict__ H, int64_t ldh, double* __restrict__ hb,
                     int64_t ctiles) {
  constexpr int N = 1 << K, TC = tile_cols<K>();
  extern __shared__ double2 smem[];
  double2* z = smem;
  double2* wN = smem + N * TC;
  const int64_t n = n2 << K;
  const int64_t k2 = blockIdx.x / ctiles, c0 = (blockIdx.x % ctiles) * TC;
  const double2* src = Z + (k2 << K) * ldz + c0;
  load_wN<K>(wN, tw, n);
  __syncthreads();
  auto ld = [&](int, int, int j1, int c) { return src[(int64_t)j1 * ldz + c]; };
  const bool mirror = k2 > 0 && 2 * k2 < n2;
  dif_rounds<K, TC, K, 4, (K >= 9 ? 5 : 4)>(z, wN, ld, [&](int i, int c, double2 v) {
    const int64_t col = c0 + c;
    if (col > d || (col == d && !hb)) return;
    const int64_t k = k2 + n2 * bitrev(i, K);
    double* dst = col < d ? H + col : hb;
    const int64_t stride = col < d ? ldh : 1;
    dst[k * stride] = v.x - v.y;
    if (mirror) dst[(n - k) * stride] = v.x + v.y;
  });
}

template <int K>
int launch_A(int64_t n1, int64_t d, const double* A, int64_t lda, const double* b, uint64_t dkey, const double2* tw,
             double2* Z, int64_t ldz, cudaStream_t st) {
  constexpr int N = 1 << K;
  const int64_t ctiles = ldz / (2 * tile_cols<K>());
  const size_t sm = sizeof(double2) * (size_t)(N * tile_cols<K>() + N / 2) + sizeof(double) * N;
  cudaFuncSetAttribute(dht_passA_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dht_passA_kernel<K><<<(unsigned)(n1 * ctiles), kThreads, sm, st>>>(n1, d, A, lda, b, dkey, tw, Z, ldz, ctiles);
  note_launch();
  return check_launch("dht pass A");
}

template <int K>
int launch_B(int64_t n2, int64_t d, const double2* Z, int64_t ldz, const double2* tw, double* H, int64_t ldh,
             double* hb, cudaStream_t st) {
  constexpr int N = 1 << K;
  const int64_t ctiles = ldz / tile_cols<K>();
  const size_t sm = sizeof(double2) * (size_t)(N * tile_cols<K>() + N / 2);
  cudaFuncSetAttribute(dht_passB_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dht_passB_kernel<K><<<(unsigned)((n2 / 2 + 1) * ctiles), kThreads, sm, st>>>(n2, d, Z, ldz, tw, H, ldh, hb,
                                                                               ctiles);
  note_launch();
  return check_launch("dht pass B");
}

template <int K = 1>
int dispatch_A(int k, int64_t n1, int64_t d, const double* A, int64_t lda, const double* b, uint64_t dkey,
               const double2* tw, double2* Z, int64_t ldz, cudaStream_t st) {
  if constexpr (K > 9) {
    return SKH_EINVAL;
  } else {
    if (k == K) return launch_A<K>(n1, d, A, lda, b, dkey, tw, Z, ldz, st);
    return dispatch_A<K + 1>(k, n1, d, A, lda, b, dkey, tw, Z, ldz, st);
  }
}

template <int K = 1>
int dispatch_B(int k, int64_t n2, int64_t d, const double2* Z, int64_t ldz, const double2* tw, double* H,
               int64_t ldh, double* hb, cudaStream_t st) {
  if constexpr (K > 9) {
    return SKH_EINVAL;
  } else {
    if (k == K) return launch_B<K>(n2, d, Z, ldz, tw, H, ldh, hb, st);
    return dispatch_B<K + 1>(k, n2, d, Z, ldz, tw, H, ldh, hb, st);
  }
}

int ilog2(int64_t n) {
  int L = 0;
  while ((1ll << L) < n) ++L;
  return L;
}

// pass B (contiguous rows) takes the larger half of an odd L: measured faster
// than a 9-bit strided pass A (C3HD: 6.32 vs 7.32 ms with 8-column tiles)
int split_L1(int L) { return (L + 1) / 2; }

}  // namespace

bool dht_pow2_supported(int64_t n) { return n >= 4 && n <= (1ll << 18) && (n & (n - 1)) == 0; }

// columns of Z (complex), a multiple of both tile widths
int64_t dht_pow2_ldz(int64_t ncol) { return (ncol + 15) / 16 * 16; }

size_t dht_pow2_z_elems(int64_t n, int64_t ncol) {
  const int L = ilog2(n), L1 = split_L1(L), L2 = L - L1;
  return (size_t)(((1ll << L2) / 2 + 1) << L1) * (size_t)dht_pow2_ldz(ncol);
}

// H (row-major, ldh) and hb = Fhat D [A | b], unnormalised (sum, no n^{-1/2}).
// Z: dht_pow2_z_elems complex; tw: n/2 + 1 complex.
int launch_dht_pow2(int64_t n, int64_t d, const double* A, int64_t lda, const double* b, uint64_t dkey,
                    double2* Z, double2* tw, double* H, int64_t ldh, double* hb, cudaStream_t st) {
  const int L = ilog2(n), L1 = split_L1(L), L2 = L - L1;
  const int64_t n1 = 1ll << L1, n2 = 1ll << L2;
  const int64_t ldz = dht_pow2_ldz(d + (b ? 1 : 0));
  twiddle_kernel<<<(unsigned)((n / 2 + 1 + 255) / 256), 256, 0, st>>>(n, tw);
  note_launch();
  int rc = check_launch("dht twiddles");
  if (rc) return rc;
  skh_trace_mark(st, "twiddle");
  if ((rc = dispatch_A(L2, n1, d, A, lda, b, dkey, tw, Z, ldz, st))) return rc;
  skh_trace_mark(st, "dht_passA");
  if ((rc = dispatch_B(L1, n2, d, Z, ldz, tw, H, ldh, b ? hb : nullptr, st))) return rc;
  skh_trace_mark(st, "dht_passB");
  return SKH_OK;
}

}  // namespace skh
