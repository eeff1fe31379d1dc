// cm.cu -- the sketch of a COLUMN-MAJOR A (the paper's own LAPACK/FFTW layout,
// PAPER.md L1073-1081): S_h H D A in two HBM passes with the
// gather fused into the second, and plain S A in one.
//
// Column c of A is a contiguous n-vector, so
//  * pass 1 applies D (L793) and the butterflies of the low 13 row bits to
//    contiguous 64 KiB chunks (cm_pass1_kernel), and
//  * pass 2 applies the remaining K2 = L - 13 <= 8 bits to tiles of 2^K2 rows
//    at stride 2^13 x W contiguous rows (4096 positions per column), and never
//    writes the transformed rows back: each tile's final values are added
//    straight into the column's sketch, whose m entries stay in shared memory
//    while one CTA sweeps the column (two CTAs per SM).
// HBM traffic is 2|A| + |A| + |SA| instead of the 7|A| of the row-major
// three-pass plan.
//
// Determinism without atomics: the rows of a pass-2 tile are the same for every
// column, so its (position p, draw q) entries are sorted once per sketch by
// rank -- the number of earlier positions of the tile hashed to the same bucket
// -- into a tile list (cm_lists_kernel).  Pass 2 adds every rank-0 entry (all in
// distinct buckets), syncs, then rank 1, and so on: a bucket receives a tile's
// entries in ascending row order and the tiles in order.  That order is fixed
// (bitwise reproducible), but for the transform path it is not the oracle's
// ascending order across the whole bucket (R17): SA agrees with the
// oracle to rounding (BASELINE tolerance 1e-12 relative Frobenius) and bit for
// bit on integer inputs.  Without the transform the tiles are consecutive
// 4096-row blocks, so the order IS ascending and the result is bit-identical.
// Butterfly stages still run low bit to high bit, so H D A itself is
// bit-identical to the oracle's (skh_rht_stages_colmajor).
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kP1Bits = 13;            // pass-1 tile: 2^13 contiguous rows (64 KiB)
constexpr int kLE = 12;                // pass-2 tile: 4096 positions per column
constexpr int kE = 1 << kLE;
constexpr int kRounds = 32;            // rank rounds per tile; the last one is serial
constexpr int kBucketBits = 19;        // list word: p (12) | bucket (19) | sign (1)
constexpr uint32_t kPadWord = 0xFFFFFFFFu;  // empty slot (bucket field >= any m)
constexpr int kRoffStride = 36;             // round offsets per tile (33 used; 144 B, 16-byte aligned)

// Words of one tile list: E s entries + 25 % for the bank-class padding.
__host__ __device__ constexpr int list_cap(int s) { return kE * s + (kE * s) / 4; }

// ------------------------------------------------------------------ pass 1
// 16-byte slot swizzle: conflict-free for the three layouts below.
__device__ __forceinline__ int swz(int q) { return q ^ ((q >> 4) & 7); }

__device__ __forceinline__ void bfly2(double2& a, double2& b) {
  const double2 u = a, v = b;
  a = make_double2(u.x + v.x, u.y + v.y);
  b = make_double2(u.x - v.x, u.y - v.y);
}

__device__ __forceinline__ void stages16(double2 (&x)[16]) {
#pragma unroll
  for (int h = 1; h < 16; h <<= 1) {
#pragma unroll
    for (int v = 0; v < 16; ++v)
      if (!(v & h)) bfly2(x[v], x[v + h]);
  }
}

__device__ __forceinline__ const double* col_in(const double* X, int64_t ldx, int64_t ncolX, const double* xb,
                                                int64_t c) {
  return c < ncolX ? X + c * ldx : xb;
}

// One CTA = one 2^13-row chunk of one column: rows base .. base + 8191, as 4096
// double2 q (rows 2q, 2q+1).  Element bit 0 is inside a double2; q bits 0-3,
// 4-7, 8-11 are the register phases, with two shared-memory exchanges; the
// load and the store use the q = t + 256 v layout (fully coalesced).
template <bool DIAG, bool VEC>
__global__ void __launch_bounds__(256, 3)
    cm_pass1_kernel(const double* __restrict__ X, int64_t ldx, int64_t ncolX, const double* __restrict__ xb,
                    double* __restrict__ Y, int64_t ldy, int64_t nvalid, int64_t nchunks, uint64_t dkey,
                    int64_t row0) {
  extern __shared__ double2 sm[];  // [4096], swizzled
  const int t = threadIdx.x;
  const int64_t c = blockIdx.x / nchunks;
  const int64_t base = (blockIdx.x % nchunks) << kP1Bits;
  const double* src = col_in(X, ldx, ncolX, xb, c) + base;
  double* dst = Y + c * ldy + base;
  const int64_t left = nvalid - base;  // valid rows in this chunk (may be <= 0 or >= 8192)
  double2 x[16];
  if (left >= (1 << kP1Bits)) {
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      const int q = t + 256 * v;
      if (VEC) {
        x[v] = __ldg(reinterpret_cast<const double2*>(src) + q);
      } else {
        x[v].x = __ldg(src + 2 * q);
        x[v].y = __ldg(src + 2 * q + 1);
      }
    }
  } else {
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      const int q = t + 256 * v;
      x[v].x = 2 * q < left ? __ldg(src + 2 * q) : 0.0;
      x[v].y = 2 * q + 1 < left ? __ldg(src + 2 * q + 1) : 0.0;
    }
  }
#pragma unroll
  for (int v = 0; v < 16; ++v) sm[swz(t + 256 * v)] = x[v];
  __syncthreads();
  // phase 0: q = v | t << 4 -> rows 32t .. 32t+31 of the chunk
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sm[swz(v | (t << 4))];
  if (DIAG) {
    // 32 consecutive global rows g0 .. g0+31: bits (g0 & 63) .. of the
    // splitmix64 word pair at u(key_DIAG, g0 >> 6); padding rows keep +0.
    const int64_t g0 = row0 + base + 32 * t;
    const int sh = (int)(g0 & 63);
    uint64_t win = stream_u(dkey, (uint64_t)(g0 >> 6)) >> sh;
    if (sh > 32) win |= stream_u(dkey, (uint64_t)((g0 >> 6) + 1)) << (64 - sh);
    uint32_t neg = (uint32_t)win;
    const int64_t lv = left - 32 * t;
    if (lv < 32) neg &= lv <= 0 ? 0u : ((1u << lv) - 1u);
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      if ((neg >> (2 * v)) & 1u) x[v].x = -x[v].x;
      if ((neg >> (2 * v + 1)) & 1u) x[v].y = -x[v].y;
    }
  }
#pragma unroll
  for (int v = 0; v < 16; ++v) {  // element bit 0
    const double a = x[v].x, b = x[v].y;
    x[v] = make_double2(a + b, a - b);
  }
  stages16(x);  // element bits 1-4
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 16; ++v) sm[swz(v | (t << 4))] = x[v];
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sm[swz((t & 15) | (v << 4) | ((t >> 4) << 8))];
  stages16(x);  // element bits 5-8
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 16; ++v) sm[swz((t & 15) | (v << 4) | ((t >> 4) << 8))] = x[v];
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sm[swz(t | (v << 8))];
  stages16(x);  // element bits 9-12
#pragma unroll
  for (int v = 0; v < 16; ++v) {
    const int q = t | (v << 8);
    if (VEC) {
      reinterpret_cast<double2*>(dst)[q] = x[v];
    } else {
      dst[2 * q] = x[v].x;
      dst[2 * q + 1] = x[v].y;
    }
  }
}

// Columns of at most 2^12 rows: the whole column in shared memory, stages one
// at a time (small problems only).
template <bool DIAG>
__global__ void cm_small_kernel(const double* __restrict__ X, int64_t ldx, int64_t ncolX,
                                const double* __restrict__ xb, double* __restrict__ Y, int64_t ldy, int64_t nvalid,
                                int L, uint64_t dkey, int64_t row0) {
  extern __shared__ double sv[];
  const int64_t c = blockIdx.x;
  const double* src = col_in(X, ldx, ncolX, xb, c);
  const int n = 1 << L;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v = i < nvalid ? src[i] : 0.0;
    if (DIAG && i < nvalid) {
      const int64_t g = row0 + i;
      if ((stream_u(dkey, (uint64_t)(g >> 6)) >> (g & 63)) & 1ull) v = -v;
    }
    sv[i] = v;
  }
  for (int bit = 0; bit < L; ++bit) {
    __syncthreads();
    const int h = 1 << bit;
    for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
      const int lo = i & (h - 1);
      const int a = ((i >> bit) << (bit + 1)) | lo;
      const double u = sv[a], w = sv[a + h];
      sv[a] = u + w;
      sv[a + h] = u - w;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) Y[c * ldy + i] = sv[i];
}

// ------------------------------------------------------------------ pass 2
// Tile tt of a pass over bits [lo, lo + K2): with W = 4096 >> K2 and
// nj = 2^lo / W j-blocks, position p = k W + j (k < 2^K2, j < W) is row
//   r = (tt / nj) 2^(lo+K2) + (tt % nj) W + j + k 2^lo.
// K2 = 0 (no stages) uses lo = 12: r = tt 4096 + p.
__device__ __forceinline__ int64_t tile_row(int64_t tt, int p, int K2, int lo) {
  const int lw = kLE - K2;  // W = 2^lw, nj = 2^(lo - lw): shifts and masks only
  const int k = p >> lw, j = p & ((1 << lw) - 1);
  const int64_t jb = tt & ((((int64_t)1) << (lo - lw)) - 1), hi = tt >> (lo - lw);
  return (hi << (lo + K2)) + (jb << lw) + j + ((int64_t)k << lo);
}

// Registers: phase 0 holds k bits 0..KR-1 (KR = min(K2, 4)) and VJ = 16 >> KR
// positions j; phase 1 (K2 > 4) holds k bits K2-4 .. K2-1.
template <int K2>
struct Geo {
  static constexpr int KR = K2 < 4 ? K2 : 4;
  static constexpr int VJ = 16 >> KR;
  static constexpr int W = kE >> K2;
  static constexpr int WT = W / VJ;  // threads per k group in phase 0
  __device__ static __forceinline__ int p0(int t, int v) {  // phase-0 position of value v
    const int vk = v / VJ, u = v % VJ;
    const int k = vk | ((t / WT) << KR);
    return k * W + (t % WT) + WT * u;
  }
  __device__ static __forceinline__ int p1(int t, int v) {  // phase-1 position (K2 > 4)
    const int k = (t / W) | (v << (K2 > 4 ? K2 - 4 : 0));
    return k * W + (t % W);
  }
  __device__ static __forceinline__ int pf(int t, int v) {  // position of the final values
    if constexpr (K2 > 4) return p1(t, v);
    else return p0(t, v);
  }
};

template <int K2>
__device__ __forceinline__ void phase0_stages(double (&x)[16]) {
  constexpr int KR = Geo<K2>::KR, VJ = Geo<K2>::VJ;
#pragma unroll
  for (int i = 0; i < KR; ++i) {
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      if (!(v & (VJ << i))) {
        const double a = x[v], b = x[v + (VJ << i)];
        x[v] = a + b;
        x[v + (VJ << i)] = a - b;
      }
    }
  }
}

template <int K2>
__device__ __forceinline__ void phase1_stages(double (&x)[16]) {
#pragma unroll
  for (int kb = 4; kb < K2; ++kb) {
    const int h = 1 << (kb - (K2 > 4 ? K2 - 4 : 0));
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      if (!(v & h)) {
        const double a = x[v], b = x[v + h];
        x[v] = a + b;
        x[v + h] = a - b;
      }
    }
  }
}

struct PassArgs {
  const double* X;  // input columns c < ncolX at X + c ldx, column ncolX at xb
  int64_t ldx, ncolX;
  const double* xb;
  int64_t ncols;   // columns processed (ncolX + (xb != NULL))
  int64_t nvalid;  // rows >= nvalid read as zero
  int64_t ntiles;  // tiles per column
  int lo;
  double* Y;       // !GATHER: output column c at Y + c ldy
  int64_t ldy;
  const uint32_t* lists;  // GATHER: [ntiles][4096 s] rank-sorted tile entries
  const int32_t* roff;    // [ntiles][kRounds + 1] round offsets
  int s;
  int b0, nb;             // buckets [b0, b0 + nb) accumulated by this launch
  double* SA;             // output column c < ncolSA at SA + c ldsa, column ncolSA at Sb
  int64_t ldsa, ncolSA;
  double* Sb;
  double alpha;
};

template <int K2>
__device__ __forceinline__ void load_tile(const PassArgs& a, int64_t col, int64_t tt, int t, double (&x)[16]) {
  const double* src = col < a.ncols ? col_in(a.X, a.ldx, a.ncolX, a.xb, col) : nullptr;
  const int64_t rb = tile_row(tt, Geo<K2>::p0(t, 0), K2, a.lo);
#pragma unroll
  for (int v = 0; v < 16; ++v) {
    // rows of this thread's values: rb + (k - k0) 2^lo + WT u, one base + strides
    const int vk = v / Geo<K2>::VJ, u = v % Geo<K2>::VJ;
    const int64_t r = rb + ((int64_t)vk << a.lo) + (int64_t)Geo<K2>::WT * u;
    x[v] = (src && r < a.nvalid) ? __ldg(src + r) : 0.0;
  }
}

// Value type of NC columns at one position.
template <int NC> struct Vec;
template <> struct Vec<1> {
  using T = double;
  __device__ static __forceinline__ T zero() { return 0.0; }
  __device__ static __forceinline__ T addsub(T acc, T v, bool neg) { return neg ? acc - v : acc + v; }
  __device__ static __forceinline__ double get(T v, int) { return v; }
};

// Persistent: CTA works on column groups (NC = 1 column) blockIdx.x,
// + gridDim.x, ...; for each, the ntiles tiles in order.  The next work item's
// 16 values per thread are loaded into registers while the current one is
// transformed and gathered.  256 threads per column.  Measured on B200 (C5):
// bound by shared-memory traffic and barrier latency of the rank-round scatter
// (~0.5 wavefronts per element against an HBM budget of ~0.3 cycles per
// element), not by HBM; a cp.async ring (3 tiles in flight) and two columns
// per CTA were both slower.
template <int K2, bool GATHER, int NC>
__global__ void __launch_bounds__(256 * NC, 2 / NC) cm_pass2_kernel(const PassArgs a) {
  using V = typename Vec<NC>::T;
  constexpr int NT = 256 * NC;
  extern __shared__ __align__(16) unsigned char smraw[];
  // [0, NC*32K): exchange buffer (NC x 4096 doubles) / final tile (4096 x NC doubles)
  constexpr int kTileBytes = NC * kE * 8;
  double* ex = reinterpret_cast<double*>(smraw);
  V* tile = reinterpret_cast<V*>(smraw);
  int32_t* sroff = reinterpret_cast<int32_t*>(smraw + kTileBytes);                   // [kRounds + 1] (+pad)
  uint32_t* slst = reinterpret_cast<uint32_t*>(smraw + kTileBytes + 256);            // [list_cap(s)]
  V* sa = reinterpret_cast<V*>(smraw + kTileBytes + 256 + (size_t)4 * list_cap(a.s));  // [nb]

  const int tid = threadIdx.x, h = tid >> 8, t = tid & 255;
  const int64_t ngroups = (a.ncols + NC - 1) / NC;
  const int64_t my_groups = ngroups > blockIdx.x ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nitems = my_groups * a.ntiles;
  const int nlw = GATHER ? list_cap(a.s) / 4 : 0;  // 16-byte chunks of one tile list

  auto group_of = [&](int64_t i) { return (int64_t)blockIdx.x + (i / a.ntiles) * gridDim.x; };
  auto issue_list = [&](int64_t tt) {
    if (!GATHER) return;
    const uint4* gl = reinterpret_cast<const uint4*>(a.lists + tt * (int64_t)list_cap(a.s));
    for (int i = tid; i < nlw; i += NT) {
      const unsigned dsts = (unsigned)__cvta_generic_to_shared(slst + 4 * i);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dsts), "l"(gl + i));
    }
    if (tid < kRounds + 1) sroff[tid] = a.roff[tt * kRoffStride + tid];
    asm volatile("cp.async.commit_group;\n" ::);
  };

  double x[16], xn[16];
  if (nitems > 0) {
    load_tile<K2>(a, NC * group_of(0) + h, 0, t, xn);
    issue_list(0);
  }
  for (int64_t i = 0; i < nitems; ++i) {
    const int64_t grp = group_of(i), tt = i % a.ntiles;
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = xn[v];
    if (i + 1 < nitems) load_tile<K2>(a, NC * group_of(i + 1) + h, (i + 1) % a.ntiles, t, xn);
    if (GATHER && tt == 0) {
      for (int b = tid; b < a.nb; b += NT) sa[b] = Vec<NC>::zero();
    }
    phase0_stages<K2>(x);
    if constexpr (K2 > 4) {
#pragma unroll
      for (int v = 0; v < 16; ++v) ex[h * kE + Geo<K2>::p0(t, v)] = x[v];
      __syncthreads();
#pragma unroll
      for (int v = 0; v < 16; ++v) x[v] = ex[h * kE + Geo<K2>::p1(t, v)];
      phase1_stages<K2>(x);
    }
    if (!GATHER) {
      const int64_t col = NC * grp + h;
      if (col < a.ncols) {
        double* dst = a.Y + col * a.ldy;
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const int p = Geo<K2>::pf(t, v);
          const int64_t r = tile_row(tt, p, K2, a.lo);
          if (r < a.nvalid) dst[r] = x[v];
        }
      }
      if constexpr (K2 > 4) __syncthreads();  // ex is rewritten by the next item
      continue;
    }
    __syncthreads();  // exchange reads done (K2 > 4) / previous walk done
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      const int p = Geo<K2>::pf(t, v);
      reinterpret_cast<double*>(tile)[NC * p + h] = x[v];
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    // rank rounds: every entry of round rho hits a distinct bucket
    for (int rho = 0; rho < kRounds; ++rho) {
      const int e0 = sroff[rho], e1 = sroff[rho + 1];
      if (e0 == e1) break;
      if (rho < kRounds - 1) {
        // entries of one round hit distinct buckets: kU of them in flight per thread
        constexpr int kU = 4;
        for (int e = e0 + tid; e < e1; e += kU * NT) {
          uint32_t w[kU];
          int bk[kU];
          V v[kU], acc[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int eu = e + u * NT;
            w[u] = eu < e1 ? slst[eu] : kPadWord;
            bk[u] = (int)((w[u] >> kLE) & ((1u << kBucketBits) - 1)) - a.b0;
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            if ((unsigned)bk[u] < (unsigned)a.nb) {
              v[u] = tile[w[u] & (kE - 1)];
              acc[u] = sa[bk[u]];
            }
          }
#pragma unroll
          for (int u = 0; u < kU; ++u)
            if ((unsigned)bk[u] < (unsigned)a.nb) sa[bk[u]] = Vec<NC>::addsub(acc[u], v[u], w[u] >> 31);
        }
      } else if (tid == 0) {  // ranks >= kRounds - 1, in list (= per-bucket rank) order
        for (int e = e0; e < e1; ++e) {
          const uint32_t w = slst[e];
          const int bk = (int)((w >> kLE) & ((1u << kBucketBits) - 1)) - a.b0;
          if ((unsigned)bk < (unsigned)a.nb) sa[bk] = Vec<NC>::addsub(sa[bk], tile[w & (kE - 1)], w >> 31);
        }
      }
      __syncthreads();
    }
    __syncthreads();  // every thread is past its last read of sroff / slst
    if (i + 1 < nitems) issue_list((i + 1) % a.ntiles);
    if (tt == a.ntiles - 1) {  // column group done: SA columns out
      for (int hh = 0; hh < NC; ++hh) {
        const int64_t c = NC * grp + hh;
        if (c >= a.ncols) break;
        double* o = c < a.ncolSA ? a.SA + c * a.ldsa : a.Sb;
        for (int b = tid; b < a.nb; b += NT) o[a.b0 + b] = a.alpha * Vec<NC>::get(sa[b], hh);
      }
      __syncthreads();  // sa is zeroed by the next group
    }
  }
}

// Warp-specialised pass 2 (GATHER, one column per CTA at a time, 512 threads):
// warps 0-7 produce -- load a tile, butterflies, the final values into tile
// buffer b (and the tile's list into list buffer b) -- while warps 8-15 consume
// the other buffer with the rank rounds.  The halves meet only at named
// barriers: FULL[b] (producers arrive, consumers wait) and EMPTY[b] (consumers
// arrive, producers wait); the exchange and the rank rounds each use a barrier
// of their own half.  Same arithmetic and order as cm_pass2_kernel.
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr int kBarProd = 1, kBarCons = 2, kBarFull = 3, kBarEmpty = 5;
// consumer threads: 384 measured slower than 256 (C3HD pass 2 3.52 vs 3.39 ms,
// C5 40.8 vs 39.4 ms) -- the halves share the shared-memory pipe, not threads
#ifndef SKH_WS_CONS
#define SKH_WS_CONS 256
#endif
constexpr int kRoffPad = 48;

__host__ __device__ constexpr size_t ws_smem_bytes(int s, int nb) {
  return 2 * (size_t)kE * 8 + 2 * (size_t)4 * list_cap(s) + 2 * sizeof(int32_t) * kRoffPad + 8 * (size_t)nb;
}

template <int K2, int CONS>
__global__ void __launch_bounds__(256 + CONS, 1) cm_pass2_ws_kernel(const PassArgs a) {
  constexpr int NALL = 256 + CONS;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int cap = list_cap(a.s);
  double* buf = reinterpret_cast<double*>(smraw);                                   // [2][kE]
  uint32_t* lst = reinterpret_cast<uint32_t*>(smraw + 2 * (size_t)kE * 8);          // [2][cap]
  int32_t* ro = reinterpret_cast<int32_t*>(smraw + 2 * (size_t)kE * 8 + 2 * (size_t)4 * cap);  // [2][kRoffPad]
  double* sa = reinterpret_cast<double*>(smraw + 2 * (size_t)kE * 8 + 2 * (size_t)4 * cap +
                                         2 * sizeof(int32_t) * kRoffPad);  // [nb]
  const int tid = threadIdx.x;
  const bool producer = tid < 256;
  const int t = producer ? tid : tid - 256;
  const int64_t my_cols = a.ncols > blockIdx.x ? (a.ncols - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nitems = my_cols * a.ntiles;
  auto col_of = [&](int64_t i) { return (int64_t)blockIdx.x + (i / a.ntiles) * gridDim.x; };
  if (producer) {
    double x[16], xn[16];
    if (nitems > 0) load_tile<K2>(a, col_of(0), 0, t, xn);
    for (int64_t i = 0; i < nitems; ++i) {
      const int b = (int)(i & 1);
      const int64_t tt = i % a.ntiles;
#pragma unroll
      for (int v = 0; v < 16; ++v) x[v] = xn[v];
      if (i + 1 < nitems) load_tile<K2>(a, col_of(i + 1), (i + 1) % a.ntiles, t, xn);
      phase0_stages<K2>(x);
      if (i >= 2) nbar_sync(kBarEmpty + b, NALL);  // the consumers are done with buffer b
      double* ex = buf + (size_t)b * kE;
      // this tile's list and round offsets into list buffer b
      const uint4* gl = reinterpret_cast<const uint4*>(a.lists + tt * (int64_t)cap);
      uint32_t* dl = lst + (size_t)b * cap;
      for (int k = t; k < cap / 4; k += 256) {
        const unsigned dsts = (unsigned)__cvta_generic_to_shared(dl + 4 * k);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dsts), "l"(gl + k));
      }
      asm volatile("cp.async.commit_group;\n" ::);
      if (t < kRounds + 1) ro[b * kRoffPad + t] = a.roff[tt * kRoffStride + t];
      if constexpr (K2 > 4) {
#pragma unroll
        for (int v = 0; v < 16; ++v) ex[Geo<K2>::p0(t, v)] = x[v];
        nbar_sync(kBarProd, 256);
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = ex[Geo<K2>::p1(t, v)];
        phase1_stages<K2>(x);
        nbar_sync(kBarProd, 256);  // exchange reads done before the final values overwrite it
      }
#pragma unroll
      for (int v = 0; v < 16; ++v) ex[Geo<K2>::pf(t, v)] = x[v];
      asm volatile("cp.async.wait_all;\n" ::);
      nbar_arrive(kBarFull + b, NALL);
    }
  } else {
    for (int64_t i = 0; i < nitems; ++i) {
      const int b = (int)(i & 1);
      const int64_t tt = i % a.ntiles, col = col_of(i);
      if (tt == 0) {
        for (int k = t; k < a.nb; k += CONS) sa[k] = 0.0;
        nbar_sync(kBarCons, CONS);
      }
      nbar_sync(kBarFull + b, NALL);
      const double* tile = buf + (size_t)b * kE;
      const uint32_t* slst = lst + (size_t)b * cap;
      const int32_t* sroff = ro + b * kRoffPad;
      for (int rho = 0; rho < kRounds; ++rho) {
        const int e0 = sroff[rho], e1 = sroff[rho + 1];
        if (e0 == e1) break;
        if (rho < kRounds - 1) {
          constexpr int kU = 4;
          for (int e = e0 + t; e < e1; e += kU * CONS) {
            uint32_t w[kU];
            int bk[kU];
            double v[kU], acc[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const int eu = e + u * CONS;
              w[u] = eu < e1 ? slst[eu] : kPadWord;
              bk[u] = (int)((w[u] >> kLE) & ((1u << kBucketBits) - 1)) - a.b0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              if ((unsigned)bk[u] < (unsigned)a.nb) {
                v[u] = tile[w[u] & (kE - 1)];
                acc[u] = sa[bk[u]];
              }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u)
              if ((unsigned)bk[u] < (unsigned)a.nb) sa[bk[u]] = (w[u] >> 31) ? acc[u] - v[u] : acc[u] + v[u];
          }
        } else if (t == 0) {
          for (int e = e0; e < e1; ++e) {
            const uint32_t w = slst[e];
            const int bk = (int)((w >> kLE) & ((1u << kBucketBits) - 1)) - a.b0;
            if ((unsigned)bk < (unsigned)a.nb) sa[bk] = (w >> 31) ? sa[bk] - tile[w & (kE - 1)] : sa[bk] + tile[w & (kE - 1)];
          }
        }
        nbar_sync(kBarCons, CONS);
      }
      if (i + 2 < nitems) nbar_arrive(kBarEmpty + b, NALL);  // buffer b free (no arrival left unmatched)
      if (tt == a.ntiles - 1) {  // column done: SA column out (the last round ended with a consumer barrier)
        if (col < a.ncols) {
          double* o = col < a.ncolSA ? a.SA + col * a.ldsa : a.Sb;
          for (int k = t; k < a.nb; k += CONS) o[a.b0 + k] = a.alpha * sa[k];
        }
        nbar_sync(kBarCons, CONS);  // sa is zeroed for the next column
      }
    }
  }
}

int g_nsm = 0;
int num_sms() {
  if (!g_nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, dev);
    if (g_nsm <= 0) g_nsm = 148;
  }
  return g_nsm;
}

template <typename F>
int set_smem(F* f, size_t bytes) {
  if (bytes > 48 * 1024) {
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
      cudaGetLastError();
      set_error("cannot reserve %zu bytes of shared memory", bytes);
      return SKH_ECUDA;
    }
  }
  return SKH_OK;
}

// ------------------------------------------------------------------ launch helpers
// ------------------------------------------------------------------ tile lists
// One warp per tile.  Entries e = p s + q (q = draw) in ascending e; the rank of
// an entry is the number of earlier entries of the tile in the same bucket
// (warp __match_any_sync + per-bucket counters in shared memory, so it is
// deterministic).  Rank group rho (ranks clamped to kRounds - 1) occupies
// [roff[rho], roff[rho+1]).  Within a group the buckets are distinct, so the
// order is free: slot off + ncls i + c holds the i-th entry whose bucket is = c
// (mod ncls), empty slots are kPadWord.  With ncls = 16 (one column per CTA,
// 8-byte SA entries) every half-warp, and with ncls = 8 (column pairs, 16-byte
// entries) every quarter-warp, then addresses distinct banks of the SA.  A tile whose padded groups would exceed list_cap(s) keeps the
// plain ascending-e order instead (correct, only slower).
__global__ void cm_lists_kernel(const int32_t* __restrict__ col_rows, const int8_t* __restrict__ col_signs, int s,
                                int64_t m, int K2, int lo, int64_t nvalid, int ncls, uint32_t* __restrict__ lists,
                                int32_t* __restrict__ roff) {
  extern __shared__ unsigned char smraw[];
  int32_t* hist = reinterpret_cast<int32_t*>(smraw);      // [32][16]
  int32_t* cur = hist + 512;                              // [32][16]
  int32_t* off = cur + 512;                               // [34]: offsets + padded flag
  uint16_t* cnt = reinterpret_cast<uint16_t*>(smraw + 8192);  // [m]
  const int lane = threadIdx.x;
  const int64_t tt = blockIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  const int cap = list_cap(s);
  uint32_t* out = lists + tt * (int64_t)cap;
  const int ne = kE * s;
  bool padded = true;
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t b = lane; b < m; b += 32) cnt[b] = 0;
    if (pass == 0)
      for (int i = lane; i < 512; i += 32) hist[i] = 0;
    __syncwarp();
    for (int e0 = 0; e0 < ne; e0 += 32) {
      const int e = e0 + lane;
      const int p = e / s, q = e - p * s;
      const int64_t r = tile_row(tt, p, K2, lo);
      const bool valid = r < nvalid;
      if (__ballot_sync(0xffffffffu, valid) == 0u) continue;
      int bk = -1, neg = 0;
      if (valid) {
        bk = col_rows[r * s + q];
        neg = col_signs[r * s + q] < 0;
      }
      const unsigned grp = __match_any_sync(0xffffffffu, bk);
      const int base = valid ? (int)cnt[bk] : 0;
      __syncwarp();
      const int rank = base + __popc(grp & lt);
      if (valid && ((grp >> lane) >> 1) == 0u) cnt[bk] = (uint16_t)(base + __popc(grp));
      __syncwarp();
      const int rk = min(rank, kRounds - 1);
      const int key = rk * 16 + (padded ? (bk & (ncls - 1)) : 0);
      if (pass == 0) {
        if (valid) atomicAdd(&hist[rk * 16 + (bk & (ncls - 1))], 1);
      } else {
        const unsigned g2 = __match_any_sync(0xffffffffu, valid ? key : -1);
        const int idx = valid ? cur[key] + __popc(g2 & lt) : 0;
        __syncwarp();
        if (valid && ((g2 >> lane) >> 1) == 0u) cur[key] += __popc(g2);
        __syncwarp();
        if (valid) {
          const int slot = padded ? off[rk] + ncls * idx + (bk & (ncls - 1)) : off[rk] + idx;
          out[slot] = (uint32_t)p | ((uint32_t)bk << kLE) | ((uint32_t)neg << 31);
        }
      }
    }
    __syncwarp();
    if (pass == 0) {
      if (lane == 0) {
        int acc = 0;
        for (int i = 0; i < kRounds; ++i) {  // padded group lengths
          int mx = 0;
          for (int c = 0; c < ncls; ++c) mx = max(mx, hist[i * 16 + c]);
          off[i] = acc;
          acc += ncls * mx;
        }
        off[kRounds] = acc;
        if (acc > cap) {  // plain order
          acc = 0;
          for (int i = 0; i < kRounds; ++i) {
            int t = 0;
            for (int c = 0; c < ncls; ++c) t += hist[i * 16 + c];
            off[i] = acc;
            acc += t;
          }
          off[kRounds] = acc;
          off[kRounds + 1] = 0;
        } else {
          off[kRounds + 1] = 1;
        }
        for (int i = 0; i <= kRounds; ++i) roff[tt * kRoffStride + i] = off[i];
      }
      __syncwarp();
      padded = off[kRounds + 1] != 0;
      for (int i = lane; i < 512; i += 32) cur[i] = 0;
      if (padded)
        for (int i = lane; i < off[kRounds]; i += 32) out[i] = kPadWord;
      __syncwarp();
    }
  }
}

// The same lists from W warps per tile (W <= 8, limited by W per-warp bucket
// counters of m uint16 in shared memory): the tile's entries are cut into W
// contiguous segments; (1) each warp counts its segment's buckets; (2) a
// prefix over warps gives every warp the number of earlier same-bucket entries,
// so it ranks its segment exactly as the one-warp walk would, adding to the
// rank-group histogram and to per-warp key counts; (3) prefixes of those
// counts give every warp its first slot per key, and a second ranking walk
// places the entries.  The lists are identical to cm_lists_kernel's.
__global__ void cm_lists_par_kernel(const int32_t* __restrict__ col_rows, const int8_t* __restrict__ col_signs,
                                    int s, int64_t m, int K2, int lo, int64_t nvalid, int ncls,
                                    uint32_t* __restrict__ lists, int32_t* __restrict__ roff) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int W = blockDim.x >> 5;
  int32_t* hist = reinterpret_cast<int32_t*>(smraw);  // [512]
  int32_t* off = hist + 512;                          // [64]: offsets + padded flag
  int32_t* kcp = off + 64;                            // [W][512] key counts (padded keys)
  int32_t* kcq = kcp + W * 512;                       // [W][32]  key counts (plain keys)
  uint16_t* cntw = reinterpret_cast<uint16_t*>(kcq + W * 32);  // [W][m]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t tt = blockIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  const int cap = list_cap(s);
  uint32_t* out = lists + tt * (int64_t)cap;
  const int ne = kE * s, seg = ne / W, e_lo = w * seg, e_hi = e_lo + seg;
  uint16_t* cnt = cntw + (int64_t)w * m;
  for (int64_t b = lane; b < m; b += 32) cnt[b] = 0;
  for (int i = lane; i < 512; i += 32) kcp[w * 512 + i] = 0;
  kcq[w * 32 + lane] = 0;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) hist[i] = 0;
  auto entry = [&](int e, int& bk, int& neg) {
    const int p = e / s, q = e - p * s;
    const int64_t r = tile_row(tt, p, K2, lo);
    bk = -1;
    neg = 0;
    if (r < nvalid) {
      bk = col_rows[r * s + q];
      neg = col_signs[r * s + q] < 0;
    }
  };
  __syncthreads();
  // (1) per-warp bucket counts
  for (int e0 = e_lo; e0 < e_hi; e0 += 32) {
    int bk, neg;
    entry(e0 + lane, bk, neg);
    const unsigned grp = __match_any_sync(0xffffffffu, bk);
    if (bk >= 0 && (grp & lt) == 0) cnt[bk] = (uint16_t)(cnt[bk] + __popc(grp));
    __syncwarp();
  }
  __syncthreads();
  for (int64_t b = threadIdx.x; b < m; b += blockDim.x) {  // exclusive prefix over warps
    int run = 0;
    for (int v = 0; v < W; ++v) {
      const int c = cntw[(int64_t)v * m + b];
      cntw[(int64_t)v * m + b] = (uint16_t)run;
      run += c;
    }
  }
  __syncthreads();
  // (2) ranks -> rank-group histogram and per-warp key counts
  for (int e0 = e_lo; e0 < e_hi; e0 += 32) {
    int bk, neg;
    entry(e0 + lane, bk, neg);
    const bool valid = bk >= 0;
    const unsigned grp = __match_any_sync(0xffffffffu, bk);
    const int base = valid ? (int)cnt[bk] : 0;
    __syncwarp();
    const int rank = base + __popc(grp & lt);
    if (valid && (grp & lt) == 0) cnt[bk] = (uint16_t)(base + __popc(grp));
    __syncwarp();
    if (valid) {
      const int rk = min(rank, kRounds - 1);
      atomicAdd(&hist[rk * 16 + (bk & (ncls - 1))], 1);
      atomicAdd(&kcp[w * 512 + rk * 16 + (bk & (ncls - 1))], 1);
      atomicAdd(&kcq[w * 32 + rk], 1);
    }
  }
  __syncthreads();
  for (int64_t b = threadIdx.x; b < m; b += blockDim.x) {  // counters back to the prefixes
    for (int v = W - 1; v >= 1; --v) cntw[(int64_t)v * m + b] = cntw[(int64_t)(v - 1) * m + b];
    cntw[b] = 0;
  }
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < kRounds; ++i) {  // padded group lengths
      int mx = 0;
      for (int c = 0; c < ncls; ++c) mx = max(mx, hist[i * 16 + c]);
      off[i] = acc;
      acc += ncls * mx;
    }
    off[kRounds] = acc;
    if (acc > cap) {  // plain order
      acc = 0;
      for (int i = 0; i < kRounds; ++i) {
        int t = 0;
        for (int c = 0; c < ncls; ++c) t += hist[i * 16 + c];
        off[i] = acc;
        acc += t;
      }
      off[kRounds] = acc;
      off[kRounds + 1] = 0;
    } else {
      off[kRounds + 1] = 1;
    }
    for (int i = 0; i <= kRounds; ++i) roff[tt * kRoffStride + i] = off[i];
  }
  __syncthreads();
  const bool padded = off[kRounds + 1] != 0;
  // per-warp first slot index per key: exclusive prefix over warps
  for (int key = threadIdx.x; key < 512; key += blockDim.x) {
    int run = 0;
    for (int v = 0; v < W; ++v) {
      int* c = padded ? &kcp[v * 512 + key] : (key < 32 ? &kcq[v * 32 + key] : nullptr);
      if (!c) break;
      const int x = *c;
      *c = run;
      run += x;
    }
  }
  if (padded)
    for (int i = threadIdx.x; i < off[kRounds]; i += blockDim.x) out[i] = kPadWord;
  __syncthreads();
  // (3) rank again and place
  int32_t* cur = padded ? kcp + w * 512 : kcq + w * 32;
  for (int e0 = e_lo; e0 < e_hi; e0 += 32) {
    const int e = e0 + lane;
    int bk, neg;
    entry(e, bk, neg);
    const bool valid = bk >= 0;
    const unsigned grp = __match_any_sync(0xffffffffu, bk);
    const int base = valid ? (int)cnt[bk] : 0;
    __syncwarp();
    const int rank = base + __popc(grp & lt);
    if (valid && (grp & lt) == 0) cnt[bk] = (uint16_t)(base + __popc(grp));
    __syncwarp();
    const int rk = min(rank, kRounds - 1);
    const int key = padded ? rk * 16 + (bk & (ncls - 1)) : rk;
    const unsigned g2 = __match_any_sync(0xffffffffu, valid ? key : -1);
    const int idx = valid ? cur[key] + __popc(g2 & lt) : 0;
    __syncwarp();
    if (valid && (g2 & lt) == 0) cur[key] += __popc(g2);
    __syncwarp();
    if (valid) {
      const int slot = padded ? off[rk] + ncls * idx + (bk & (ncls - 1)) : off[rk] + idx;
      out[slot] = (uint32_t)(e / s) | ((uint32_t)bk << kLE) | ((uint32_t)neg << 31);
    }
  }
}

// Warp-specialised pass 2 where it measured faster: C3HD (K2 = 4, s = 2) pass 2
// 4.48 -> 3.39 ms; C2 (K2 = 3, s = 1) equal; C5 (K2 = 8, s = 1) 38.5 -> 39.4 ms,
// so the 8-bit exchange case keeps the two-CTA kernel.  SKH_CM_WS=0/1 forces.
bool use_ws(int K2, int s) {
  static const int forced = [] {
    const char* e = getenv("SKH_CM_WS");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return forced >= 0 ? forced == 1 : (K2 <= 4 || s >= 2);
}

template <int K2>
int launch_pass2_ws(const PassArgs& a, cudaStream_t st) {
  const size_t smem = ws_smem_bytes(a.s, a.nb);
  constexpr int CONS = SKH_WS_CONS;
  auto* f = cm_pass2_ws_kernel<K2, CONS>;
  int rc = set_smem(f, smem);
  if (rc) return rc;
  const int64_t grid = std::min<int64_t>(a.ncols, (int64_t)num_sms());
  if (grid < 1) return SKH_OK;
  f<<<(unsigned)grid, 256 + CONS, smem, st>>>(a);
  note_launch();
  return check_launch("cm_pass2_ws");
}

template <int K2, bool GATHER, int NC>
int launch_pass2_nc(const PassArgs& a, cudaStream_t st) {
  if constexpr (GATHER && NC == 1) {
    if (use_ws(K2, a.s) && ws_smem_bytes(a.s, a.nb) <= 227 * 1024) return launch_pass2_ws<K2>(a, st);
  }
  const size_t tileb = (size_t)NC * kE * 8;
  const size_t smem = GATHER ? tileb + 256 + (size_t)4 * list_cap(a.s) + 8 * NC * (size_t)a.nb : tileb;
  auto* f = cm_pass2_kernel<K2, GATHER, NC>;
  int rc = set_smem(f, smem);
  if (rc) return rc;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, 256 * NC, smem);
  if (per_sm < 1) {
    set_error("cm pass 2: %zu bytes of shared memory do not fit an SM", smem);
    return SKH_EINVAL;
  }
  const int64_t ngroups = (a.ncols + NC - 1) / NC;
  const int64_t grid = std::min<int64_t>(ngroups, (int64_t)num_sms() * per_sm);
  if (grid < 1) return SKH_OK;
  f<<<(unsigned)grid, 256 * NC, smem, st>>>(a);
  note_launch();
  return check_launch("cm_pass2");
}

template <int K2, bool GATHER>
int launch_pass2_t(const PassArgs& a, cudaStream_t st) {
  return launch_pass2_nc<K2, GATHER, 1>(a, st);
}

}  // namespace

// Largest bucket range one pass-2 launch accumulates on chip for draw count s
// (one CTA per SM; smaller ranges let two CTAs share an SM).
int cm_max_buckets(int s) {
  const size_t avail = 227 * 1024 - (size_t)kE * 8 - 256 - (size_t)4 * list_cap(s);
  return s > 8 ? 0 : (int)(avail / 8);
}

// Pass 1 of columns of 2^L rows: bits [0, min(L, 13)).
int launch_cm_pass1(uint64_t seed, const double* X, int64_t ldx, int64_t ncolX, const double* xb, double* Y,
                    int64_t ldy, int64_t nvalid, int L, int apply_diag, int64_t row0, cudaStream_t st) {
  const int64_t ncols = ncolX + (xb ? 1 : 0);
  if (ncols == 0) return SKH_OK;
  const uint64_t dkey = key_diag(seed);
  if (L < kP1Bits) {
    const size_t smem = sizeof(double) << L;
    if (apply_diag)
      cm_small_kernel<true><<<(unsigned)ncols, 256, smem, st>>>(X, ldx, ncolX, xb, Y, ldy, nvalid, L, dkey, row0);
    else
      cm_small_kernel<false><<<(unsigned)ncols, 256, smem, st>>>(X, ldx, ncolX, xb, Y, ldy, nvalid, L, dkey, row0);
    note_launch();
    return check_launch("cm_small");
  }
  const int64_t nchunks = ((int64_t)1 << L) >> kP1Bits;
  const int64_t grid = ncols * nchunks;
  if (grid >= (1ll << 31)) {
    set_error("cm pass 1 grid too large");
    return SKH_EOVERFLOW;
  }
  const bool vec = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(xb) |
                     reinterpret_cast<uintptr_t>(Y)) % 16 == 0) &&
                   (ldx % 2 == 0 || ncolX <= 1) && (ldy % 2 == 0);
  const size_t smem = 65536;
#define SKH_P1(D, V)                                                                                       \
  do {                                                                                                     \
    int rc = set_smem(cm_pass1_kernel<D, V>, smem);                                                        \
    if (rc) return rc;                                                                                     \
    cm_pass1_kernel<D, V><<<(unsigned)grid, 256, smem, st>>>(X, ldx, ncolX, xb, Y, ldy, nvalid, nchunks, dkey, \
                                                             row0);                                        \
  } while (0)
  if (apply_diag) {
    if (vec) SKH_P1(true, true); else SKH_P1(true, false);
  } else {
    if (vec) SKH_P1(false, true); else SKH_P1(false, false);
  }
#undef SKH_P1
  note_launch();
  return check_launch("cm_pass1");
}

// Strided pass over bits [lo, lo + K2) (K2 <= 8), in place on Y (no gather).
int launch_cm_mid(double* Y, int64_t ldy, int64_t ncols, int64_t nrows, int lo, int K2, cudaStream_t st) {
  PassArgs a{};
  a.X = Y;
  a.ldx = ldy;
  a.ncolX = ncols;
  a.ncols = ncols;
  a.nvalid = nrows;
  a.ntiles = nrows >> kLE;
  a.lo = lo;
  a.Y = Y;
  a.ldy = ldy;
  a.s = 1;
  switch (K2) {
    case 1: return launch_pass2_t<1, false>(a, st);
    case 2: return launch_pass2_t<2, false>(a, st);
    case 3: return launch_pass2_t<3, false>(a, st);
    case 4: return launch_pass2_t<4, false>(a, st);
    case 5: return launch_pass2_t<5, false>(a, st);
    case 6: return launch_pass2_t<6, false>(a, st);
    case 7: return launch_pass2_t<7, false>(a, st);
    case 8: return launch_pass2_t<8, false>(a, st);
    default: set_error("cm mid pass: K2 = %d", K2); return SKH_EINVAL;
  }
}

size_t cm_lists_bytes(int64_t ntiles, int s) {
  return align_up(sizeof(uint32_t) * (size_t)ntiles * list_cap(s)) +
         align_up(sizeof(int32_t) * (size_t)ntiles * kRoffStride + 16);
}

// Tile lists of the final pass (bits [lo, lo + K2), or K2 = 0 row blocks).
int launch_cm_lists(const int32_t* col_rows, const int8_t* col_signs, int s, int64_t m, int K2, int lo,
                    int64_t nvalid, int64_t ntiles, void* lists_ws, cudaStream_t st) {
  uint32_t* lists = static_cast<uint32_t*>(lists_ws);
  int32_t* roff = reinterpret_cast<int32_t*>(static_cast<char*>(lists_ws) +
                                             align_up(sizeof(uint32_t) * (size_t)ntiles * list_cap(s)));
  const int ncls = 16;  // 8-byte SA entries: conflict-free half-warps
  static const bool one_warp = [] {
    const char* e = getenv("SKH_CM_LISTS_1W");
    return e && e[0] == '1';
  }();
  // W warps per tile while W per-warp m-entry counters fit (<= 200 KB)
  int W = 8;
  while (W > 1 && (size_t)W * (sizeof(int32_t) * 544 + sizeof(uint16_t) * (size_t)m) + 2304 > 200 * 1024) W >>= 1;
  if (!one_warp && W >= 2) {
    const size_t smem = 2304 + (size_t)W * sizeof(int32_t) * 544 + align_up(sizeof(uint16_t) * (size_t)W * m, 16);
    int rc = set_smem(cm_lists_par_kernel, smem);
    if (rc) return rc;
    cm_lists_par_kernel<<<(unsigned)ntiles, 32 * W, smem, st>>>(col_rows, col_signs, s, m, K2, lo, nvalid, ncls,
                                                                 lists, roff);
    note_launch();
    return check_launch("cm_lists_par");
  }
  const size_t smem = 8192 + align_up(sizeof(uint16_t) * (size_t)m, 16);
  int rc = set_smem(cm_lists_kernel, smem);
  if (rc) return rc;
  cm_lists_kernel<<<(unsigned)ntiles, 32, smem, st>>>(col_rows, col_signs, s, m, K2, lo, nvalid, ncls, lists, roff);
  note_launch();
  return check_launch("cm_lists");
}

// Final pass: bits [lo, lo + K2) then gather into SA columns (buckets in
// ranges of at most cm_max_buckets(s), one launch per range).
int launch_cm_gather(const double* X, int64_t ldx, int64_t ncolX, const double* xb, int64_t nvalid, int64_t ntiles,
                     int lo, int K2, const void* lists_ws, int s, int64_t m, double* SA, int64_t ldsa,
                     int64_t ncolSA, double* Sb, double alpha, cudaStream_t st) {
  PassArgs a{};
  a.X = X;
  a.ldx = ldx;
  a.ncolX = ncolX;
  a.xb = xb;
  a.ncols = ncolX + (xb ? 1 : 0);
  a.nvalid = nvalid;
  a.ntiles = ntiles;
  a.lo = lo;
  a.lists = static_cast<const uint32_t*>(lists_ws);
  a.roff = reinterpret_cast<const int32_t*>(static_cast<const char*>(lists_ws) +
                                            align_up(sizeof(uint32_t) * (size_t)ntiles * list_cap(s)));
  a.s = s;
  a.SA = SA;
  a.ldsa = ldsa;
  a.ncolSA = ncolSA;
  a.Sb = Sb;
  a.alpha = alpha;
  const int cap = cm_max_buckets(s);
  if (cap < 1) {
    set_error("column-major gather supports s <= 8");
    return SKH_EINVAL;
  }
  for (int64_t b0 = 0; b0 < m; b0 += cap) {
    a.b0 = (int)b0;
    a.nb = (int)std::min<int64_t>(cap, m - b0);
    int rc;
    switch (K2) {
      case 0: rc = launch_pass2_t<0, true>(a, st); break;
      case 1: rc = launch_pass2_t<1, true>(a, st); break;
      case 2: rc = launch_pass2_t<2, true>(a, st); break;
      case 3: rc = launch_pass2_t<3, true>(a, st); break;
      case 4: rc = launch_pass2_t<4, true>(a, st); break;
      case 5: rc = launch_pass2_t<5, true>(a, st); break;
      case 6: rc = launch_pass2_t<6, true>(a, st); break;
      case 7: rc = launch_pass2_t<7, true>(a, st); break;
      case 8: rc = launch_pass2_t<8, true>(a, st); break;
      default: set_error("cm gather: K2 = %d", K2); return SKH_EINVAL;
    }
    if (rc) return rc;
  }
  return SKH_OK;
}

}  // namespace skh
