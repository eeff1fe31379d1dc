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
// column, so a plan built once per sketch (cm_plan_kernel) gives each bucket
// the tile hits to exactly ONE consumer thread, with all of that bucket's
// entries of the tile in ascending row order; threads add only into their own
// buckets and tiles are separated by one barrier.  A bucket receives a tile's
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
constexpr int kP1Ring = 3;             // persistent pass 1: chunks in the shared-memory ring
constexpr int kLE = 12;                // pass-2 tile: 4096 positions per column
constexpr int kE = 1 << kLE;

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

// Persistent pass 1 for full chunks (nvalid covers every chunk, 16-byte
// aligned columns): one CTA per SM walks chunks blockIdx.x, + gridDim.x, ...;
// the next kP1Ring - 1 chunks are copied by cp.async straight into the other
// slots of a chunk ring in shared memory (already in the swizzled exchange
// layout) while this chunk's butterflies run in place in its slot, so HBM
// reads stay in flight across the compute.  Same stages, same order as
// cm_pass1_kernel.
template <bool DIAG>
__global__ void __launch_bounds__(256, 1)
    cm_pass1p_kernel(const double* __restrict__ X, int64_t ldx, int64_t ncolX, const double* __restrict__ xb,
                     double* __restrict__ Y, int64_t ldy, int64_t nchunks, int64_t total, uint64_t dkey,
                     int64_t row0) {
  extern __shared__ __align__(16) double2 smp[];  // [kP1Ring][4096], swizzled
  const int t = threadIdx.x;
  auto issue = [&](int64_t item, int half) {
    const int64_t c = item / nchunks;
    const double2* src = reinterpret_cast<const double2*>(col_in(X, ldx, ncolX, xb, c) + ((item % nchunks) << kP1Bits));
    double2* dsm = smp + half * 4096;
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      const int q = t + 256 * v;
      const unsigned d = (unsigned)__cvta_generic_to_shared(dsm + swz(q));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + q));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  int64_t item = blockIdx.x;
#pragma unroll
  for (int r = 0; r < kP1Ring - 1; ++r) {  // prologue: the first kP1Ring - 1 chunks in flight
    if (item + (int64_t)r * gridDim.x < total) issue(item + (int64_t)r * gridDim.x, r);
    else asm volatile("cp.async.commit_group;\n" ::);  // empty group: keeps the group count uniform
  }
  for (int i = 0; item < total; item += gridDim.x, ++i) {
    const int half = i % kP1Ring;
    __syncthreads();  // every read of the slot being refilled (chunk i - 1) is done
    const int64_t ahead = item + (int64_t)(kP1Ring - 1) * gridDim.x;
    if (ahead < total) issue(ahead, (i + kP1Ring - 1) % kP1Ring);
    else asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kP1Ring - 1));
    __syncthreads();  // this chunk has landed
    double2* sm = smp + half * 4096;
    const int64_t c = item / nchunks;
    const int64_t base = (item % nchunks) << kP1Bits;
    double2 x[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = sm[swz(v | (t << 4))];
    if (DIAG) {
      const int64_t g0 = row0 + base + 32 * t;
      const int sh = (int)(g0 & 63);
      uint64_t win = stream_u(dkey, (uint64_t)(g0 >> 6)) >> sh;
      if (sh > 32) win |= stream_u(dkey, (uint64_t)((g0 >> 6) + 1)) << (64 - sh);
      const uint32_t neg = (uint32_t)win;
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
    double2* dst = reinterpret_cast<double2*>(Y + c * ldy + base);
#pragma unroll
    for (int v = 0; v < 16; ++v) dst[t | (v << 8)] = x[v];
  }
}

// mbarrier helpers (CTA scope)
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void nbar(int id) { asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory"); }

// Persistent pass 1 with two teams of 8 warps per CTA (512 threads, one CTA
// per SM): team k takes the CTA's chunks i = k, k + 2, ...; chunk i lives in
// ring slot i % 3.  At the start of chunk i a team issues the cp.async copies
// of chunk i + 1 -- the OTHER team's next chunk -- into slot (i + 1) % 3, which
// held chunk i - 2 (its own, finished); each issuing thread's copies arrive on
// the slot's mbarrier (cp.async.mbarrier.arrive.noinc, 256 arrivals per
// phase), on which the other team waits.  While one team runs its butterflies
// the other's shared-memory phases and loads are in flight: twice the warps of
// cm_pass1p_kernel per SM.  Same stages, same order: bit-identical to it.
template <bool DIAG>
__global__ void __launch_bounds__(512, 1)
    cm_pass1t_kernel(const double* __restrict__ X, int64_t ldx, int64_t ncolX, const double* __restrict__ xb,
                     double* __restrict__ Y, int64_t ldy, int64_t nchunks, int64_t total, uint64_t dkey,
                     int64_t row0) {
  extern __shared__ __align__(16) double2 smp[];  // [3][4096], swizzled
  __shared__ __align__(8) uint64_t full[3];
  const int tid = threadIdx.x, team = tid >> 8, t = tid & 255;
  if (tid < 3) mbar_init(&full[tid], 256);
  __syncthreads();
  auto issue = [&](int64_t item, int slot) {  // 256 threads of one team
    const int64_t c = item / nchunks;
    const double2* src = reinterpret_cast<const double2*>(col_in(X, ldx, ncolX, xb, c) + ((item % nchunks) << kP1Bits));
    double2* dsm = smp + slot * 4096;
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      const int q = t + 256 * v;
      const unsigned d = (unsigned)__cvta_generic_to_shared(dsm + swz(q));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + q));
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&full[slot]))
                 : "memory");
  };
  const int64_t G = gridDim.x;
  if (team == 0 && (int64_t)blockIdx.x < total) issue(blockIdx.x, 0);  // chunk 0
  const int bar = 1 + team;
  for (int64_t i = team;; i += 2) {
    const int64_t item = (int64_t)blockIdx.x + i * G;
    if (item >= total) break;
    const int slot = (int)(i % 3);
    nbar(bar);  // this team's reads of chunk i - 2 (slot (i + 1) % 3) are done
    if (item + G < total) issue(item + G, (int)((i + 1) % 3));
    mbar_wait(&full[slot], (unsigned)((i / 3) & 1));
    double2* sm = smp + slot * 4096;
    const int64_t c = item / nchunks;
    const int64_t base = (item % nchunks) << kP1Bits;
    double2 x[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = sm[swz(v | (t << 4))];
    if (DIAG) {
      const int64_t g0 = row0 + base + 32 * t;
      const int sh = (int)(g0 & 63);
      uint64_t win = stream_u(dkey, (uint64_t)(g0 >> 6)) >> sh;
      if (sh > 32) win |= stream_u(dkey, (uint64_t)((g0 >> 6) + 1)) << (64 - sh);
      const uint32_t neg = (uint32_t)win;
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
    nbar(bar);
#pragma unroll
    for (int v = 0; v < 16; ++v) sm[swz(v | (t << 4))] = x[v];
    nbar(bar);
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = sm[swz((t & 15) | (v << 4) | ((t >> 4) << 8))];
    stages16(x);  // element bits 5-8
    nbar(bar);
#pragma unroll
    for (int v = 0; v < 16; ++v) sm[swz((t & 15) | (v << 4) | ((t >> 4) << 8))] = x[v];
    nbar(bar);
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = sm[swz(t | (v << 8))];
    stages16(x);  // element bits 9-12
    double2* dst = reinterpret_cast<double2*>(Y + c * ldy + base);
#pragma unroll
    for (int v = 0; v < 16; ++v) dst[t | (v << 8)] = x[v];
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

// Geo<K2>::pf for a runtime K2 (the plan kernel serves every pass width)
__device__ __forceinline__ int pf_rt(int K2, int t, int v) {
  switch (K2) {
    case 0: return Geo<0>::pf(t, v);
    case 1: return Geo<1>::pf(t, v);
    case 2: return Geo<2>::pf(t, v);
    case 3: return Geo<3>::pf(t, v);
    case 4: return Geo<4>::pf(t, v);
    case 5: return Geo<5>::pf(t, v);
    case 6: return Geo<6>::pf(t, v);
    case 7: return Geo<7>::pf(t, v);
    default: return Geo<8>::pf(t, v);
  }
}

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
  double* Y;       // mid passes: output column c at Y + c ldy
  int64_t ldy;
  const uint32_t* words;  // gather: [ntiles][plan_jcap(s)][kNC] owner plan words
  const int32_t* hdr;     // gather: [ntiles] steps J of the tile (< 0: serial list of -J words)
  const uint64_t* pbank;  // gather: [ntiles][kNP] staging bank of each producer value (4 bits per register)
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
  // rows of this thread's values: rb + vk 2^lo + WT u -- one base pointer and
  // compile-time multiples of the two strides; the bounds test is per tile
  const int64_t last = rb + ((int64_t)(16 / Geo<K2>::VJ - 1) << a.lo) + (int64_t)Geo<K2>::WT * (Geo<K2>::VJ - 1);
  if (src && last < a.nvalid) {
    const double* p = src + rb;
    const int64_t sk = (int64_t)1 << a.lo;
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = __ldg(p + (v / Geo<K2>::VJ) * sk + Geo<K2>::WT * (v % Geo<K2>::VJ));
    return;
  }
#pragma unroll
  for (int v = 0; v < 16; ++v) {
    const int vk = v / Geo<K2>::VJ, u = v % Geo<K2>::VJ;
    const int64_t r = rb + ((int64_t)vk << a.lo) + (int64_t)Geo<K2>::WT * u;
    x[v] = (src && r < a.nvalid) ? __ldg(src + r) : 0.0;
  }
}

// Mid pass (no gather): bits [lo, lo + K2) of 4096-position tiles, in place.
// Persistent CTA over (column, tile) items; the next item's 16 values per
// thread are loaded while the current one is transformed.
template <int K2>
__global__ void __launch_bounds__(256, 2) cm_mid_kernel(const PassArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  double* ex = reinterpret_cast<double*>(smraw);  // [4096] exchange buffer
  const int t = threadIdx.x;
  const int64_t my_cols = a.ncols > blockIdx.x ? (a.ncols - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nitems = my_cols * a.ntiles;
  auto col_of = [&](int64_t i) { return (int64_t)blockIdx.x + (i / a.ntiles) * gridDim.x; };
  double x[16], xn[16];
  if (nitems > 0) load_tile<K2>(a, col_of(0), 0, t, xn);
  for (int64_t i = 0; i < nitems; ++i) {
    const int64_t tt = i % a.ntiles, col = col_of(i);
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = xn[v];
    if (i + 1 < nitems) load_tile<K2>(a, col_of(i + 1), (i + 1) % a.ntiles, t, xn);
    phase0_stages<K2>(x);
    if constexpr (K2 > 4) {
#pragma unroll
      for (int v = 0; v < 16; ++v) ex[Geo<K2>::p0(t, v)] = x[v];
      __syncthreads();
#pragma unroll
      for (int v = 0; v < 16; ++v) x[v] = ex[Geo<K2>::p1(t, v)];
      phase1_stages<K2>(x);
      __syncthreads();  // ex is rewritten by the next item
    }
    if (col < a.ncols) {
      double* dst = a.Y + col * a.ldy;
#pragma unroll
      for (int v = 0; v < 16; ++v) {
        const int64_t r = tile_row(tt, Geo<K2>::pf(t, v), K2, a.lo);
        if (r < a.nvalid) dst[r] = x[v];
      }
    }
  }
}

// ------------------------------------------------------------------ fused final pass: owner plan
// The final pass applies the last K2 butterfly stages to a 4096-position tile
// and adds every final value into the column's sketch, which stays in shared
// memory while one CTA sweeps the column.  Determinism without atomics comes
// from OWNERSHIP: the rows of a tile are the same for every column, so a plan
// built once per sketch (cm_plan_kernel) hands every bucket that the tile hits
// to exactly one consumer thread, together with all of that bucket's entries
// of the tile in ascending position order.  A thread adds its entries one after
// the other (a read-modify-write of its own buckets, no other thread touches
// them during the tile); tiles are separated by one barrier.  A bucket thus
// receives the rows of each tile in ascending order, tile after tile -- the
// fixed order of DESIGN.md R17 -- with no rank rounds.
//
// Consumer thread c handles bucket class c & 15 (bucket = 16 kb + class), so
// the 16 lanes of a half-warp always address 16 distinct shared-memory banks of
// the sketch; the plan balances a class's entries over its 16 threads
// (slot u = 2 (c >> 5) + ((c >> 4) & 1)).
//
// Plan word: bits 0-11 position p in the tile, 12-27 kb (serial list: the local
// bucket), 28 first entry of its bucket in this thread's tile list, 29 valid
// (serial list only), 30 last entry of its bucket, 31 sign.  Padding words are 0.
// A tile's plan holds J steps (a multiple of 8) per consumer thread, stored as
// uint4 quads [j / 4][thread]; padding words are 0 (invalid), and the
// consumer predicates them off instead of branching.
constexpr int kNP = 256;  // producer threads (load, butterflies, stage)
constexpr int kNC = 256;  // consumer threads (owner adds)
constexpr int kNBuf = 2;  // staged tiles
constexpr uint32_t kHead = 1u << 28, kValid = 1u << 29, kLast = 1u << 30, kNeg = 1u << 31;
constexpr uint32_t kKbMask = (1u << 16) - 1;

__host__ __device__ constexpr int plan_jcap(int s) { return 24 * s + 16; }  // multiple of 4
__host__ __device__ constexpr int64_t plan_tile_words(int s) { return (int64_t)plan_jcap(s) * kNC; }
__host__ __device__ constexpr int nb_pad(int nb) { return (nb + 15) & ~15; }
__host__ __device__ __forceinline__ int64_t plan_index(int j, int c) { return ((int64_t)(j >> 2) * kNC + c) * 4 + (j & 3); }

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr int kBarProd = 1, kBarCons = 2, kBarFull = 3, kBarEmpty = 3 + kNBuf;

// cm_plan_kernel: sorted entries (4 B per entry) + class-major counters
__host__ __device__ constexpr size_t plan_smem_bytes(int s, int nb) {
  return (size_t)4 * kE * s + sizeof(int) * (size_t)nb_pad(nb) + 16;
}
__host__ __device__ constexpr size_t gather_smem_bytes(int nb, int ncol = 1) {
  return (size_t)ncol * ((size_t)kNBuf * kE * 8 + 8 * (size_t)nb_pad(nb));
}

// Warp-specialised (one CTA per SM, 512 threads): warps 0-7 produce -- load a
// tile (the next one is in flight in registers), run its butterflies (one
// exchange through the staging buffer when K2 > 4), leave the final values in
// staging buffer b -- while warps 8-15 consume the other buffer with the owner
// plan.  FULL[b] / EMPTY[b] named barriers hand the buffers over.
// NCOL = 2 (small m): the CTA carries TWO columns through every tile -- the
// producers stage both columns' tiles (two halves of buffer b), the consumers
// decode each plan word once and add it into both sketches (each column's adds
// in the same order as NCOL = 1: bit-identical results).
template <int K2, int NCOL>
__global__ void __launch_bounds__(kNP + kNC, 1) cm_gather_kernel(const PassArgs a) {
  constexpr int NALL = kNP + kNC;
  extern __shared__ __align__(16) unsigned char smraw[];
  double* buf = reinterpret_cast<double*>(smraw);                                   // [kNBuf][NCOL][kE]
  double* sa = reinterpret_cast<double*>(smraw + (size_t)kNBuf * NCOL * kE * 8);   // [NCOL][nb_pad]
  const int tid = threadIdx.x;
  const int nbp = nb_pad(a.nb);
  // the CTA's column groups g = blockIdx.x, + gridDim.x, ...; group g = columns NCOL g .. NCOL g + NCOL - 1
  const int64_t ngroups = (a.ncols + NCOL - 1) / NCOL;
  const int64_t my_groups = ngroups > blockIdx.x ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nitems = my_groups * a.ntiles;
  if (tid < kNP && K2 <= 4) {
    // no exchange (K2 <= 4): two register tiles with alternating roles (the loop
    // is unrolled by two), so the tile in flight is never copied into the one
    // being transformed (same-box A/B: C3HD pass 2 2.248 -> 2.216 ms, C2 unchanged;
    // with the exchange the doubled producer code measured slower on C5, so
    // K2 > 4 keeps the copy)
    const int t = tid;
    double xa[16], xb[16];
    uint64_t pba = 0, pbb = 0;
    int64_t ngrp = blockIdx.x, ntt = 0;  // the (group, tile) of the loads in flight
    int nh = 0;                          // ... and which column of the group
    const int64_t nq = nitems * NCOL;    // (item, column) steps
    if (nq > 0) {
      load_tile<K2>(a, NCOL * ngrp, ntt, t, xa);
      pba = __ldg(a.pbank + ntt * kNP + t);
    }
    auto step = [&](int64_t q, double (&x)[16], uint64_t pb, double (&xn)[16], uint64_t& pbn) {
      const int64_t i = q / NCOL;
      const int h = (int)(q - i * NCOL);
      const int b = (int)(i % kNBuf);
      if (++nh == NCOL) {
        nh = 0;
        if (++ntt == a.ntiles) {
          ntt = 0;
          ngrp += gridDim.x;
        }
      }
      if (q + 1 < nq) {
        load_tile<K2>(a, NCOL * ngrp + nh, ntt, t, xn);
        pbn = __ldg(a.pbank + ntt * kNP + t);
      }
      phase0_stages<K2>(x);
      if (h == 0 && i >= kNBuf) nbar_sync(kBarEmpty + b, NALL);
      double* ex = buf + ((size_t)b * NCOL + h) * kE;
#pragma unroll
      for (int v = 0; v < 16; ++v) ex[16 * (16 * v + (t >> 4)) + (int)((pb >> (4 * v)) & 15u)] = x[v];
      if (h == NCOL - 1) nbar_arrive(kBarFull + b, NALL);
    };
    for (int64_t q = 0; q < nq; q += 2) {
      step(q, xa, pba, xb, pbb);
      if (q + 1 < nq) step(q + 1, xb, pbb, xa, pba);
    }
    return;
  }
  if (tid < kNP) {
    const int t = tid;
    double x[16], xn[16];
    int64_t ngrp = blockIdx.x, ntt = 0;  // the (group, tile) of the loads in flight
    int nh = 0;                          // ... and which column of the group
    uint64_t pbn = 0;
    if (nitems > 0) {
      load_tile<K2>(a, NCOL * ngrp, ntt, t, xn);
      pbn = __ldg(a.pbank + ntt * kNP + t);
    }
    for (int64_t i = 0; i < nitems; ++i) {
      const int b = (int)(i % kNBuf);
#pragma unroll
      for (int h = 0; h < NCOL; ++h) {
        const uint64_t pb = pbn;
#pragma unroll
        for (int v = 0; v < 16; ++v) x[v] = xn[v];
        if (++nh == NCOL) {  // advance (group, tile, column)
          nh = 0;
          if (++ntt == a.ntiles) {
            ntt = 0;
            ngrp += gridDim.x;
          }
        }
        if (i + 1 < nitems || h + 1 < NCOL) {
          load_tile<K2>(a, NCOL * ngrp + nh, ntt, t, xn);
          pbn = __ldg(a.pbank + ntt * kNP + t);
        }
        phase0_stages<K2>(x);
        if (h == 0 && i >= kNBuf) nbar_sync(kBarEmpty + b, NALL);  // the consumers are done with buffer b
        double* ex = buf + ((size_t)b * NCOL + h) * kE;
        if constexpr (K2 > 4) {
#pragma unroll
          for (int v = 0; v < 16; ++v) ex[Geo<K2>::p0(t, v)] = x[v];
          nbar_sync(kBarProd, kNP);
#pragma unroll
          for (int v = 0; v < 16; ++v) x[v] = ex[Geo<K2>::p1(t, v)];
          phase1_stages<K2>(x);
          nbar_sync(kBarProd, kNP);  // exchange reads done before the final values overwrite it
        }
        // final values into the staging rows: store v of half-warp t / 16 fills row
        // 16 v + t / 16, each lane in the bank the plan chose (a permutation per
        // row), so that these stores and the consumers' reads are conflict-free
#pragma unroll
        for (int v = 0; v < 16; ++v) ex[16 * (16 * v + (t >> 4)) + (int)((pb >> (4 * v)) & 15u)] = x[v];
      }
      nbar_arrive(kBarFull + b, NALL);
    }
    return;
  }
  // ---- consumers: blocks of up to JB plan steps per thread (6 uint4 of words),
  // the next block in flight in registers while the current one is added
  constexpr int JB = 24;
  const int c = tid - kNP, cls = c & 15;
  const int64_t tw4 = plan_tile_words(a.s) / 4;
  const uint4* w4 = reinterpret_cast<const uint4*>(a.words) + c;
  const uint4 dq = make_uint4(0u, 0u, 0u, 0u);  // words past J: invalid (predicated off)
  auto load_block = [&](int64_t tt, int bk, int J8, uint4 (&dst)[6]) {
    const uint4* p = w4 + tt * tw4 + (int64_t)bk * (JB / 4) * kNC;
#pragma unroll
    for (int q = 0; q < 6; ++q) dst[q] = bk * JB + 4 * q < J8 ? __ldg(p + q * kNC) : dq;
  };
  uint4 cw[6], nw[6];
  double run[NCOL];  // running value of the open bucket run, per column
#pragma unroll
  for (int h = 0; h < NCOL; ++h) run[h] = 0.0;
  int Jc = nitems > 0 ? __ldg(a.hdr + 0) : 0;
  if (Jc > 0) load_block(0, 0, Jc, nw);
  int64_t grp = blockIdx.x, tt = 0;
  for (int64_t i = 0; i < nitems; ++i) {
    const int b = (int)(i % kNBuf);
    const int64_t ttn = tt + 1 == a.ntiles ? 0 : tt + 1;
    if (tt == 0) {
      for (int k = c; k < NCOL * nbp; k += kNC) sa[k] = 0.0;
      nbar_sync(kBarCons, kNC);
    }
    const int Jn = i + 1 < nitems ? __ldg(a.hdr + ttn) : 0;
    const int nbk = Jc > 0 ? (Jc + JB - 1) / JB : 0;
    nbar_sync(kBarFull + b, NALL);
    const double* tile = buf + (size_t)b * NCOL * kE;
    for (int bk = 0; bk < nbk; ++bk) {
#pragma unroll
      for (int q = 0; q < 6; ++q) cw[q] = nw[q];
      if (bk + 1 < nbk) load_block(tt, bk + 1, Jc, nw);
      else if (Jn > 0) load_block(ttn, 0, Jn, nw);
      const int steps = min(JB, Jc - bk * JB);
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        if (q * 4 >= steps) break;
        const uint32_t w[4] = {cw[q].x, cw[q].y, cw[q].z, cw[q].w};
        // a bucket's entries of the tile are consecutive in the thread's list and
        // are added in ascending row order with the running value kept in a
        // register: one shared-memory read at the head, one write at the last
        // entry (the order is that of one add per entry).  Padding words are 0:
        // they read tile[0] (a broadcast) and neither load nor store the sketch.
        double v[NCOL][4], a0[NCOL][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int p = w[u] & (kE - 1);
          const int kk = (int)((w[u] >> 12 & kKbMask) << 4) + cls;
          SKH_CHECK(kk < nbp);
#pragma unroll
          for (int h = 0; h < NCOL; ++h) {
            v[h][u] = tile[h * kE + p];
            if (w[u] & kHead) a0[h][u] = sa[h * nbp + kk];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kk = (int)((w[u] >> 12 & kKbMask) << 4) + cls;
#pragma unroll
          for (int h = 0; h < NCOL; ++h) {
            const double x = __hiloint2double(__double2hiint(v[h][u]) ^ (int)(w[u] & kNeg), __double2loint(v[h][u]));
            run[h] = ((w[u] & kHead) ? a0[h][u] : run[h]) + x;
            if (w[u] & kLast) sa[h * nbp + kk] = run[h];
          }
        }
      }
    }
    if (nbk == 0 && Jn > 0) load_block(ttn, 0, Jn, nw);
    if (Jc < 0 && c < NCOL) {  // serial list (a tile whose buckets could not be balanced), ascending entry order
      const uint32_t* sl = a.words + tt * plan_tile_words(a.s);
      double* sh = sa + c * nbp;
      const double* th = tile + c * kE;
      for (int e = 0; e < -Jc; ++e) {
        const uint32_t x = __ldg(sl + e);
        if (!(x & kValid)) continue;
        const int k = (int)((x >> 12) & kKbMask);
        SKH_CHECK(k < a.nb);
        const double vv = th[x & (kE - 1)];
        sh[k] = (x & kNeg) ? sh[k] - vv : sh[k] + vv;
      }
    }
    nbar_sync(kBarCons, kNC);                                   // every add of this tile is done
    if (i + kNBuf < nitems) nbar_arrive(kBarEmpty + b, NALL);  // buffer b free (no arrival left unmatched)
    if (tt == a.ntiles - 1) {                                   // group done: its SA columns out
#pragma unroll
      for (int h = 0; h < NCOL; ++h) {
        const int64_t col = NCOL * grp + h;
        if (col >= a.ncols) continue;
        double* o = col < a.ncolSA ? a.SA + col * a.ldsa : a.Sb;
        // same k -> thread map as the zeroing above, so no barrier is needed before the next group's zeroing
        for (int k = c; k < a.nb; k += kNC) o[a.b0 + k] = a.alpha * sa[h * nbp + k];
      }
    }
    Jc = Jn;
    if (ttn == 0) grp += gridDim.x;
    tt = ttn;
  }
}

// ------------------------------------------------------------------ owner plan (once per sketch)
// One CTA per tile.  (1) count the tile's entries per local bucket k, keyed
// class-major (o = (k & 15) nkb + (k >> 4)); (2) exclusive scan; (3) place the
// entries (atomic slot claims), then sort every bucket run by entry index e =
// p s + q -- a run is tiny and the sorted result is unique, so the plan does not
// depend on the order of the claims; (4) split each class's runs over its 16
// slots (runs are never split); (5) write the words, [step j][consumer thread].
// A tile whose longest slot exceeds plan_jcap(s) steps (only for very small m)
// becomes a serial list in ascending e.
__device__ __forceinline__ int block_excl_scan_256(int v, int* tmp, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < 8 ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < 8) tmp[8 + lane] = t;
  }
  __syncthreads();
  total = tmp[15];
  const int r = (w > 0 ? tmp[8 + w - 1] : 0) + x - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) cm_plan_kernel(const int32_t* __restrict__ col_rows,
                                                      const int8_t* __restrict__ col_signs, int s, int K2, int lo,
                                                      int64_t nvalid, int b0, int nb, uint32_t* __restrict__ words,
                                                      int32_t* __restrict__ hdr, uint64_t* __restrict__ pbank) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ int tmp[16];
  __shared__ uint8_t gpos[kE];     // staging row (producer store group) of position p
  __shared__ int bnk[kE];          // its bank in that row (0xFF: not chosen yet)
  __shared__ unsigned avail[256];  // banks still free per row
  __shared__ int bnd[16][17];
  __shared__ int cstart[17];
  __shared__ int jmax;
  const int tid = threadIdx.x;
  const int64_t tt = blockIdx.x;
  const int E = kE * s;
  const int nkb = (nb + 15) >> 4;
  const int no = 16 * nkb;
  uint32_t* sorted = reinterpret_cast<uint32_t*>(smraw);        // [E]: e | kb << 15 | neg << 31
  int* off = reinterpret_cast<int*>(smraw + sizeof(uint32_t) * E);  // [no]
  for (int o = tid; o < no; o += 256) off[o] = 0;
  if (tid == 0) jmax = 0;
  for (int v = 0; v < 16; ++v) {  // producer thread tid stores its register v as row 16 v + tid / 16
    const int p = pf_rt(K2, tid, v);
    gpos[p] = (uint8_t)(16 * v + (tid >> 4));
    bnk[p] = 0xFF;
  }
  avail[tid] = 0xFFFFu;
  __syncthreads();
  auto entry = [&](int e, int& k, int& neg) {  // local bucket of entry e (-1: none in this launch)
    const int p = e / s, q = e - p * s;
    const int64_t r = tile_row(tt, p, K2, lo);
    k = -1;
    neg = 0;
    if (r < nvalid) {
      const int bk = col_rows[r * s + q] - b0;
      if ((unsigned)bk < (unsigned)nb) {
        k = bk;
        neg = col_signs[r * s + q] < 0;
      }
    }
  };
  // (1) counts
  for (int e = tid; e < E; e += 256) {
    int k, neg;
    entry(e, k, neg);
    if (k >= 0) atomicAdd(&off[(k & 15) * nkb + (k >> 4)], 1);
  }
  __syncthreads();
  // (2) exclusive scan over o: contiguous segments per thread
  const int seg = (no + 255) / 256, o0 = min(no, tid * seg), o1 = min(no, o0 + seg);
  int sum = 0;
  for (int o = o0; o < o1; ++o) sum += off[o];
  int total;
  int run = block_excl_scan_256(sum, tmp, total);
  for (int o = o0; o < o1; ++o) {
    const int cnt = off[o];
    off[o] = run;
    run += cnt;
  }
  __syncthreads();
  if (tid < 16) cstart[tid] = off[tid * nkb];
  if (tid == 0) cstart[16] = total;
  __syncthreads();
  // (3) place (off[o] advances to the end of run o), then sort runs by e
  for (int e = tid; e < E; e += 256) {
    int k, neg;
    entry(e, k, neg);
    if (k >= 0) {
      const int pos = atomicAdd(&off[(k & 15) * nkb + (k >> 4)], 1);
      SKH_CHECK(pos >= 0 && pos < E);
      sorted[pos] = (uint32_t)e | ((uint32_t)(k >> 4) << 15) | ((uint32_t)neg << 31);
    }
  }
  __syncthreads();
  for (int o = tid; o < no; o += 256) {
    const int r0 = o == 0 ? 0 : off[o - 1], r1 = off[o];
    for (int i = r0 + 1; i < r1; ++i) {  // insertion sort by e (low 15 bits)
      const uint32_t x = sorted[i];
      int j = i - 1;
      while (j >= r0 && (sorted[j] & 0x7FFFu) > (x & 0x7FFFu)) {
        sorted[j + 1] = sorted[j];
        --j;
      }
      sorted[j + 1] = x;
    }
  }
  __syncthreads();
  // (4) slots: thread (cl, u) starts at the first run start at or after u T
  const int cl = tid & 15, u = tid >> 4;
  const int cs = cstart[cl], C = cstart[cl + 1] - cs;
  const int T = (C + 15) / 16;
  {
    int i = min(u * T, C);
    while (i > 0 && i < C && ((sorted[cs + i] >> 15) & 0xFFFFu) == ((sorted[cs + i - 1] >> 15) & 0xFFFFu)) ++i;
    bnd[cl][u] = i;
    if (u == 15) bnd[cl][16] = C;
  }
  __syncthreads();
  const int i0 = bnd[cl][u], cnt = bnd[cl][u + 1] - i0;
  atomicMax(&jmax, cnt);
  __syncthreads();
  const int J8 = (jmax + 3) & ~3;  // steps: a multiple of 4 (one uint4 of words)
  uint32_t* out = words + tt * plan_tile_words(s);
  // claim a free bank of row g for position p (unique per row), preferring the
  // banks in `want`; returns the bank
  // (s = 1: every position is claimed once, and a row never has more claims
  // than its 16 banks)
  auto claim = [&](int p, unsigned want) {
    const int g = gpos[p];
    for (;;) {
      const unsigned av = *(volatile unsigned*)&avail[g];
      unsigned m = av & want;
      if (!m) m = av;
      const int b = __ffs(m) - 1;
      if ((atomicAnd(&avail[g], ~(1u << b)) >> b) & 1u) {
        bnk[p] = b;
        return b;
      }
    }
  };
  auto slot_of = [&](int p) { return 16 * (int)gpos[p] + (int)bnk[p]; };
  // the staging colouring is built for s = 1 (one entry per position: each
  // position claims one bank of its row once); s > 1 and serial tiles keep the
  // natural banks (bank = producer lane)
  const bool colour = s == 1 && J8 <= plan_jcap(s);
  if (!colour) {
    for (int v = 0; v < 16; ++v) bnk[pf_rt(K2, tid, v)] = tid & 15;
    __syncthreads();
  }
  if (J8 > plan_jcap(s)) {  // serial list in ascending e
    for (int e = tid; e < E; e += 256) {
      int k, neg;
      entry(e, k, neg);
      out[e] = k < 0 ? 0u : ((uint32_t)slot_of(e / s) | ((uint32_t)k << 12) | kValid | ((uint32_t)neg << 31));
    }
    uint64_t pb = 0;
    for (int v = 0; v < 16; ++v) pb |= (uint64_t)(tid & 15) << (4 * v);
    pbank[tt * kNP + tid] = pb;
    if (tid == 0) hdr[tt] = -E;
    return;
  }
  // (5) words: the thread's runs in order, each run's entries in ascending e,
  // flagged head (first of its bucket) and last.  (Reordering the runs per step
  // so a half-warp reads distinct banks was measured: a greedy leaves ~1.95
  // wavefronts per half-warp step.)  Instead the STAGING LAYOUT is coloured: a
  // position's slot is (producer store row, bank) and, step by step, the 16
  // lanes of a consumer half-warp claim distinct banks, each from the free banks
  // of its position's row -- a bipartite edge colouring (rows x half-warp steps,
  // 16 colours, which exists by Konig's theorem); the greedy claim falls back to
  // any free bank of the row, a rare 2-way conflict.
  const uint32_t* mine = sorted + cs + i0;
  const int c = 32 * (u >> 1) + 16 * (u & 1) + cl;  // consumer thread of (class cl, slot u)
  for (int j = 0; j < J8; ++j) {
    uint32_t wd = 0;
    int p = -1;
    if (j < cnt) {
      const uint32_t x = mine[j];
      const uint32_t kb = (x >> 15) & 0xFFFFu;
      const bool head = j == 0 || ((mine[j - 1] >> 15) & 0xFFFFu) != kb;
      const bool last = j + 1 == cnt || ((mine[j + 1] >> 15) & 0xFFFFu) != kb;
      p = (int)(x & 0x7FFFu) / s;
      wd = (kb << 12) | (x & 0x80000000u) | (head ? kHead : 0u) | (last ? kLast : 0u);
    }
    if (colour) {
      unsigned used = 0;  // banks taken by the lanes before, this step, this half-warp
      for (int L = 0; L < 16; ++L) {
        if (cl == L && p >= 0) used |= 1u << claim(p, ~used);
        used = __shfl_sync(0xffffffffu, used, (tid & 16) + L);
      }
    }
    if (p >= 0) wd |= (uint32_t)slot_of(p);
    out[plan_index(j, c)] = wd;
  }
  __syncthreads();
  if (colour)
    for (int p = tid; p < kE; p += 256)  // positions no entry reads: any free bank of their row
      if (bnk[p] == 0xFF) claim(p, 0xFFFFu);
  __syncthreads();
  uint64_t pb = 0;  // producer thread tid's banks, 4 bits per register
  for (int v = 0; v < 16; ++v) pb |= (uint64_t)bnk[pf_rt(K2, tid, v)] << (4 * v);
  pbank[tt * kNP + tid] = pb;
  if (tid == 0) hdr[tt] = J8;
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


template <int K2>
int launch_mid_t(const PassArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)kE * 8;
  auto* f = cm_mid_kernel<K2>;
  int rc = set_smem(f, smem);
  if (rc) return rc;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, 256, smem);
  const int64_t grid = std::min<int64_t>(a.ncols * a.ntiles, (int64_t)num_sms() * std::max(per_sm, 1));
  if (grid < 1) return SKH_OK;
  f<<<(unsigned)grid, 256, smem, st>>>(a);
  note_launch();
  return check_launch("cm_mid");
}

template <int K2, int NCOL>
int launch_gather_nt(const PassArgs& a, cudaStream_t st) {
  const size_t smem = gather_smem_bytes(a.nb, NCOL);
  auto* f = cm_gather_kernel<K2, NCOL>;
  int rc = set_smem(f, smem);
  if (rc) return rc;
  const int64_t grid = std::min<int64_t>((a.ncols + NCOL - 1) / NCOL, (int64_t)num_sms());
  if (grid < 1) return SKH_OK;
  f<<<(unsigned)grid, kNP + kNC, smem, st>>>(a);
  note_launch();
  return check_launch("cm_gather");
}

// Two columns per CTA where both sketches and staging pairs fit on chip (small
// m) and there are columns for every SM twice over (SKH_CM_NCOL=1 turns it off)
template <int K2>
int launch_gather_t(const PassArgs& a, cudaStream_t st) {
  static const bool two = [] {
    const char* e = getenv("SKH_CM_NCOL");
    return !(e && atoi(e) == 1);
  }();
  if (two && gather_smem_bytes(a.nb, 2) <= (size_t)227 * 1024 && a.ncols >= 2 * (int64_t)num_sms())
    return launch_gather_nt<K2, 2>(a, st);
  return launch_gather_nt<K2, 1>(a, st);
}

size_t plan_range_bytes(int64_t ntiles, int s) {
  return align_up(sizeof(uint32_t) * (size_t)ntiles * (size_t)plan_tile_words(s)) +
         align_up(sizeof(int32_t) * (size_t)ntiles) + align_up(sizeof(uint64_t) * (size_t)ntiles * kNP);
}
// [words][hdr][pbank] of one bucket range
const int32_t* plan_hdr(const char* base, int64_t ntiles, int s) {
  return reinterpret_cast<const int32_t*>(base + align_up(sizeof(uint32_t) * (size_t)ntiles * plan_tile_words(s)));
}
const uint64_t* plan_pbank(const char* base, int64_t ntiles, int s) {
  return reinterpret_cast<const uint64_t*>(base + align_up(sizeof(uint32_t) * (size_t)ntiles * plan_tile_words(s)) +
                                           align_up(sizeof(int32_t) * (size_t)ntiles));
}

}  // namespace

// Largest bucket range one fused-pass launch accumulates on chip (one CTA per
// SM: the staged tiles + the sketch column in shared memory).
int cm_max_buckets(int s) {
  if (s < 1 || s > 8) return 0;
  const size_t avail = 227 * 1024 - (size_t)kNBuf * kE * 8;                // gather: staged tiles + SA
  const size_t avail_plan = 227 * 1024 - (size_t)4 * kE * s - 16 - 24 * 1024;  // plan: entries, counters, colouring
  return (int)(std::min(avail / 8, avail_plan / 4) & ~(size_t)15);
}

// Pass 1 of columns of 2^L rows: bits [0, min(L, 13)).
// reserve_sms: SMs the persistent kernel leaves free (for side-stream work that
// runs beside it)
int launch_cm_pass1(uint64_t seed, const double* X, int64_t ldx, int64_t ncolX, const double* xb, double* Y,
                    int64_t ldy, int64_t nvalid, int L, int apply_diag, int64_t row0, cudaStream_t st,
                    int reserve_sms) {
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
  static const bool teams = [] {  // SKH_P1_TEAMS=0: the one-team persistent kernel
    const char* e = getenv("SKH_P1_TEAMS");
    return !(e && e[0] == '0');
  }();
  if (teams && vec && nvalid >= ((int64_t)1 << L)) {  // every chunk full: two teams per CTA
    const size_t smem = (size_t)kP1Ring * 65536;
    const int64_t total = grid;
    const int64_t g = std::min<int64_t>(total, (int64_t)std::max(1, num_sms() - std::max(0, reserve_sms)));
    int rc = apply_diag ? set_smem(cm_pass1t_kernel<true>, smem) : set_smem(cm_pass1t_kernel<false>, smem);
    if (rc) return rc;
    if (apply_diag)
      cm_pass1t_kernel<true><<<(unsigned)g, 512, smem, st>>>(X, ldx, ncolX, xb, Y, ldy, nchunks, total, dkey, row0);
    else
      cm_pass1t_kernel<false><<<(unsigned)g, 512, smem, st>>>(X, ldx, ncolX, xb, Y, ldy, nchunks, total, dkey, row0);
    note_launch();
    return check_launch("cm_pass1t");
  }
  if (vec && nvalid >= ((int64_t)1 << L)) {  // every chunk full: the persistent double-buffered kernel
    const size_t smem = (size_t)kP1Ring * 65536;
    const int64_t total = grid;
    const int64_t g = std::min<int64_t>(total, (int64_t)std::max(1, num_sms() - std::max(0, reserve_sms)));
    int rc = apply_diag ? set_smem(cm_pass1p_kernel<true>, smem) : set_smem(cm_pass1p_kernel<false>, smem);
    if (rc) return rc;
    if (apply_diag)
      cm_pass1p_kernel<true><<<(unsigned)g, 256, smem, st>>>(X, ldx, ncolX, xb, Y, ldy, nchunks, total, dkey, row0);
    else
      cm_pass1p_kernel<false><<<(unsigned)g, 256, smem, st>>>(X, ldx, ncolX, xb, Y, ldy, nchunks, total, dkey, row0);
    note_launch();
    return check_launch("cm_pass1p");
  }
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
    case 1: return launch_mid_t<1>(a, st);
    case 2: return launch_mid_t<2>(a, st);
    case 3: return launch_mid_t<3>(a, st);
    case 4: return launch_mid_t<4>(a, st);
    case 5: return launch_mid_t<5>(a, st);
    case 6: return launch_mid_t<6>(a, st);
    case 7: return launch_mid_t<7>(a, st);
    case 8: return launch_mid_t<8>(a, st);
    default: set_error("cm mid pass: K2 = %d", K2); return SKH_EINVAL;
  }
}

// Owner plans of the final pass, one per bucket range of at most
// cm_max_buckets(s) buckets: [range][tile][plan_jcap(s)][kNC] words + [range][tile] steps.
size_t cm_lists_bytes(int64_t ntiles, int s, int64_t m) {
  const int cap = cm_max_buckets(s);
  const int64_t nr = cap > 0 ? (m + cap - 1) / cap : 1;
  return (size_t)nr * plan_range_bytes(ntiles, s);
}

// Plans of the final pass (bits [lo, lo + K2), or K2 = 0 row blocks).
int launch_cm_lists(const int32_t* col_rows, const int8_t* col_signs, int s, int64_t m, int K2, int lo,
                    int64_t nvalid, int64_t ntiles, void* lists_ws, cudaStream_t st) {
  const int cap = cm_max_buckets(s);
  if (cap < 1) {
    set_error("column-major gather supports s <= 8");
    return SKH_EINVAL;
  }
  char* base = static_cast<char*>(lists_ws);
  for (int64_t b0 = 0; b0 < m; b0 += cap) {
    const int nb = (int)std::min<int64_t>(cap, m - b0);
    uint32_t* words = reinterpret_cast<uint32_t*>(base);
    int32_t* hdr = const_cast<int32_t*>(plan_hdr(base, ntiles, s));
    uint64_t* pbank = const_cast<uint64_t*>(plan_pbank(base, ntiles, s));
    const size_t smem = plan_smem_bytes(s, nb);
    // the kernel also holds ~22 KB of static shared memory (the staging colouring)
    if (cudaFuncSetAttribute(cm_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      set_error("cm plan: %zu bytes of shared memory", smem);
      return SKH_ECUDA;
    }
    int rc;
    cm_plan_kernel<<<(unsigned)ntiles, 256, smem, st>>>(col_rows, col_signs, s, K2, lo, nvalid, (int)b0, nb, words,
                                                         hdr, pbank);
    note_launch();
    if ((rc = check_launch("cm_plan"))) return rc;
    base += plan_range_bytes(ntiles, s);
  }
  return SKH_OK;
}

// Final pass: bits [lo, lo + K2) then the owner-planned gather into SA columns
// (one launch per bucket range).
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
  const char* base = static_cast<const char*>(lists_ws);
  for (int64_t b0 = 0; b0 < m; b0 += cap) {
    a.b0 = (int)b0;
    a.nb = (int)std::min<int64_t>(cap, m - b0);
    a.words = reinterpret_cast<const uint32_t*>(base);
    a.hdr = plan_hdr(base, ntiles, s);
    a.pbank = plan_pbank(base, ntiles, s);
    int rc;
    switch (K2) {
      case 0: rc = launch_gather_t<0>(a, st); break;
      case 1: rc = launch_gather_t<1>(a, st); break;
      case 2: rc = launch_gather_t<2>(a, st); break;
      case 3: rc = launch_gather_t<3>(a, st); break;
      case 4: rc = launch_gather_t<4>(a, st); break;
      case 5: rc = launch_gather_t<5>(a, st); break;
      case 6: rc = launch_gather_t<6>(a, st); break;
      case 7: rc = launch_gather_t<7>(a, st); break;
      case 8: rc = launch_gather_t<8>(a, st); break;
      default: set_error("cm gather: K2 = %d", K2); return SKH_EINVAL;
    }
    if (rc) return rc;
    base += plan_range_bytes(ntiles, s);
  }
  return SKH_OK;
}

}  // namespace skh
