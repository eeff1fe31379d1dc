// fwht_fused.cu -- wide FWHT passes (K = 7 + KB bits, KB = 1..4) with ONE HBM
// read and ONE HBM write per element (Def. def::HRHT, PAPER.md L790-801;
// DESIGN.md §5).  A unit (one butterfly group of 2^K rows x 64 columns, <= 1 MiB)
// is processed as 2^KB A-tasks (the low 7 bits of 128 rows: registers + one smem
// redistribution, D fused in the first pass) followed by 2^KB B-tasks (the KB
// high bits for 128/2^KB low indices: registers only), the B-tasks reading the
// A results back from L2.
//
// Schedule: a cooperative (co-resident) grid; CTA c runs tasks c, c+G, c+2G, ...
// in order, no task counter and no per-task fetch barrier.  Tasks are ordered
// A_0 .. A_{lag-1}, then (A_{lag+i}, B_i) blocks, then the last B's, so a B-task's
// A-tasks precede it by ~2*lag*2^KB tasks (several scheduling rounds) and are
// normally done; the B-task's thread 0 still acquires the unit's counter (the
// A-tasks release it after their stores) before the CTA reads.  Every
// dependency has a smaller task index and all CTAs are resident, so the lowest
// unfinished task can always run: no deadlock.  Stage order stays low -> high.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kT = 256;
constexpr int kCP = 32;  // 64 columns

__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

template <int NB>
__device__ __forceinline__ void decode(int64_t t, int64_t nunits, int64_t lag, int64_t& u, int& sub, bool& isA) {
  const int64_t k = t / NB;
  sub = (int)(t % NB);
  if (k < lag) {
    u = k;
    isA = true;
  } else if (k < lag + 2 * (nunits - lag)) {
    const int64_t j = k - lag;
    isA = (j & 1) == 0;
    u = isA ? lag + j / 2 : j / 2;
  } else {
    isA = false;
    u = (nunits - lag) + (k - lag - 2 * (nunits - lag));
  }
}

template <int KB, bool DIAG>
__global__ void __launch_bounds__(kT, 2) fwht_fused2_kernel(
    const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy, int64_t nvalid, int lo,
    int64_t d, int64_t ntc, int64_t g_begin, int64_t nunits, int64_t lag, uint32_t* __restrict__ done,
    uint64_t dkey, int64_t row0, double alpha) {
  constexpr int K = 7 + KB;
  constexpr int NB = 1 << KB;
  constexpr int NA = 16 / NB;  // low indices per thread in a B-task
  extern __shared__ double2 tile[];  // [128][kCP]
  const int cp = threadIdx.x % kCP, rs = threadIdx.x / kCP;  // rs 0..7
  const int64_t ntasks = 2 * nunits * NB;
  for (int64_t t = blockIdx.x; t < ntasks; t += gridDim.x) {
    int64_t u;
    int sub;
    bool isA;
    decode<NB>(t, nunits, lag, u, sub, isA);
    const int64_t g = g_begin + u / ntc;
    const int64_t tc = u % ntc;
    const int64_t low = g & (((int64_t)1 << lo) - 1);
    const int64_t hi = g >> lo;
    const int64_t rbase = (hi << (lo + K)) + low;
    const int64_t c = tc * (2 * kCP) + 2 * cp;
    const bool cv = c < d;
    double2 x[16];
    if (isA) {
      // rows mid = 128*sub + rs*16 + v (phase 0: 16 consecutive mids)
      const int64_t r0 = rbase + ((int64_t)(128 * sub + rs * 16) << lo);
      {
        const int64_t left = nvalid - r0;
        const int nv =
            left <= 0 ? 0 : (left >= ((int64_t)16 << lo) ? 16 : (int)((left + ((int64_t)1 << lo) - 1) >> lo));
        const double2* p = reinterpret_cast<const double2*>(X + r0 * ldx + c);
        const int64_t step = (ldx << lo) / 2;
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          x[v] = make_double2(0.0, 0.0);
          if (cv && v < nv) x[v] = __ldg(p + v * step);
        }
      }
      if (DIAG) {
        uint32_t negmask = 0;
        if (lo == 0) {
          const int64_t g0 = row0 + r0;
          const uint64_t wa = stream_u(dkey, (uint64_t)(g0 >> 6));
          const int sh = (int)(g0 & 63);
          uint64_t win = wa >> sh;
          if (sh > 48) win |= stream_u(dkey, (uint64_t)((g0 >> 6) + 1)) << (64 - sh);
          const int64_t left = nvalid - r0;
          const uint32_t vmask = left >= 16 ? 0xFFFFu : (left <= 0 ? 0u : ((1u << left) - 1u));
          negmask = (uint32_t)(win & 0xFFFFull) & vmask;
        } else {
#pragma unroll
          for (int v = 0; v < 16; ++v) {
            const int64_t r = r0 + ((int64_t)v << lo);
            const int64_t gr = row0 + r;
            if (r < nvalid) negmask |= (uint32_t)((stream_u(dkey, (uint64_t)(gr >> 6)) >> (gr & 63)) & 1ull) << v;
          }
        }
#pragma unroll
        for (int v = 0; v < 16; ++v)
          if ((negmask >> v) & 1u) x[v] = make_double2(-x[v].x, -x[v].y);
      }
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        const int h = 1 << bb;
#pragma unroll
        for (int v = 0; v < 16; ++v)
          if (!(v & h)) {
            const double2 a = x[v], b = x[v + h];
            x[v] = add2(a, b);
            x[v + h] = sub2(a, b);
          }
      }
      // redistribute: each thread rewrites the slots it owns (rows rs*16 + v), then
      // reads phase-1 rows 2*rs + g + 16*j (v = 8g + j); the previous task's
      // readers are past the publish/acquire barrier, so one barrier suffices
#pragma unroll
      for (int v = 0; v < 16; ++v) tile[(rs * 16 + v) * kCP + cp] = x[v];
      __syncthreads();
#pragma unroll
      for (int v = 0; v < 16; ++v) x[v] = tile[(2 * rs + (v >> 3) + 16 * (v & 7)) * kCP + cp];
#pragma unroll
      for (int bb = 0; bb < 3; ++bb) {
        const int h = 1 << bb;
#pragma unroll
        for (int v = 0; v < 16; ++v)
          if (!(v & h)) {
            const double2 a = x[v], b = x[v + h];
            x[v] = add2(a, b);
            x[v + h] = sub2(a, b);
          }
      }
      if (cv) {
        double2* q = reinterpret_cast<double2*>(Y + (rbase + ((int64_t)(128 * sub + 2 * rs) << lo)) * ldy + c);
        const int64_t sg = (ldy << lo) / 2, sj = (ldy << (lo + 4)) / 2;
#pragma unroll
        for (int v = 0; v < 16; ++v) q[(v >> 3) * sg + (v & 7) * sj] = x[v];
      }
      __syncthreads();  // all stores of this A-task issued; tile free for the next task
      if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(done + u) : "memory");
    } else {
      if (threadIdx.x == 0) {
        unsigned ns = 32;
        for (;;) {
          uint32_t v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + u) : "memory");
          if (v >= (uint32_t)NB) break;
          __nanosleep(ns);
          if (ns < 1024) ns *= 2;
        }
      }
      __syncthreads();
      // value v = aa*NB + b: low index a = sub*(128/NB) + rs*NA + aa, high bits b
      const int a0 = sub * (128 / NB) + rs * NA;
      double2* q = reinterpret_cast<double2*>(Y + (rbase + ((int64_t)a0 << lo)) * ldy + c);
      const int64_t sa = (ldy << lo) / 2, sb = (ldy << (lo + 7)) / 2;
#pragma unroll
      for (int v = 0; v < 16; ++v)
        x[v] = cv ? __ldcg(q + (v / NB) * sa + (v % NB) * sb) : make_double2(0.0, 0.0);
#pragma unroll
      for (int bb = 0; bb < KB; ++bb) {
        const int h = 1 << bb;
#pragma unroll
        for (int v = 0; v < 16; ++v)
          if (!(v & h)) {
            const double2 a = x[v], b = x[v + h];
            x[v] = add2(a, b);
            x[v + h] = sub2(a, b);
          }
      }
      if (cv) {
#pragma unroll
        for (int v = 0; v < 16; ++v)
          q[(v / NB) * sa + (v % NB) * sb] = make_double2(alpha * x[v].x, alpha * x[v].y);
      }
    }
  }
}

int sm_count_fused() {
  static int v = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}

template <int KB, bool DIAG>
int launch_fused2(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nvalid, int lo, int64_t d,
                  int64_t g_begin, int64_t g_count, uint32_t* counters, uint64_t dkey, int64_t row0, double alpha,
                  cudaStream_t st) {
  constexpr int NB = 1 << KB;
  const size_t smem = 128 * kCP * sizeof(double2);
  auto kern = fwht_fused2_kernel<KB, DIAG>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kT, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t ntc = (d + 2 * kCP - 1) / (2 * kCP);
  int64_t nunits = g_count * ntc;
  const int64_t ntasks = 2 * nunits * NB;
  const int64_t grid = std::min<int64_t>((int64_t)per_sm * sm_count_fused(), ntasks);
  int64_t lag = std::max<int64_t>(1, (2 * grid + 2 * NB - 1) / (2 * NB));
  if (lag > nunits) lag = nunits;
  uint32_t* done = counters + 64;
  cudaMemsetAsync(done, 0, sizeof(uint32_t) * (size_t)nunits, st);
  void* args[] = {(void*)&X,       (void*)&ldx,    (void*)&Y,   (void*)&ldy,  (void*)&nvalid, (void*)&lo,
                  (void*)&d,       (void*)&ntc,    (void*)&g_begin, (void*)&nunits, (void*)&lag, (void*)&done,
                  (void*)&dkey,    (void*)&row0,   (void*)&alpha};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)grid), dim3(kT), args, smem, st);
  note_launch();
  if (e != cudaSuccess) {
    set_error("fwht_fused2 launch: %s", cudaGetErrorString(e));
    return SKH_ECUDA;
  }
  return check_launch("fwht_fused2");
}

}  // namespace

// K in [8, 11]; X/Y 16-byte aligned, even ld, even d.
int launch_fused2_k(int K, bool diag, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nvalid, int lo,
                    int64_t d, int64_t g_begin, int64_t g_count, uint32_t* counters, uint64_t dkey, int64_t row0,
                    double alpha, cudaStream_t st) {
#define SKH_F2(KB)                                                                                              \
  return diag ? launch_fused2<KB, true>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, counters, dkey, row0,  \
                                        alpha, st)                                                              \
              : launch_fused2<KB, false>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, counters, dkey, row0, \
                                         alpha, st)
  switch (K) {
    case 8: SKH_F2(1);
    case 9: SKH_F2(2);
    case 10: SKH_F2(3);
    case 11: SKH_F2(4);
    default: break;
  }
#undef SKH_F2
  set_error("internal: bad fused pass width %d", K);
  return SKH_EINVAL;
}

}  // namespace skh
