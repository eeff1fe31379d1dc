// fwht_pipe.cu -- the HBM-pass kernel of R3/R4 (Def. def::HRHT, PAPER.md
// L790-801): a persistent, warp-specialised, bulk-copy-fed
// pipeline for passes of K = 7 + KB bits (KB = 0..4).
//
//  * One CTA per SM: a producer warp and 8 consumer warps, 3 shared-memory
//    stages of 64 KiB (128 rows x 64 columns of fp64).
//  * The producer claims tasks from a global counter and fills a stage with 128
//    row segments of 512 B through cp.async.bulk (the TMA engine) completing on
//    the stage's mbarrier, so two stages of loads are always in flight without
//    holding registers.
//  * A unit is a butterfly group of 2^K rows (stride 2^lo) x 64 columns.  Its
//    A-tasks (2^KB of them) each transform 128 rows on the low 7 mid bits
//    (registers + one smem redistribution, D fused in the first pass) and store
//    them; its B-tasks (2^KB) run the KB high mid bits for 128 / 2^KB low mids,
//    reading the A-task results back from L2 (a unit is at most 1 MiB and only
//    ~LAG units are in flight, so they are still there): one HBM read and one
//    HBM write per element for all K bits.
//  * A-tasks publish with a CTA barrier + one gpu-scope release; the producer of
//    a B-task acquires the unit's counter and issues fence.proxy.async before its
//    bulk copies.  Tasks are claimed in an order where every dependency has a
//    smaller index and only producers wait, so the schedule cannot deadlock.
//  * Stage order is low bit -> high bit everywhere: results are bit-identical to
//    the oracle (R9).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kStages = 3;
constexpr int kRows = 128;  // rows per task
constexpr int kCP = 32;     // column pairs per task (64 columns, 512 B per row)
constexpr int kConsumers = 256;
constexpr int kThreads = kConsumers + 32;
constexpr size_t kStageBytes = (size_t)kRows * kCP * sizeof(double2);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }

__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// 7-bit tile mapping (same as fwht.cu mid_of<7, P>): phase 0 = 16 consecutive mids.
__device__ __forceinline__ int mid7_p0(int rs, int v) { return rs * 16 + v; }
__device__ __forceinline__ int mid7_p1(int rs, int v) {
  // phase 1 covers bits 4..6: J = 8 values of bits 4..6, NG = 2 groups
  const int g = v >> 3, j = v & 7;
  const int other = rs * 2 + g;  // 4 low bits
  return other | (j << 4);
}

struct Task {
  int64_t u;
  int sub;
  bool isA;
};

// Claim order: blocks of NB tasks; A_0..A_{lag-1}, then (A_{lag+i}, B_i) pairs, then the last B's.
template <int NB, bool FUSED>
__device__ __forceinline__ Task decode(int64_t t, int64_t nunits, int64_t lag) {
  Task r;
  if (!FUSED) {
    r.u = t;
    r.sub = 0;
    r.isA = true;
    return r;
  }
  const int64_t k = t / NB;
  r.sub = (int)(t % NB);
  if (k < lag) {
    r.u = k;
    r.isA = true;
  } else if (k < lag + 2 * (nunits - lag)) {
    const int64_t j = k - lag;
    r.isA = (j & 1) == 0;
    r.u = r.isA ? lag + j / 2 : j / 2;
  } else {
    r.isA = false;
    r.u = (nunits - lag) + (k - lag - 2 * (nunits - lag));
  }
  return r;
}

template <int KB, bool DIAG>
__global__ void __launch_bounds__(kThreads, 1) fwht_pipe_kernel(
    const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy, int64_t nvalid, int lo,
    int64_t d, int64_t ntc, int64_t g_begin, int64_t nunits, int64_t lag, uint32_t* __restrict__ counters,
    uint64_t dkey, int64_t row0, double alpha) {
  constexpr int K = 7 + KB;
  constexpr int NB = 1 << KB;
  constexpr bool FUSED = KB > 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* stages = reinterpret_cast<double2*>(smem_raw);
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ int64_t task_of[kStages];
  uint32_t* task_ctr = counters;
  uint32_t* done = counters + 64;
  const int64_t ntasks = FUSED ? 2 * nunits * NB : nunits;
  const int64_t lagc = lag < nunits ? lag : nunits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kConsumers / 32) {
    // ------------------------------------------------------------ producer warp
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      int64_t t = 0;
      if (lane == 0) t = (int64_t)atomicAdd(task_ctr, 1u);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntasks) {
        if (lane == 0) {
          mbar_wait(&empty_bar[stage], phase ^ 1u);
          task_of[stage] = -1;
          mbar_arrive(&full_bar[stage]);
        }
        break;
      }
      const Task tk = decode<NB, FUSED>(t, nunits, lagc);
      if (FUSED && !tk.isA) {
        if (lane == 0) {
          unsigned ns = 64;
          for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + tk.u) : "memory");
            if (v >= (uint32_t)NB) break;
            __nanosleep(ns);
            if (ns < 2048) ns *= 2;
          }
        }
        __syncwarp();
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      const int64_t g = g_begin + tk.u / ntc;
      const int64_t tc = tk.u % ntc;
      const int64_t low = g & (((int64_t)1 << lo) - 1);
      const int64_t hi = g >> lo;
      const int64_t rbase = (hi << (lo + K)) + low;
      const int64_t c0 = tc * (2 * kCP);
      const uint32_t seg = (uint32_t)(min((int64_t)(2 * kCP), d - c0) * (int64_t)sizeof(double));
      const double* src = tk.isA ? X : Y;
      const int64_t lds = tk.isA ? ldx : ldy;
      const int64_t nv = tk.isA ? nvalid : ((int64_t)1 << 62);
      // rows j = lane*4 .. lane*4+3 of this task
      int64_t rows[4];
      int nval = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = lane * 4 + q;
        int mid;
        if (tk.isA) {
          mid = j + kRows * tk.sub;
        } else {
          const int a = tk.sub * (kRows / NB) + j / NB, b = j % NB;
          mid = a + kRows * b;
        }
        rows[q] = rbase + ((int64_t)mid << lo);
        nval += rows[q] < nv;
      }
      int tot = nval;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      double2* sb = stages + (size_t)stage * kRows * kCP;
      if (lane == 0) {
        mbar_wait(&empty_bar[stage], phase ^ 1u);
        task_of[stage] = t;
        if (tot > 0)
          mbar_expect_tx(&full_bar[stage], (uint32_t)tot * seg);
        else
          mbar_arrive(&full_bar[stage]);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (rows[q] < nv) bulk_g2s(sb + (lane * 4 + q) * kCP, src + rows[q] * lds + c0, seg, &full_bar[stage]);
      }
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1u;
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int cp = threadIdx.x % kCP, rs = threadIdx.x / kCP;  // rs in 0..7
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    mbar_wait(&full_bar[stage], phase);
    const int64_t t = task_of[stage];
    if (t < 0) break;
    const Task tk = decode<NB, FUSED>(t, nunits, lagc);
    const int64_t g = g_begin + tk.u / ntc;
    const int64_t tc = tk.u % ntc;
    const int64_t low = g & (((int64_t)1 << lo) - 1);
    const int64_t hi = g >> lo;
    const int64_t rbase = (hi << (lo + K)) + low;
    const int64_t c = tc * (2 * kCP) + 2 * cp;
    const bool cv = c < d;
    double2* sb = stages + (size_t)stage * kRows * kCP;
    double2 x[16];
    if (tk.isA) {
      const int64_t rb = rbase + ((int64_t)(kRows * tk.sub) << lo);
      uint32_t negmask = 0;
      if (DIAG) {
        if (lo == 0) {
          const int64_t g0 = row0 + rb + mid7_p0(rs, 0);
          const uint64_t wa = stream_u(dkey, (uint64_t)(g0 >> 6)), wb = stream_u(dkey, (uint64_t)((g0 + 15) >> 6));
#pragma unroll
          for (int v = 0; v < 16; ++v) {
            const int64_t gr = g0 + v;
            const uint64_t w = ((gr >> 6) == (g0 >> 6)) ? wa : wb;
            if (gr - row0 < nvalid) negmask |= (uint32_t)((w >> (gr & 63)) & 1ull) << v;
          }
        } else {
#pragma unroll
          for (int v = 0; v < 16; ++v) {
            const int64_t r = rb + ((int64_t)mid7_p0(rs, v) << lo);
            const int64_t gr = row0 + r;
            if (r < nvalid) negmask |= (uint32_t)((stream_u(dkey, (uint64_t)(gr >> 6)) >> (gr & 63)) & 1ull) << v;
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 16; ++v) {
        const int64_t r = rb + ((int64_t)mid7_p0(rs, v) << lo);
        x[v] = (cv && r < nvalid) ? sb[mid7_p0(rs, v) * kCP + cp] : make_double2(0.0, 0.0);
      }
      if (DIAG) {
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
      // redistribute through the stage: each thread rewrites exactly the slots it
      // read, so only the read-after-write needs a barrier
#pragma unroll
      for (int v = 0; v < 16; ++v) sb[mid7_p0(rs, v) * kCP + cp] = x[v];
      consumer_sync();
#pragma unroll
      for (int v = 0; v < 16; ++v) x[v] = sb[mid7_p1(rs, v) * kCP + cp];
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
      const double sc = FUSED ? 1.0 : alpha;
      if (cv) {
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const int64_t r = rb + ((int64_t)mid7_p1(rs, v) << lo);
          *reinterpret_cast<double2*>(Y + r * ldy + c) = make_double2(sc * x[v].x, sc * x[v].y);
        }
      }
      // the stage's generic-proxy writes must precede its next bulk refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (FUSED) {
        consumer_sync();  // all stores of this A-task issued
        if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(done + tk.u) : "memory");
      }
    } else {
      // rows j = rs*16 + v, v = aa*NB + b: low mid a = sub*(128/NB) + rs*(16/NB) + aa, high bits b
#pragma unroll
      for (int v = 0; v < 16; ++v) x[v] = cv ? sb[(rs * 16 + v) * kCP + cp] : make_double2(0.0, 0.0);
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
        for (int v = 0; v < 16; ++v) {
          const int aa = v / NB, b = v % NB;
          const int a = tk.sub * (kRows / NB) + rs * (16 / NB) + aa;
          const int64_t r = rbase + ((int64_t)(a + kRows * b) << lo);
          *reinterpret_cast<double2*>(Y + r * ldy + c) = make_double2(alpha * x[v].x, alpha * x[v].y);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[stage]);
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1u;
    }
  }
}

int sm_count_pipe() {
  static int v = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}

template <int KB, bool DIAG>
int launch_pipe(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nvalid, int lo, int64_t d,
                int64_t g_begin, int64_t g_count, uint32_t* counters, uint64_t dkey, int64_t row0, double alpha,
                cudaStream_t st) {
  constexpr int NB = 1 << KB;
  const size_t smem = kStages * kStageBytes;
  auto kern = fwht_pipe_kernel<KB, DIAG>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntc = (d + 2 * kCP - 1) / (2 * kCP);
  const int64_t nunits = g_count * ntc;
  const int64_t ntasks = KB > 0 ? 2 * nunits * NB : nunits;
  const int64_t resident = sm_count_pipe();
  const int64_t lag = std::max<int64_t>(2, (resident * (kStages + 1) + 2 * NB - 1) / (2 * NB));
  const int64_t grid = std::min<int64_t>(resident, std::max<int64_t>(1, ntasks));
  cudaMemsetAsync(counters, 0, sizeof(uint32_t) * (size_t)(64 + (KB > 0 ? nunits : 0)), st);
  kern<<<(unsigned)grid, kThreads, smem, st>>>(X, ldx, Y, ldy, nvalid, lo, d, ntc, g_begin, nunits, lag, counters,
                                               dkey, row0, alpha);
  note_launch();
  return check_launch("fwht_pipe");
}

}  // namespace

// K in [7, 11] (KB = K - 7); X/Y 16-byte aligned, even ld, even d.
int launch_pipe_k(int K, bool diag, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t nvalid, int lo,
                  int64_t d, int64_t g_begin, int64_t g_count, uint32_t* counters, uint64_t dkey, int64_t row0,
                  double alpha, cudaStream_t st) {
#define SKH_PIPE(KB)                                                                                            \
  return diag ? launch_pipe<KB, true>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, counters, dkey, row0,    \
                                      alpha, st)                                                                \
              : launch_pipe<KB, false>(X, ldx, Y, ldy, nvalid, lo, d, g_begin, g_count, counters, dkey, row0,   \
                                       alpha, st)
  switch (K) {
    case 7: SKH_PIPE(0);
    case 8: SKH_PIPE(1);
    case 9: SKH_PIPE(2);
    case 10: SKH_PIPE(3);
    case 11: SKH_PIPE(4);
    default: break;
  }
#undef SKH_PIPE
  set_error("internal: bad pipe pass width %d", K);
  return SKH_EINVAL;
}

}  // namespace skh
