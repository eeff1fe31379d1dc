// gather.cu -- R5 for dense X: SA[b, :] = alpha * (ascending-row signed sum of
// X rows in bucket b)  (Alg. 1 Step 1; R10).
//
// Work units (VEC2 layouts, even d > 64): s > 1 -- gather_group_kernel, a group
// of 16 lanes = one bucket x 64 columns (32 contiguous bytes per lane per row),
// two buckets per warp; s = 1 -- gather_wide_kernel, one warp = one bucket x 128
// columns.  gather_dense_kernel (other layouts): one warp = one bucket x one
// 64-column tile; each lane owns two adjacent columns (one 16-byte load per row).
// Every lane adds the bucket's rows sequentially in list order, so every output
// is the oracle's exact sum.  No atomics, no cross-lane reduction.  Rows are
// prefetched a few at a time (row ids broadcast by shuffle) to keep 32-128
// bytes per lane in flight.
//
// Scheduling: CTAs are ordered column-tile-major, so at any time
// the grid works on one column slice of X; for s > 1 the s reads of a row
// segment hit L2 instead of HBM as long as that slice fits in L2 -- the
// 64-column slice does (C3: 131072 x 512 B = 64 MiB < 126 MB), the 128-column
// one does not (128 MiB: C3 DRAM reads 1.39 |A| -> 1.12 |A|).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kWarps = 4;       // buckets per CTA (8: C3 gather 0.956 ms, 4: 0.943, 2: 0.940)
constexpr int kTileCols = 64;   // columns per warp
constexpr int kU = 8;           // rows in flight per lane

template <bool VEC2>
__global__ void __launch_bounds__(kWarps * 32) gather_dense_kernel(
    int64_t m, int64_t nbgroups, const int32_t* __restrict__ ptr, const int32_t* __restrict__ rows,
    const int8_t* __restrict__ sg, int64_t d, const double* __restrict__ X, int64_t ldx,
    double* __restrict__ SA, int64_t ldsa, double alpha) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x / nbgroups;
  const int64_t b = (blockIdx.x % nbgroups) * kWarps + w;
  if (b >= m) return;
  const int64_t c0 = tile * kTileCols;
  // VEC2: lane owns columns c0 + 2 lane, c0 + 2 lane + 1; else c0 + lane, c0 + 32 + lane.
  const int64_t ca = VEC2 ? c0 + 2 * lane : c0 + lane;
  const int64_t cb = VEC2 ? ca + 1 : c0 + 32 + lane;
  const bool va = ca < d, vb = cb < d;
  double acc0 = 0.0, acc1 = 0.0;
  const int beg = ptr[b], end = ptr[b + 1];
  SKH_CHECK(0 <= beg && beg <= end);
  for (int t0 = beg; t0 < end; t0 += 32) {
    const int cnt = min(32, end - t0);
    int my_row = 0, my_neg = 0;
    if (lane < cnt) {
      my_row = rows[t0 + lane];
      my_neg = sg[t0 + lane] < 0;
    }
    for (int u0 = 0; u0 < cnt; u0 += kU) {
      double x0[kU], x1[kU];
      int ng[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int src = u0 + u;
        const int r = __shfl_sync(0xffffffffu, my_row, src & 31);
        ng[u] = __shfl_sync(0xffffffffu, my_neg, src & 31);
        x0[u] = 0.0;
        x1[u] = 0.0;
        if (src < cnt) {
          const double* p = X + (int64_t)r * ldx;
          if (VEC2) {
            if (vb) {
              const double2 v = __ldg(reinterpret_cast<const double2*>(p + ca));
              x0[u] = v.x;
              x1[u] = v.y;
            } else if (va) {
              x0[u] = __ldg(p + ca);
            }
          } else {
            if (va) x0[u] = __ldg(p + ca);
            if (vb) x1[u] = __ldg(p + cb);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (u0 + u < cnt) {  // sequential, list order: the oracle's exact sum
          acc0 = ng[u] ? acc0 - x0[u] : acc0 + x0[u];
          acc1 = ng[u] ? acc1 - x1[u] : acc1 + x1[u];
        }
      }
    }
  }
  double* o = SA + b * ldsa;
  if (VEC2) {
    if (vb) {
      double2 v;
      v.x = alpha * acc0;
      v.y = alpha * acc1;
      *reinterpret_cast<double2*>(o + ca) = v;
    } else if (va) {
      o[ca] = alpha * acc0;
    }
  } else {
    if (va) o[ca] = alpha * acc0;
    if (vb) o[cb] = alpha * acc1;
  }
}

// Wide variant: one warp = one bucket x 128 columns (two 512-byte row segments
// per row, lane owns columns c0 + 2 lane + {0,1} and c0 + 64 + 2 lane + {0,1}),
// 4 rows in flight per lane.  VEC2 layouts only.
__global__ void __launch_bounds__(kWarps * 32) gather_wide_kernel(
    int64_t m, int64_t nbgroups, const int32_t* __restrict__ ptr, const int32_t* __restrict__ rows,
    const int8_t* __restrict__ sg, int64_t d, const double* __restrict__ X, int64_t ldx,
    double* __restrict__ SA, int64_t ldsa, double alpha) {
  constexpr int kW = 4;  // 2: C3 0.983 ms, 8: 1.085 ms (102 registers)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x / nbgroups;
  const int64_t b = (blockIdx.x % nbgroups) * kWarps + w;
  if (b >= m) return;
  const int64_t ca = tile * 128 + 2 * lane, cb = ca + 64;
  const bool va = ca < d, vb = cb < d;  // d even: pairs are whole
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  const int beg = ptr[b], end = ptr[b + 1];
  SKH_CHECK(0 <= beg && beg <= end);
  for (int t0 = beg; t0 < end; t0 += 32) {
    const int cnt = min(32, end - t0);
    int my_row = 0, my_neg = 0;
    if (lane < cnt) {
      my_row = rows[t0 + lane];
      my_neg = sg[t0 + lane] < 0;
    }
    for (int u0 = 0; u0 < cnt; u0 += kW) {
      double2 xa[kW], xb[kW];
      int ng[kW];
#pragma unroll
      for (int u = 0; u < kW; ++u) {
        const int src = u0 + u;
        const int r = __shfl_sync(0xffffffffu, my_row, src & 31);
        ng[u] = __shfl_sync(0xffffffffu, my_neg, src & 31);
        xa[u] = make_double2(0.0, 0.0);
        xb[u] = make_double2(0.0, 0.0);
        if (src < cnt) {
          const double* p = X + (int64_t)r * ldx;
          if (va) xa[u] = __ldg(reinterpret_cast<const double2*>(p + ca));
          if (vb) xb[u] = __ldg(reinterpret_cast<const double2*>(p + cb));
        }
      }
#pragma unroll
      for (int u = 0; u < kW; ++u) {
        if (u0 + u < cnt) {
          a0 = ng[u] ? a0 - xa[u].x : a0 + xa[u].x;
          a1 = ng[u] ? a1 - xa[u].y : a1 + xa[u].y;
          b0 = ng[u] ? b0 - xb[u].x : b0 + xb[u].x;
          b1 = ng[u] ? b1 - xb[u].y : b1 + xb[u].y;
        }
      }
    }
  }
  double* o = SA + b * ldsa;
  if (va) *reinterpret_cast<double2*>(o + ca) = make_double2(alpha * a0, alpha * a1);
  if (vb) *reinterpret_cast<double2*>(o + cb) = make_double2(alpha * b0, alpha * b1);
}

// Lane-group variant: a group of GL lanes = one bucket x 4 GL columns (one
// 32 GL-byte row segment per row; lane l of the group owns columns c0 + 4 l ..
// c0 + 4 l + 3, two 16-byte loads), 32 / GL buckets per warp, 4 rows in flight
// per lane.  The grid is column-tile-major over 4 GL-column tiles, so the slice
// of X being read at any time is n x 32 GL bytes (C3, GL = 16: 64 MiB) and fits
// in L2: the s reads of a row segment cost one HBM read.  VEC2 layouts (d even).
template <int GL>
__global__ void __launch_bounds__(kWarps * 32) gather_group_kernel(
    int64_t m, int64_t nbgroups, const int32_t* __restrict__ ptr, const int32_t* __restrict__ rows,
    const int8_t* __restrict__ sg, int64_t d, const double* __restrict__ X, int64_t ldx,
    double* __restrict__ SA, int64_t ldsa, double alpha) {
  constexpr int kW = 4, NG = 32 / GL;
  const int lane = threadIdx.x & 31, hl = lane % GL, grp = lane / GL, w = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x / nbgroups;
  const int64_t b = ((blockIdx.x % nbgroups) * kWarps + w) * NG + grp;
  const bool live = b < m;
  const int64_t ca = tile * (4 * GL) + 4 * hl, cb = ca + 2;
  const bool va = live && ca < d, vb = live && cb < d;  // d even: pairs are whole
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  const int beg = live ? ptr[b] : 0, end = live ? ptr[b + 1] : 0;
  SKH_CHECK(0 <= beg && beg <= end);
  const int len = end - beg;
  int lmax = len;  // the warp runs the longest bucket's trips
#pragma unroll
  for (int x = GL; x < 32; x <<= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, x));
  for (int t0 = 0; t0 < lmax; t0 += GL) {
    const int cnt = min(GL, len - t0);  // this group's rows in the chunk (<= 0: none)
    int my_row = 0;
    if (hl < cnt) my_row = rows[beg + t0 + hl] | (sg[beg + t0 + hl] < 0 ? (int)0x80000000 : 0);
    const int cmax = min(GL, lmax - t0);
    for (int u0 = 0; u0 < cmax; u0 += kW) {
      double2 xa[kW], xb[kW];
      int rr[kW];
#pragma unroll
      for (int u = 0; u < kW; ++u) {
        const int src = u0 + u;
        rr[u] = __shfl_sync(0xffffffffu, my_row, grp * GL + (src % GL));
        xa[u] = make_double2(0.0, 0.0);
        xb[u] = make_double2(0.0, 0.0);
        if (src < cnt) {
          const double* p = X + (int64_t)(rr[u] & 0x7fffffff) * ldx;
          if (va) xa[u] = __ldg(reinterpret_cast<const double2*>(p + ca));
          if (vb) xb[u] = __ldg(reinterpret_cast<const double2*>(p + cb));
        }
      }
#pragma unroll
      for (int u = 0; u < kW; ++u) {
        if (u0 + u < cnt) {  // sequential, list order: the oracle's exact sum
          const bool ng = rr[u] < 0;
          a0 = ng ? a0 - xa[u].x : a0 + xa[u].x;
          a1 = ng ? a1 - xa[u].y : a1 + xa[u].y;
          b0 = ng ? b0 - xb[u].x : b0 + xb[u].x;
          b1 = ng ? b1 - xb[u].y : b1 + xb[u].y;
        }
      }
    }
  }
  double* o = SA + b * ldsa;
  if (va) *reinterpret_cast<double2*>(o + ca) = make_double2(alpha * a0, alpha * a1);
  if (vb) *reinterpret_cast<double2*>(o + cb) = make_double2(alpha * b0, alpha * b1);
}

// Sb: one warp per bucket.  Up to 4 x 32 entries are loaded at once (one per
// lane per chunk, all loads in flight together), then added to the running sum
// in list order via shuffles -- the same sequential order as the oracle.
__global__ void gather_vec_kernel(int64_t m, const int32_t* __restrict__ ptr, const int32_t* __restrict__ rows,
                                  const int8_t* __restrict__ sg, const double* __restrict__ x,
                                  double* __restrict__ out, double alpha) {
  constexpr int kU = 4;
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= m) return;
  const int beg = ptr[b], end = ptr[b + 1];
  SKH_CHECK(0 <= beg && beg <= end);
  double acc = 0.0;
  for (int t0 = beg; t0 < end; t0 += 32 * kU) {
    int r[kU];
    int8_t g[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int t = t0 + 32 * u + lane;
      r[u] = t < end ? rows[t] : -1;
      g[u] = t < end ? sg[t] : 1;
    }
    double v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      v[u] = r[u] >= 0 ? __ldg(x + r[u]) : 0.0;
      if (g[u] < 0) v[u] = -v[u];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int cnt = min(32, end - (t0 + 32 * u));
      for (int k = 0; k < cnt; ++k) acc = acc + __shfl_sync(0xffffffffu, v[u], k);
    }
  }
  if (lane == 0) out[b] = alpha * acc;
}

}  // namespace

int launch_gather_dense(int64_t m, const int32_t* ptr, const int32_t* rows, const int8_t* sg, int64_t d,
                        const double* X, int64_t ldx, double* SA, int64_t ldsa, double alpha, cudaStream_t st, int s) {
  const int64_t nbgroups = (m + kWarps - 1) / kWarps;
  const int64_t ntiles = (d + kTileCols - 1) / kTileCols;
  const int64_t grid = nbgroups * ntiles;
  if (grid >= (1ll << 31)) {
    set_error("gather grid too large");
    return SKH_EOVERFLOW;
  }
  const bool vec2 = ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(SA)) % 16 == 0) &&
                    (ldx % 2 == 0) && (ldsa % 2 == 0);
  // 128 columns per warp (1 KB of each row) unless SKH_GATHER_WIDE=0; measured
  // C3 gather 1.019 -> 0.956 ms, C5 10.01 -> 9.72 ms
  static const bool wide = [] {
    const char* e = getenv("SKH_GATHER_WIDE");
    return !(e && e[0] == '0');
  }();
  // s > 1: the lane-group kernel with SKH_GATHER_GL lanes per bucket (16
  // default, 8; 0: the 128-column wide kernel, whose n x 1 KB slice exceeds L2
  // at C3, so part of the s reads go to HBM again -- measured C3 gather 0.939 ->
  // 0.814 ms, C3HD 1.011 -> 0.886); s = 1 has no re-read and keeps the wide
  // kernel (C5 row gather 9.80 vs 10.06 ms)
  static const int gl = [] {
    const char* e = getenv("SKH_GATHER_GL");
    return e ? atoi(e) : 16;
  }();
  if (s > 1 && (gl == 8 || gl == 16) && wide && vec2 && d % 2 == 0 && d > 64) {
    const int64_t nt = (d + 4 * gl - 1) / (4 * gl);
    const int64_t per_cta = (int64_t)kWarps * (32 / gl);
    const int64_t nbg = (m + per_cta - 1) / per_cta;
    if (nbg * nt >= (1ll << 31)) {
      set_error("gather grid too large");
      return SKH_EOVERFLOW;
    }
    if (gl == 16)
      gather_group_kernel<16><<<(unsigned)(nbg * nt), kWarps * 32, 0, st>>>(m, nbg, ptr, rows, sg, d, X, ldx, SA, ldsa,
                                                                           alpha);
    else
      gather_group_kernel<8><<<(unsigned)(nbg * nt), kWarps * 32, 0, st>>>(m, nbg, ptr, rows, sg, d, X, ldx, SA, ldsa,
                                                                          alpha);
    note_launch();
    return check_launch("gather_group");
  }
  if (wide && vec2 && d % 2 == 0 && d > 64) {
    const int64_t nt = (d + 127) / 128;
    gather_wide_kernel<<<(unsigned)(nbgroups * nt), kWarps * 32, 0, st>>>(m, nbgroups, ptr, rows, sg, d, X, ldx, SA,
                                                                          ldsa, alpha);
    note_launch();
    return check_launch("gather_wide");
  }
  if (vec2)
    gather_dense_kernel<true><<<(unsigned)grid, kWarps * 32, 0, st>>>(m, nbgroups, ptr, rows, sg, d, X, ldx, SA,
                                                                       ldsa, alpha);
  else
    gather_dense_kernel<false><<<(unsigned)grid, kWarps * 32, 0, st>>>(m, nbgroups, ptr, rows, sg, d, X, ldx, SA,
                                                                        ldsa, alpha);
  note_launch();
  return check_launch("gather_dense");
}

int launch_gather_vec(int64_t m, const int32_t* ptr, const int32_t* rows, const int8_t* sg, const double* b,
                      double* Sb, double alpha, cudaStream_t st) {
  gather_vec_kernel<<<(unsigned)((m * 32 + 127) / 128), 128, 0, st>>>(m, ptr, rows, sg, b, Sb, alpha);
  note_launch();
  return check_launch("gather_vec");
}

}  // namespace skh
