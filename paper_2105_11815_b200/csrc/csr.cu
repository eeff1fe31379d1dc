// csr.cu -- R5 for CSR A: dense SA[b, :] = alpha * (ascending-row
// signed sum of the sparse rows of A in bucket b), the same order as the dense
// path (R10), so results equal the oracle bit for bit.
//
// One CTA per bucket (C4: m = 16384 buckets of ~192 rows x 8 nonzeros; SA is
// 1 GiB dense, 91 % of the bytes -- the kernel is bound by writing SA once).
//   Stage   all 256 threads pull the bucket's rows in parallel (one row per
//           thread per round: row id, sign, row_ptr, then its nonzeros) and pack
//           (column, signed value) in list order into shared memory -- three
//           dependent round trips per 256 rows instead of one per nonzero.
//   Reduce  per column tile (<= 4096 columns of fp64 in shared memory, zero-filled
//           in place): warp w owns 1/8 of the tile's columns and walks the packed
//           list in order; lanes of one 32-entry step that hit the same column
//           are combined by their lowest lane in lane order (= ascending row),
//           so every column sees its terms in canonical order.
//   Write   the tile is streamed out once with 16-byte stores.
// Buckets larger than the staging capacity are processed in row chunks in
// order, which keeps the summation order.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileMax = 4096;   // fp64 accumulator columns per pass (32 KiB)
constexpr int kStageCap = 2048;  // staged nonzeros (24 KiB)

__device__ __forceinline__ int block_excl_scan_csr(int v, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const int x = lane < kWarps ? wsum[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    if (lane < kWarps) wsum[lane] = xi - x;
    if (lane == kWarps - 1) *total = xi;
  }
  __syncthreads();
  const int r = inc - v + wsum[wid];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kThreads) gather_csr_kernel(
    int64_t m, const int32_t* __restrict__ ptr, const int32_t* __restrict__ brow, const int8_t* __restrict__ bsg,
    int64_t d, int tile_cols, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
    const double* __restrict__ val, double* __restrict__ SA, int64_t ldsa, double alpha) {
  extern __shared__ double acc[];                       // [tile_cols]
  __shared__ int s_col[kStageCap];
  __shared__ double s_val[kStageCap];
  __shared__ double stage[kWarps][32];
  __shared__ int wsum[32];
  __shared__ int s_total;
  const int64_t b = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int beg = ptr[b], end = ptr[b + 1];
  const int ntiles = (int)((d + tile_cols - 1) / tile_cols);

  // column tiles one after another; within a tile the rows are staged in
  // chunks, in list order, and each chunk is reduced before the next.
  for (int t = 0; t < ntiles; ++t) {
    const int64_t c0 = (int64_t)t * tile_cols;
    const int width = (int)min((int64_t)tile_cols, d - c0);
    for (int i = threadIdx.x; i < width; i += kThreads) acc[i] = 0.0;
    int rpos = beg;  // next row (list position) to stage
    while (rpos < end) {
      // ---- stage rows [rpos, ...) while they fit kStageCap nonzeros
      int staged = 0;
      int rnext = rpos;
      while (rnext < end) {
        const int tr = rnext + (int)threadIdx.x;
        int len = 0, neg = 0;
        int64_t rs = 0;
        if (tr < end) {
          const int r = brow[tr];
          neg = bsg[tr] < 0;
          rs = row_ptr[r];
          len = (int)(row_ptr[r + 1] - rs);
        }
        const int off = block_excl_scan_csr(len, wsum, &s_total);
        // rows that fit entirely after `staged` entries (offsets grow with the
        // thread index, so the fitting rows are a prefix of this round)
        const bool fits = staged + off + len <= kStageCap;
        const int nfit = __syncthreads_count(tr < end && fits);
        if (tr < end && fits) {
          for (int k = 0; k < len; ++k) {
            s_col[staged + off + k] = col_idx[rs + k];
            const double x = val[rs + k];
            s_val[staged + off + k] = neg ? -x : x;
          }
        }
        int add = 0;
        if (nfit > 0) {
          // total staged entries of the fitting prefix = off + len of the last fitting row
          __shared__ int s_last;
          if (tr < end && fits && (threadIdx.x == nfit - 1)) s_last = off + len;
          __syncthreads();
          add = s_last;
        }
        staged += add;
        rnext += nfit;
        __syncthreads();
        if (nfit < kThreads || rnext >= end) {
          if (nfit == 0 && staged == 0) {
            // very long row (> kStageCap nonzeros): reduce it directly from global, chunk by chunk
            const int r = brow[rnext];
            const int neg = bsg[rnext] < 0;
            const int64_t rs = row_ptr[r], re = row_ptr[r + 1];
            for (int64_t q0 = rs; q0 < re; q0 += kStageCap) {
              const int cnt = (int)min((int64_t)kStageCap, re - q0);
              for (int k = threadIdx.x; k < cnt; k += kThreads) {
                s_col[k] = col_idx[q0 + k];
                const double x = val[q0 + k];
                s_val[k] = neg ? -x : x;
              }
              __syncthreads();
              // columns within one row are distinct: no ordering among them
              for (int k = threadIdx.x; k < cnt; k += kThreads) {
                const int64_t cc = (int64_t)s_col[k] - c0;
                if (cc >= 0 && cc < width) acc[cc] = acc[cc] + s_val[k];
              }
              __syncthreads();
            }
            rnext += 1;
          }
          break;
        }
      }
      // ---- reduce the staged entries [0, staged) into the tile, canonical order
      if (staged > 0) {
        const int cw = (width + kWarps - 1) / kWarps;
        const int clo = w * cw, chi = min(width, clo + cw);
        for (int e0 = 0; e0 < staged; e0 += 32) {
          const int e = e0 + lane;
          int col = -1;
          double v = 0.0;
          bool valid = false;
          if (e < staged) {
            const int64_t cc = (int64_t)s_col[e] - c0;
            valid = cc >= clo && cc < chi;
            if (valid) {
              col = (int)cc;
              v = s_val[e];
            }
          }
          const unsigned vm = __ballot_sync(0xffffffffu, valid);
          if (vm) {
            stage[w][lane] = v;
            __syncwarp();
            if (valid) {
              const unsigned peers = __match_any_sync(vm, col);
              if ((peers & lt) == 0) {
                double a = acc[col];
                unsigned pm = peers;
                while (pm) {
                  const int l = __ffs(pm) - 1;
                  pm &= pm - 1;
                  a = a + stage[w][l];
                }
                acc[col] = a;
              }
            }
            __syncwarp();
          }
        }
      }
      __syncthreads();
      rpos = rnext;
    }
    // ---- write the tile
    double* o = SA + b * ldsa + c0;
    const bool vec = ((reinterpret_cast<uintptr_t>(o) & 15) == 0) && (width % 2 == 0);
    if (vec) {
      for (int i = threadIdx.x; i < width / 2; i += kThreads) {
        const double2 x = make_double2(alpha * acc[2 * i], alpha * acc[2 * i + 1]);
        *reinterpret_cast<double2*>(o + 2 * i) = x;
      }
    } else {
      for (int i = threadIdx.x; i < width; i += kThreads) o[i] = alpha * acc[i];
    }
    __syncthreads();
  }
}

}  // namespace

int launch_gather_csr(int64_t m, const int32_t* ptr, const int32_t* rows, const int8_t* sg, int64_t d,
                      const int64_t* row_ptr, const int32_t* col_idx, const double* val, double* SA, int64_t ldsa,
                      double alpha, cudaStream_t st) {
  if (m >= (1ll << 31)) {
    set_error("csr: too many buckets");
    return SKH_EOVERFLOW;
  }
  const int tile = (int)(d < kTileMax ? d : kTileMax);
  const size_t smem = sizeof(double) * (size_t)tile;
  cudaFuncSetAttribute(gather_csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gather_csr_kernel<<<(unsigned)m, kThreads, smem, st>>>(m, ptr, rows, sg, d, tile, row_ptr, col_idx, val, SA, ldsa,
                                                         alpha);
  note_launch();
  return check_launch("gather_csr");
}

}  // namespace skh
