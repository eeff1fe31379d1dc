// csr.cu -- R5 for CSR A: dense SA[b, :] = alpha * (ascending-row
// signed sum of the sparse rows of A in bucket b), the same order as the dense
// path (R10), so results equal the oracle bit for bit.
//
// One CTA per bucket (C4: m = 16384 buckets of ~192 rows x 8 nonzeros; SA is
// 1 GiB dense, 91 % of the bytes -- the kernel is bound by writing SA once).
//   Stage   256 rows per round, one per thread: row id + sign, then row_ptr, a
//           block scan of the row lengths, then each thread copies its row's
//           nonzeros (up to 16 loads in flight) -- three dependent round trips
//           per 256 rows.  (column, signed value) pairs land in shared memory in
//           list order (= ascending row; columns are distinct inside a row).
//   Reduce  per column tile (<= 4096 fp64 columns in shared memory, zero-filled
//           in place), the staged list is consumed 256 entries at a time, one per
//           thread.  Entries of one chunk that share a column are applied in
//           rounds: each pending entry claims its column with an integer
//           atomicMin of its list index (order-free), the minimum adds its value,
//           the rest retry -- so every column sees its terms in ascending list
//           order, the canonical order.  Conflicts are rare (1536 entries over
//           8192 columns), so a chunk takes ~2 rounds.
//   Write   the tile is streamed out once with 16-byte stores.
// A bucket whose nonzeros fit the staging buffer is staged once for all column
// tiles; larger buckets are processed in row chunks, in order.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileMax = 4096;   // fp64 accumulator columns per pass (32 KiB)
constexpr int kStageCap = 2048;  // staged nonzeros (24 KiB)
constexpr int kFree = 0x7fffffff;

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

__global__ void __launch_bounds__(kThreads, 3) gather_csr_kernel(
    int64_t m, const int32_t* __restrict__ ptr, const int32_t* __restrict__ brow, const int8_t* __restrict__ bsg,
    int64_t d, int tile_cols, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
    const double* __restrict__ val, double* __restrict__ SA, int64_t ldsa, double alpha) {
  extern __shared__ double acc[];  // [tile_cols]
  __shared__ int s_col[kStageCap];
  __shared__ double s_val[kStageCap];
  __shared__ int claim[kTileMax];
  __shared__ int s_end;
  __shared__ int wsum[32];
  __shared__ int s_total;
  const int64_t b = blockIdx.x;
  const int beg = ptr[b], end = ptr[b + 1];
  const int ntiles = (int)((d + tile_cols - 1) / tile_cols);
  bool whole = false;  // the whole bucket sits in the staging buffer
  int staged = 0;

  for (int t = 0; t < ntiles; ++t) {
    const int64_t c0 = (int64_t)t * tile_cols;
    const int c0i = (int)c0;  // d < 2^31
    const int width = (int)min((int64_t)tile_cols, d - c0);
    for (int i = threadIdx.x; i < width; i += kThreads) {
      acc[i] = 0.0;
      claim[i] = kFree;
    }
    int rpos = beg;
    while (rpos < end) {
      int rnext = rpos;
      if (!whole) {
        // ---- stage rows [rpos, ...) while they fit kStageCap nonzeros
        staged = 0;
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
          // rows that fit after `staged` entries form a prefix of this round
          const bool fits = tr < end && staged + off + len <= kStageCap;
          const int nfit = __syncthreads_count(fits);
          if (fits && (int)threadIdx.x == nfit - 1) s_end = staged + off + len;
          if (fits) {
            // the first 16 nonzeros of the row are loaded together, then stored
            const int o = staged + off;
            int cbuf[16];
            double vbuf[16];
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (k < len) {
                cbuf[k] = col_idx[rs + k];
                vbuf[k] = val[rs + k];
              }
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (k < len) {
                s_col[o + k] = cbuf[k];
                s_val[o + k] = neg ? -vbuf[k] : vbuf[k];
              }
            for (int k = 16; k < len; ++k) {
              s_col[o + k] = col_idx[rs + k];
              const double x = val[rs + k];
              s_val[o + k] = neg ? -x : x;
            }
          }
          __syncthreads();
          if (nfit > 0) staged = s_end;
          rnext += nfit;
          if (nfit == 0 && staged == 0) {
            // one row longer than the staging buffer: reduce it straight from
            // global memory (its columns are distinct, so no ordering inside it)
            const int r = brow[rnext];
            const int ng = bsg[rnext] < 0;
            const int64_t rs0 = row_ptr[r], re = row_ptr[r + 1];
            for (int64_t q = rs0 + threadIdx.x; q < re; q += kThreads) {
              const int cc = col_idx[q] - c0i;
              if ((unsigned)cc < (unsigned)width) {
                const double x = val[q];
                acc[cc] = acc[cc] + (ng ? -x : x);
              }
            }
            __syncthreads();
            rnext += 1;
            break;
          }
          if (nfit < kThreads || rnext >= end) break;
        }
        if (rpos == beg && rnext >= end && staged > 0) whole = true;
      } else {
        rnext = end;
      }
      // ---- reduce the staged entries [0, staged) into the tile, canonical order
      for (int e0 = 0; e0 < staged; e0 += kThreads) {
        const int e = e0 + (int)threadIdx.x;
        int col = 0;
        double v = 0.0;
        bool pending = false;
        if (e < staged) {
          col = s_col[e] - c0i;
          pending = (unsigned)col < (unsigned)width;
          if (pending) v = s_val[e];
        }
        while (__syncthreads_or(pending)) {
          if (pending) atomicMin(&claim[col], e);
          __syncthreads();
          const bool win = pending && claim[col] == e;
          __syncthreads();
          if (win) {  // the earliest pending entry of this column in the chunk
            acc[col] = acc[col] + v;
            claim[col] = kFree;
            pending = false;
          }
        }
      }
      __syncthreads();
      if (!whole) staged = 0;
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
