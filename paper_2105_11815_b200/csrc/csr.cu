// csr.cu -- R5 for CSR A: dense SA[b, :] = alpha * (ascending-row
// signed sum of the sparse rows of A in bucket b), the same order as the dense
// path (R10), so results equal the oracle bit for bit.
//
// One CTA per (bucket, column tile of <= 8192 columns): the tile's accumulator
// lives in shared memory (zero-filled in place: SA is written exactly once,
// the output-bound part of C4).  Warp 0 walks the bucket's rows in order; each
// step expands up to 32 nonzeros (several rows) across the lanes, and lanes
// that hit the same column (different rows) are combined by their leader in
// lane order = ascending row, so every column sees its terms in canonical
// order.  Then all threads stream the tile out.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxTile = 8192;  // columns per CTA (64 KiB of fp64)

__global__ void __launch_bounds__(kThreads) gather_csr_kernel(
    int64_t m, int64_t ntiles, int tile_cols, const int32_t* __restrict__ ptr, const int32_t* __restrict__ brow,
    const int8_t* __restrict__ bsg, int64_t d, const int64_t* __restrict__ row_ptr,
    const int32_t* __restrict__ col_idx, const double* __restrict__ val, double* __restrict__ SA, int64_t ldsa,
    double alpha) {
  extern __shared__ double acc[];
  __shared__ double stage[32];
  const int64_t b = blockIdx.x / ntiles;
  const int64_t c0 = (blockIdx.x % ntiles) * (int64_t)tile_cols;
  const int width = (int)min((int64_t)tile_cols, d - c0);
  for (int i = threadIdx.x; i < width; i += kThreads) acc[i] = 0.0;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const unsigned lt = (1u << lane) - 1u;
    const int beg = ptr[b], end = ptr[b + 1];
    for (int t0 = beg; t0 < end; t0 += 32) {
      const int cnt = min(32, end - t0);
      int64_t rs = 0;
      int len = 0, neg = 0;
      if (lane < cnt) {
        const int r = brow[t0 + lane];
        neg = bsg[t0 + lane] < 0;
        rs = row_ptr[r];
        len = (int)(row_ptr[r + 1] - rs);
      }
      // inclusive scan of row lengths across the 32 rows of this chunk
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      for (int q0 = 0; q0 < total; q0 += 32) {
        const int q = q0 + lane;
        // slot = first row whose inclusive end exceeds q (binary search by shuffle)
        int lo = 0, hi = 31;
#pragma unroll
        for (int it = 0; it < 5; ++it) {
          const int mid = (lo + hi) >> 1;
          const int v = __shfl_sync(0xffffffffu, incl, mid);
          if (v > q) hi = mid; else lo = mid + 1;
        }
        const int slot = lo;
        const int s_incl = __shfl_sync(0xffffffffu, incl, slot);
        const int s_len = __shfl_sync(0xffffffffu, len, slot);
        const int64_t s_rs = __shfl_sync(0xffffffffu, rs, slot);
        const int s_neg = __shfl_sync(0xffffffffu, neg, slot);
        bool valid = q < total;
        int col = -1;
        double v = 0.0;
        if (valid) {
          const int64_t e = s_rs + (q - (s_incl - s_len));
          const int64_t c = (int64_t)col_idx[e] - c0;
          valid = c >= 0 && c < width;
          if (valid) {
            col = (int)c;
            const double x = val[e];
            v = s_neg ? -x : x;
          }
        }
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        stage[lane] = v;
        __syncwarp();
        if (valid) {
          const unsigned peers = __match_any_sync(vm, col);
          if ((peers & lt) == 0) {  // leader: lowest lane = earliest row
            double a = acc[col];
            unsigned pm = peers;
            while (pm) {
              const int l = __ffs(pm) - 1;
              pm &= pm - 1;
              a = a + stage[l];
            }
            acc[col] = a;
          }
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  double* o = SA + b * ldsa + c0;
  for (int i = threadIdx.x; i < width; i += kThreads) o[i] = alpha * acc[i];
}

}  // namespace

int launch_gather_csr(int64_t m, const int32_t* ptr, const int32_t* rows, const int8_t* sg, int64_t d,
                      const int64_t* row_ptr, const int32_t* col_idx, const double* val, double* SA, int64_t ldsa,
                      double alpha, cudaStream_t st) {
  const int tile = (int)(d < kMaxTile ? d : kMaxTile);
  const int64_t ntiles = (d + tile - 1) / tile;
  const int64_t grid = m * ntiles;
  if (grid >= (1ll << 31)) {
    set_error("csr grid too large");
    return SKH_EOVERFLOW;
  }
  const size_t smem = sizeof(double) * (size_t)tile;
  cudaFuncSetAttribute(gather_csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxTile * 8);
  gather_csr_kernel<<<(unsigned)grid, kThreads, smem, st>>>(m, ntiles, tile, ptr, rows, sg, d, row_ptr, col_idx,
                                                              val, SA, ldsa, alpha); note_launch();
  return check_launch("gather_csr");
}

}  // namespace skh
