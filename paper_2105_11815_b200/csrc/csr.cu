// csr.cu -- R5 for CSR A: dense SA[b, :] = alpha * (ascending-row
// signed sum of the sparse rows of A in bucket b), the same order as the dense
// path (R10), so results equal the oracle bit for bit.
//
// C4: m = 16384 buckets of ~192 rows x 8 nonzeros; SA is 1 GiB dense (91 % of
// the bytes), so the job is to write SA once at HBM speed.  Two phases:
//   Expand  (streaming, one thread per bucket-list entry) the list of (column,
//           signed value) pairs of S.A in bucket order, i.e. the CSR form of
//           S.A with duplicate columns: each bucket entry copies its row's
//           nonzeros to its offset (a scan of the row lengths in bucket order).
//           All entries are independent, so the random row reads of A are all in
//           flight together instead of forming per-bucket dependent chains.
//   Reduce  one CTA per bucket: its contiguous run of pairs is staged with
//           coalesced loads; per column tile (<= 4096 fp64 columns of shared
//           memory, zero-filled in place) the run is consumed 256 pairs at a
//           time; pairs of one chunk that share a column are applied in rounds
//           (integer atomicMin on a per-column claim picks the earliest pending
//           pair, which adds its value) -- every column sees its terms in list
//           order = ascending row, the canonical order.  The tile is streamed
//           out once with 16-byte stores.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kThreads = 256;
constexpr int kTileMax = 4096;   // fp64 accumulator columns per pass (32 KiB)
constexpr int kStageCap = 2048;  // staged pairs (24 KiB)
constexpr int kFree = 0x7fffffff;

struct CsrWs {
  int32_t* off;   // [N + 1] exclusive scan of row lengths in bucket order
  int64_t* rst;   // [N] row start (row_ptr[row]) of every bucket entry
  int32_t* bs;    // scan scratch
  int32_t* ecol;  // [s * nnz]
  double* eval;   // [s * nnz]
};

CsrWs csr_carve(void* ws, int64_t N, int64_t nexp) {
  CsrWs w;
  char* p = static_cast<char*>(ws);
  w.off = reinterpret_cast<int32_t*>(p);
  p += align_up(sizeof(int32_t) * (size_t)(N + 1));
  w.rst = reinterpret_cast<int64_t*>(p);
  p += align_up(sizeof(int64_t) * (size_t)std::max<int64_t>(N, 1));
  w.bs = reinterpret_cast<int32_t*>(p);
  p += align_up(sizeof(int32_t) * (size_t)scan_scratch_ints(N + 1));
  w.eval = reinterpret_cast<double*>(p);
  p += align_up(sizeof(double) * (size_t)std::max<int64_t>(nexp, 1));
  w.ecol = reinterpret_cast<int32_t*>(p);
  return w;
}

// Row lengths in bucket order (scanned into off) and each entry's row start, so
// the expand reads both coalesced instead of two random row_ptr words per entry.
__global__ void csr_len_kernel(int64_t N, const int32_t* __restrict__ brow, const int64_t* __restrict__ row_ptr,
                               int32_t* __restrict__ off, int64_t* __restrict__ rst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > N) return;
  if (t == N) {
    off[N] = 0;
    return;
  }
  const int r = brow[t];
  const int64_t a = row_ptr[r];
  off[t] = (int32_t)(row_ptr[r + 1] - a);
  rst[t] = a;
}

__global__ void __launch_bounds__(256, 6) csr_expand_kernel(int64_t N, const int8_t* __restrict__ bsg,
                                                            const int64_t* __restrict__ rst,
                                                            const int32_t* __restrict__ col_idx,
                                                            const double* __restrict__ val,
                                                            const int32_t* __restrict__ off,
                                                            int32_t* __restrict__ ecol, double* __restrict__ eval) {
  // 8 lanes per entry: each quarter-warp copies one row's run with contiguous
  // (coalesced) loads and stores, 4 entries per warp instruction
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t t = gt >> 3;
  const int j = (int)(gt & 7);
  if (t >= N) return;
  const bool neg = bsg[t] < 0;
  const int64_t rs = rst[t];
  const int o = off[t];
  const int len = off[t + 1] - o;
  for (int k = j; k < len; k += 8) {
    const int c = col_idx[rs + k];
    const double x = val[rs + k];
    ecol[o + k] = c;
    eval[o + k] = neg ? -x : x;
  }
}

__global__ void __launch_bounds__(kThreads, 3) csr_reduce_kernel(
    int64_t m, const int32_t* __restrict__ ptr, const int32_t* __restrict__ off, const int32_t* __restrict__ ecol,
    const double* __restrict__ eval, int64_t d, int tile_cols, double* __restrict__ SA, int64_t ldsa, double alpha) {
  extern __shared__ double acc[];  // [tile_cols]
  __shared__ int s_col[kStageCap];
  __shared__ double s_val[kStageCap];
  __shared__ int claim[kTileMax];
  const int64_t b = blockIdx.x;
  const int e_beg = off[ptr[b]], e_end = off[ptr[b + 1]];
  const int ntiles = (int)((d + tile_cols - 1) / tile_cols);
  const bool whole = e_end - e_beg <= kStageCap;
  if (whole) {
    for (int e = e_beg + (int)threadIdx.x; e < e_end; e += kThreads) {
      s_col[e - e_beg] = ecol[e];
      s_val[e - e_beg] = eval[e];
    }
  }
  for (int t = 0; t < ntiles; ++t) {
    const int64_t c0 = (int64_t)t * tile_cols;
    const int c0i = (int)c0;  // d < 2^31
    const int width = (int)min((int64_t)tile_cols, d - c0);
    for (int i = threadIdx.x; i < width; i += kThreads) {
      acc[i] = 0.0;
      claim[i] = kFree;
    }
    for (int s0 = e_beg; s0 < e_end; s0 += kStageCap) {
      const int cnt = min(kStageCap, e_end - s0);
      if (!whole) {
        __syncthreads();
        for (int e = (int)threadIdx.x; e < cnt; e += kThreads) {
          s_col[e] = ecol[s0 + e];
          s_val[e] = eval[s0 + e];
        }
      }
      __syncthreads();
      // every thread holds up to kPer pairs (e = tid + k*256); a round applies,
      // for each column, its earliest pending pair of the whole staged run, so
      // the number of rounds is the largest column multiplicity (a few)
      constexpr int kPer = kStageCap / kThreads;
      int pcol[kPer];
      unsigned pend = 0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int e = (int)threadIdx.x + k * kThreads;
        pcol[k] = 0;
        if (e < cnt) {
          const int cc = s_col[e] - c0i;
          if ((unsigned)cc < (unsigned)width) {
            pcol[k] = cc;
            pend |= 1u << k;
          }
        }
      }
      while (__syncthreads_or(pend != 0)) {
#pragma unroll
        for (int k = 0; k < kPer; ++k)
          if ((pend >> k) & 1u) atomicMin(&claim[pcol[k]], (int)threadIdx.x + k * kThreads);
        __syncthreads();
        unsigned win = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k)
          if (((pend >> k) & 1u) && claim[pcol[k]] == (int)threadIdx.x + k * kThreads) win |= 1u << k;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPer; ++k)
          if ((win >> k) & 1u) {  // the earliest pending pair of this column
            acc[pcol[k]] = acc[pcol[k]] + s_val[threadIdx.x + k * kThreads];
            claim[pcol[k]] = kFree;
          }
        pend &= ~win;
      }
    }
    __syncthreads();
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

size_t csr_ws_bytes(int64_t nrows, int s, int64_t nnz) {
  const int64_t N = nrows * (int64_t)s;
  const int64_t nexp = nnz * (int64_t)s;
  return align_up(sizeof(int32_t) * (size_t)(N + 1)) + align_up(sizeof(int64_t) * (size_t)std::max<int64_t>(N, 1)) +
         align_up(sizeof(int32_t) * (size_t)scan_scratch_ints(N + 1)) +
         align_up(sizeof(double) * (size_t)std::max<int64_t>(nexp, 1)) +
         align_up(sizeof(int32_t) * (size_t)std::max<int64_t>(nexp, 1));
}

int launch_gather_csr(int64_t m, int s, const int32_t* ptr, const int32_t* rows, const int8_t* sg, int64_t nrows,
                      int64_t d, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                      double* SA, int64_t ldsa, double alpha, void* ws, cudaStream_t st) {
  const int64_t N = nrows * (int64_t)s;
  CsrWs w = csr_carve(ws, N, nnz * (int64_t)s);
  int rc;
  csr_len_kernel<<<(unsigned)((N + 1 + 255) / 256), 256, 0, st>>>(N, rows, row_ptr, w.off, w.rst);
  note_launch();
  rc = launch_excl_scan_i32(w.off, N + 1, w.bs, st);
  if (rc) return rc;
  if (N > 0) {
    csr_expand_kernel<<<(unsigned)((N * 8 + 255) / 256), 256, 0, st>>>(N, sg, w.rst, col_idx, val, w.off, w.ecol,
                                                                        w.eval);
    note_launch();
  }
  const int tile = (int)(d < kTileMax ? d : kTileMax);
  const size_t smem = sizeof(double) * (size_t)tile;
  cudaFuncSetAttribute(csr_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  csr_reduce_kernel<<<(unsigned)m, kThreads, smem, st>>>(m, ptr, w.off, w.ecol, w.eval, d, tile, SA, ldsa, alpha);
  note_launch();
  return check_launch("gather_csr");
}

}  // namespace skh
