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
//   Reduce  one CTA per bucket: its contiguous run of pairs is loaded into
//           registers once; per column tile (<= 4096 fp64 columns of shared
//           memory, zero-filled in place) every pair takes an arrival rank on
//           its column; single pairs store, pairs of two add (IEEE addition
//           commutes), longer columns are summed by one thread in list order
//           (= ascending row, the canonical order); claim rounds are the
//           fallback for long runs and heavy columns (csr_reduce_kernel).  The
//           tile is streamed out once with 16-byte stores.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kThreads = 256;
constexpr int kTileMax = 4096;   // fp64 accumulator columns per pass (32 KiB)
constexpr int kChunk = 2048;     // pairs held in registers (8 per thread)
constexpr int kPer = 2048 / 256;
constexpr int kFree = 0x7fffffff;
constexpr int kSideCap = 256;    // side list (pairs of columns with >= 3) per tile


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

constexpr int kExpE = 2;  // bucket-list entries per 8-lane group (all their loads in flight together)

__global__ void __launch_bounds__(256) csr_expand_kernel(int64_t N, const int8_t* __restrict__ bsg,
                                                         const int64_t* __restrict__ rst,
                                                         const int32_t* __restrict__ col_idx,
                                                         const double* __restrict__ val,
                                                         const int32_t* __restrict__ off,
                                                         int32_t* __restrict__ ecol, double* __restrict__ eval) {
  // 8 lanes per entry: each quarter-warp copies one row's run with contiguous
  // (coalesced) loads and stores; a quarter-warp takes kExpE entries spaced by
  // the grid's group count, and issues every load of its first 8 nonzeros per
  // entry before any store (the random row reads are latency-bound otherwise)
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g = gt >> 3, ngroups = ((int64_t)gridDim.x * blockDim.x) >> 3;
  const int j = (int)(gt & 7);
  int64_t rs[kExpE];
  int o[kExpE], len[kExpE];
  bool neg[kExpE];
#pragma unroll
  for (int u = 0; u < kExpE; ++u) {
    const int64_t t = g + u * ngroups;
    len[u] = 0;
    if (t < N) {
      neg[u] = bsg[t] < 0;
      rs[u] = rst[t];
      o[u] = off[t];
      len[u] = off[t + 1] - o[u];
    }
  }
  int c[kExpE];
  double x[kExpE];
#pragma unroll
  for (int u = 0; u < kExpE; ++u) {
    if (j < len[u]) {
      c[u] = col_idx[rs[u] + j];
      x[u] = val[rs[u] + j];
    }
  }
#pragma unroll
  for (int u = 0; u < kExpE; ++u) {
    if (j < len[u]) {
      ecol[o[u] + j] = c[u];
      eval[o[u] + j] = neg[u] ? -x[u] : x[u];
    }
    for (int k = j + 8; k < len[u]; k += 8) {  // rows longer than 8 nonzeros
      const int cc = col_idx[rs[u] + k];
      const double xx = val[rs[u] + k];
      ecol[o[u] + k] = cc;
      eval[o[u] + k] = neg[u] ? -xx : xx;
    }
  }
}

// Claim rounds over one chunk of pairs held in registers (pc/pv, pair e =
// tid + k * kThreads of the chunk): each round applies, for every column, its
// earliest pending pair (integer atomicMin on claim[]), so every column sees its
// terms in list order.  claim[] must be kFree on entry and is kFree on exit.
__device__ __forceinline__ void claim_rounds(double* acc, int* claim, const int (&pc)[kPer], const double (&pv)[kPer],
                                             unsigned pend) {
  while (__syncthreads_or(pend != 0)) {
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if ((pend >> k) & 1u) atomicMin(&claim[pc[k]], (int)threadIdx.x + k * kThreads);
    __syncthreads();
    unsigned win = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (((pend >> k) & 1u) && claim[pc[k]] == (int)threadIdx.x + k * kThreads) win |= 1u << k;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if ((win >> k) & 1u) {
        acc[pc[k]] = acc[pc[k]] + pv[k];
        claim[pc[k]] = kFree;
      }
    pend &= ~win;
  }
}

// One CTA per bucket.  Its run of (column, signed value) pairs (list order =
// canonical order) is loaded into registers once when it has <= kChunk pairs,
// and per column tile (<= 4096 fp64 columns of shared memory):
//   fast path: count each column's pairs (integer atomicAdd on word[c]); a
//     single pair stores 0 + v; a column of two pairs takes two fp64 shared
//     atomic adds onto 0 -- IEEE addition commutes, so (0 + a) + b == (0 + b) + a
//     is the list-order sum whatever order they land in; the pairs of columns
//     with more go to a side list, sorted by (column, index) by counting, and
//     the first pair of each column's run sums the run in list order.  A few
//     barriers per tile instead of three per round.
//   fallback (side list over capacity, or a run longer than kChunk): claim
//     rounds, chunk by chunk.
__global__ void __launch_bounds__(kThreads, 4) csr_reduce_kernel(
    int64_t m, const int32_t* __restrict__ ptr, const int32_t* __restrict__ off, const int32_t* __restrict__ ecol,
    const double* __restrict__ eval, int64_t d, int tile_cols, double* __restrict__ SA, int64_t ldsa, double alpha) {
  extern __shared__ double acc[];  // [tile_cols]
  __shared__ int word[kTileMax];
  __shared__ int side_ci[kSideCap];  // column
  __shared__ int side_ix[kSideCap];
  __shared__ double side_v[kSideCap];
  __shared__ double sorted_v[kSideCap];
  __shared__ int sorted_c[kSideCap];
  __shared__ int side_n, fallback;
  const int64_t b = blockIdx.x;
  const int e_beg = off[ptr[b]], e_end = off[ptr[b + 1]];
  SKH_CHECK(0 <= e_beg && e_beg <= e_end);
  const int ntiles = (int)((d + tile_cols - 1) / tile_cols);
  const bool whole = e_end - e_beg <= kChunk;
  int pcol[kPer];
  double pval[kPer];
  if (whole) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = e_beg + (int)threadIdx.x + k * kThreads;
      pcol[k] = e < e_end ? ecol[e] : -1;
      pval[k] = e < e_end ? eval[e] : 0.0;
    }
  }
  for (int t = 0; t < ntiles; ++t) {
    const int64_t c0 = (int64_t)t * tile_cols;
    const int c0i = (int)c0;  // d < 2^31
    const int width = (int)min((int64_t)tile_cols, d - c0);
    // acc is not zero-filled: the fast path zeroes the columns it touches and
    // the write-out emits 0 where word[] is 0 (the fallback fills acc itself)
    for (int i = threadIdx.x; i < width; i += kThreads) word[i] = 0;
    if (threadIdx.x == 0) {
      side_n = 0;
      fallback = !whole;
    }
    __syncthreads();
    if (whole) {
      // 1. multiplicity of every column of the tile
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int cc = pcol[k] - c0i;
        if (pcol[k] >= 0 && (unsigned)cc < (unsigned)width) {
          atomicAdd(&word[cc], 1);
          acc[cc] = 0.0;
        }
      }
      __syncthreads();
      // 2. one pair: store 0 + v; two pairs: two fp64 adds onto 0 in either order
      //    give (0 + a) + b == (0 + b) + a; more: to the side list
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int cc = pcol[k] - c0i;
        if (pcol[k] < 0 || (unsigned)cc >= (unsigned)width) continue;
        const int cnt = word[cc];
        if (cnt == 1) {
          acc[cc] = 0.0 + pval[k];
        } else if (cnt == 2) {
          atomicAdd(&acc[cc], pval[k]);
        } else {
          const int slot = atomicAdd(&side_n, 1);
          if (slot < kSideCap) {
            side_ci[slot] = cc;
            side_ix[slot] = (int)threadIdx.x + k * kThreads;
            side_v[slot] = pval[k];
          } else {
            fallback = 1;
          }
        }
      }
      __syncthreads();
      // 3. columns of >= 3 pairs: sort the side list by (column, index) (each
      //    entry's position = the number of entries before it), then the first
      //    entry of each column sums its run in list order
      const int ns = min(side_n, kSideCap);
      if (ns > 0 && !fallback) {
        double vi[kSideCap / kThreads];
        int pi[kSideCap / kThreads];
#pragma unroll
        for (int u = 0; u < kSideCap / kThreads; ++u) {
          const int i = (int)threadIdx.x + u * kThreads;
          pi[u] = -1;
          if (i >= ns) continue;
          const long long key = ((long long)side_ci[i] << 32) | (unsigned)side_ix[i];
          int pos = 0;
          for (int j = 0; j < ns; ++j) pos += (((long long)side_ci[j] << 32) | (unsigned)side_ix[j]) < key;
          pi[u] = pos;
          vi[u] = side_v[i];
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kSideCap / kThreads; ++u)
          if (pi[u] >= 0) {
            sorted_v[pi[u]] = vi[u];
            sorted_c[pi[u]] = side_ci[(int)threadIdx.x + u * kThreads];
          }
        __syncthreads();
        for (int p0 = threadIdx.x; p0 < ns; p0 += kThreads) {
          const int cc = sorted_c[p0];
          if (p0 > 0 && sorted_c[p0 - 1] == cc) continue;
          double sum = 0.0;
          for (int p = p0; p < ns && sorted_c[p] == cc; ++p) sum = sum + sorted_v[p];
          acc[cc] = sum;
        }
        __syncthreads();
      }
    }
    if (fallback) {  // uniform: read after a barrier
      for (int i = threadIdx.x; i < width; i += kThreads) {
        acc[i] = 0.0;
        word[i] = kFree;
      }
      for (int s0 = e_beg; s0 < e_end; s0 += kChunk) {
        int pc[kPer];
        double pv[kPer];
        unsigned pend = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
          const int e = s0 + (int)threadIdx.x + k * kThreads;
          pc[k] = 0;
          pv[k] = 0.0;
          if (e < e_end && e < s0 + kChunk) {
            const int cc = ecol[e] - c0i;
            if ((unsigned)cc < (unsigned)width) {
              pc[k] = cc;
              pv[k] = eval[e];
              pend |= 1u << k;
            }
          }
        }
        claim_rounds(acc, word, pc, pv, pend);  // starts with a barrier
      }
      __syncthreads();
    }
    double* o = SA + b * ldsa + c0;
    const bool vec = ((reinterpret_cast<uintptr_t>(o) & 15) == 0) && (width % 2 == 0);
    if (vec) {
      for (int i = threadIdx.x; i < width / 2; i += kThreads) {
        const double2 x = make_double2(word[2 * i] ? alpha * acc[2 * i] : 0.0,
                                       word[2 * i + 1] ? alpha * acc[2 * i + 1] : 0.0);
        *reinterpret_cast<double2*>(o + 2 * i) = x;
      }
    } else {
      for (int i = threadIdx.x; i < width; i += kThreads) o[i] = word[i] ? alpha * acc[i] : 0.0;
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
    csr_expand_kernel<<<(unsigned)(((N + kExpE - 1) / kExpE * 8 + 255) / 256), 256, 0, st>>>(
        N, sg, w.rst, col_idx, val, w.off, w.ecol, w.eval);
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
