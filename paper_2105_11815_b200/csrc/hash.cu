// hash.cu -- R1 (draw S_h) and R2 (transpose into bucket lists).
//
// R1: one thread per local column k of S (= row of A): s distinct rows of
//     [0, m) by rejection on the splitmix64 stream, signs from one extra word
//     (Def. def::sampling_and_hashing; R1-R4).
// R2: a stable LSD radix sort of the n*s entries by bucket id (8-bit digits).
//     The entries enter in ascending local column, so stability leaves every
//     bucket's list in ascending column: the canonical order of DESIGN.md R6.
//     Block-stable ranking uses warp __match_any_sync + per-warp digit cursors,
//     so the result is deterministic (no order-dependent atomics on outputs).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kItemsPerWarp = 512;
constexpr int kTile = kSortWarps * kItemsPerWarp;  // 4096 entries per CTA
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanChunk = kScanThreads * kScanItems;

struct HashWs {
  int32_t* status;
  uint64_t* keys_a;
  uint64_t* keys_b;
  int32_t* hist;       // [256 * ntiles]
  int32_t* blocksums;  // scan scratch
  int64_t ntiles;
};

inline int64_t ntiles_of(int64_t N) { return (N + kTile - 1) / kTile; }
inline int64_t scan_blocks(int64_t len) { return (len + kScanChunk - 1) / kScanChunk; }

HashWs carve(void* ws, int64_t N) {
  HashWs w;
  char* p = static_cast<char*>(ws);
  w.status = reinterpret_cast<int32_t*>(p);
  p += 256;
  w.keys_a = reinterpret_cast<uint64_t*>(p);
  p += align_up(sizeof(uint64_t) * (size_t)N);
  w.keys_b = reinterpret_cast<uint64_t*>(p);
  p += align_up(sizeof(uint64_t) * (size_t)N);
  w.ntiles = ntiles_of(N);
  w.hist = reinterpret_cast<int32_t*>(p);
  p += align_up(sizeof(int32_t) * 256 * (size_t)w.ntiles);
  w.blocksums = reinterpret_cast<int32_t*>(p);
  return w;
}

// ---------------------------------------------------------------- R1 kernel
template <int MAXS>
__global__ void hash_kernel(uint64_t key, int64_t m, int s, int64_t nrows, int64_t row0, int64_t blk,
                            int64_t stride, int32_t* __restrict__ col_rows, int8_t* __restrict__ col_signs,
                            uint64_t* __restrict__ keys, int32_t* __restrict__ status, int variant) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nrows) return;
  const uint64_t j = (uint64_t)row_map(k, row0, blk, stride);
  const uint64_t base = j << 16;
  uint32_t acc[MAXS];
  int na = 0;
  int t = 0;
  while (na < s) {
    if (t >= kMaxAttempts) {  // practically unreachable for s <= m; keep arrays consistent
      atomicOr(status, 1);
      for (uint32_t r = 0; na < s; ++r) {
        bool dup = false;
#pragma unroll
        for (int q = 0; q < MAXS; ++q)
          if (q < na) dup |= (acc[q] == r);
        if (!dup) {
#pragma unroll
          for (int q = 0; q < MAXS; ++q)
            if (q == na) acc[q] = r;
          ++na;
        }
      }
      break;
    }
    const uint64_t u = stream_u(key, base + (uint64_t)t);
    const uint32_t r = (uint32_t)__umul64hi(u, (uint64_t)m);
    bool dup = false;  // the s-hashing variant (Def. 7) keeps every draw
#pragma unroll
    for (int q = 0; q < MAXS; ++q)
      if (q < na) dup |= (acc[q] == r);
    if (variant || !dup) {
#pragma unroll
      for (int q = 0; q < MAXS; ++q)
        if (q == na) acc[q] = r;
      ++na;
    }
    ++t;
  }
  const uint64_t w = stream_u(key, base + kSignSlot);
#pragma unroll
  for (int q = 0; q < MAXS; ++q) {
    if (q < s) {
      const uint32_t neg = (uint32_t)((w >> q) & 1ull);
      const int64_t e = k * s + q;
      if (col_rows) col_rows[e] = (int32_t)acc[q];
      if (col_signs) col_signs[e] = neg ? (int8_t)-1 : (int8_t)1;
      // the radix sort is stable in the bucket digits only: a variant column's
      // coincident draws must enter + before - (R18), so its keys are placed by
      // their rank in (row, sign) order; for s-hashing the rows are distinct and
      // the order is irrelevant
      int pos = q;
      if (variant) {
        const uint64_t kq = ((uint64_t)acc[q] << 1) | neg;
        pos = 0;
#pragma unroll
        for (int q2 = 0; q2 < MAXS; ++q2) {
          if (q2 < s) {
            const uint64_t k2 = ((uint64_t)acc[q2] << 1) | ((w >> q2) & 1ull);
            pos += (k2 < kq) || (k2 == kq && q2 < q);
          }
        }
      }
      keys[k * s + pos] = ((uint64_t)acc[q] << 32) | ((uint64_t)((uint32_t)k << 1)) | neg;
    }
  }
}

// ---------------------------------------------------------------- scan (int32, exclusive, in place)
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total in *total.
__device__ int block_excl_scan(int v, int* total) {
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = warp_incl_scan(v);
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int nw = blockDim.x >> 5;
    int x = lane < nw ? wsum[lane] : 0;
    int xi = warp_incl_scan(x);
    if (lane < nw) wsum[lane] = xi - x;
    if (lane == nw - 1) *total = xi;
  }
  __syncthreads();
  int r = inc - v + wsum[wid];
  __syncthreads();
  return r;
}

__global__ void scan_reduce_kernel(const int32_t* __restrict__ a, int64_t len, int32_t* __restrict__ bs) {
  __shared__ int tot;
  const int64_t base = (int64_t)blockIdx.x * kScanChunk;
  int v = 0;
  for (int i = 0; i < kScanItems; ++i) {
    int64_t e = base + (int64_t)threadIdx.x * kScanItems + i;
    if (e < len) v += a[e];
  }
  block_excl_scan(v, &tot);
  if (threadIdx.x == 0) bs[blockIdx.x] = tot;
}

__global__ void scan_single_kernel(int32_t* __restrict__ bs, int64_t nb) {
  // exclusive scan of nb block sums by one CTA, sequential chunks per thread
  __shared__ int tot;
  const int64_t per = (nb + blockDim.x - 1) / blockDim.x;
  const int64_t lo = (int64_t)threadIdx.x * per;
  int v = 0;
  for (int64_t i = lo; i < lo + per && i < nb; ++i) v += bs[i];
  int off = block_excl_scan(v, &tot);
  for (int64_t i = lo; i < lo + per && i < nb; ++i) {
    int x = bs[i];
    bs[i] = off;
    off += x;
  }
}

__global__ void scan_apply_kernel(int32_t* __restrict__ a, int64_t len, const int32_t* __restrict__ bs) {
  __shared__ int tot;
  const int64_t base = (int64_t)blockIdx.x * kScanChunk + (int64_t)threadIdx.x * kScanItems;
  int x[kScanItems];
  int v = 0;
  for (int i = 0; i < kScanItems; ++i) {
    x[i] = (base + i < len) ? a[base + i] : 0;
    v += x[i];
  }
  int off = block_excl_scan(v, &tot) + bs[blockIdx.x];
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < len) a[base + i] = off;
    off += x[i];
  }
}

int excl_scan(int32_t* a, int64_t len, int32_t* bs, cudaStream_t st) {
  const int64_t nb = scan_blocks(len);
  if (nb == 0) return SKH_OK;
  scan_reduce_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(a, len, bs); note_launch();
  scan_single_kernel<<<1, kScanThreads, 0, st>>>(bs, nb); note_launch();
  scan_apply_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(a, len, bs); note_launch();
  return check_launch("scan");
}

// ---------------------------------------------------------------- radix passes
__device__ __forceinline__ int digit_of(uint64_t key, int shift) { return (int)((key >> (32 + shift)) & 0xFFu); }

__global__ void __launch_bounds__(kSortThreads) upsweep_kernel(const uint64_t* __restrict__ keys, int64_t N,
                                                               int shift, int32_t* __restrict__ hist,
                                                               int64_t ntiles) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
  for (int i = threadIdx.x; i < kTile; i += kSortThreads) {
    int64_t e = base + i;
    if (e < N) atomicAdd(&h[digit_of(keys[e], shift)], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads) downsweep_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                                 int64_t N, int shift, const int32_t* __restrict__ gofs,
                                                                 int64_t ntiles) {
  __shared__ int wcnt[kSortWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * kTile + (int64_t)w * kItemsPerWarp;
  // the warp's 512 keys in registers (16 per lane, all loads in flight at once):
  // the ranking loop below is sequential over chunks and must not wait on memory
  constexpr int kR = kItemsPerWarp / 32;
  uint64_t kv[kR];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int64_t e = wbase + r * 32 + lane;
    kv[r] = e < N ? in[e] : 0;
  }
#pragma unroll
  for (int r = 0; r < kR; ++r)
    if (wbase + r * 32 + lane < N) atomicAdd(&wcnt[w][digit_of(kv[r], shift)], 1);
  __syncthreads();
  {
    const int dg = threadIdx.x;  // 256 threads = 256 digits
    int run = gofs[(int64_t)dg * ntiles + blockIdx.x];
    for (int q = 0; q < kSortWarps; ++q) {
      int c = wcnt[q][dg];
      wcnt[q][dg] = run;
      run += c;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int64_t e = wbase + r * 32 + lane;
    const bool valid = e < N;
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    if (vmask == 0) break;
    const uint64_t key = kv[r];
    int dg = 0, rank = 0, base = 0;
    unsigned peers = 0;
    if (valid) {
      dg = digit_of(key, shift);
      peers = __match_any_sync(vmask, dg);
      rank = __popc(peers & lt);
      base = wcnt[w][dg];
    }
    __syncwarp();
    if (valid) {
      out[base + rank] = key;
      if (rank == 0) wcnt[w][dg] = base + __popc(peers);
    }
    __syncwarp();
  }
}

__global__ void finalize_kernel(const uint64_t* __restrict__ keys, int64_t N, int64_t m,
                                int32_t* __restrict__ bucket_ptr, int32_t* __restrict__ bucket_rows,
                                int8_t* __restrict__ bucket_signs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N) return;
  const uint64_t key = keys[t];
  const int64_t b = (int64_t)(key >> 32);
  SKH_CHECK(b < m && (t == 0 || (int64_t)(keys[t - 1] >> 32) <= b));  // sorted bucket ids in [0, m)
  const uint32_t lo = (uint32_t)key;
  bucket_rows[t] = (int32_t)(lo >> 1);
  bucket_signs[t] = (lo & 1u) ? (int8_t)-1 : (int8_t)1;
  const int64_t prev = t > 0 ? (int64_t)(keys[t - 1] >> 32) : -1;
  for (int64_t bb = prev + 1; bb <= b; ++bb) bucket_ptr[bb] = (int32_t)t;
  if (t == N - 1)
    for (int64_t bb = b + 1; bb <= m; ++bb) bucket_ptr[bb] = (int32_t)N;
}

__global__ void fill_i32_kernel(int32_t* p, int64_t n, int32_t v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace

namespace {

// ---------------------------------------------------------------- R2, segmented path
// For the usual shapes (m >= 64 buckets of <= ~512 entries on average) the
// transpose is: count entries per bucket (atomics on integers: order-free), one
// scan to bucket_ptr, an unordered fill through per-bucket cursors, then a
// per-bucket sort of the (row << 1 | sign) keys, which restores the canonical
// ascending-row order (R6) -- 4 kernels instead of 5 per 8-bit radix
// digit.  The result is unique, so it equals the radix path bit for bit.
constexpr int kSegCap = 1024;  // entries sorted in shared memory per warp

template <int MAXS>
__global__ void hash_count_kernel(uint64_t key, int64_t m, int s, int64_t nrows, int64_t row0, int64_t blk,
                                  int64_t stride, int32_t* __restrict__ col_rows, int8_t* __restrict__ col_signs,
                                  int32_t* __restrict__ ebucket, uint32_t* __restrict__ ekey,
                                  int32_t* __restrict__ counts, int32_t* __restrict__ status, int variant) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nrows) return;
  const uint64_t j = (uint64_t)row_map(k, row0, blk, stride);
  const uint64_t base = j << 16;
  uint32_t acc[MAXS];
  int na = 0;
  for (int t = 0; na < s; ++t) {
    uint32_t r;
    if (t < kMaxAttempts) {
      r = (uint32_t)__umul64hi(stream_u(key, base + (uint64_t)t), (uint64_t)m);
    } else {  // unreachable in practice (see hash_kernel): smallest unused row
      atomicOr(status, 1);
      r = 0;
      for (;;) {
        bool dup = false;
#pragma unroll
        for (int q = 0; q < MAXS; ++q)
          if (q < na) dup |= (acc[q] == r);
        if (!dup) break;
        ++r;
      }
    }
    bool dup = false;  // the s-hashing variant (Def. 7) keeps every draw
#pragma unroll
    for (int q = 0; q < MAXS; ++q)
      if (q < na) dup |= (acc[q] == r);
    if (variant || !dup) {
#pragma unroll
      for (int q = 0; q < MAXS; ++q)
        if (q == na) acc[q] = r;
      ++na;
    }
  }
  const uint64_t w = stream_u(key, base + kSignSlot);
#pragma unroll
  for (int q = 0; q < MAXS; ++q) {
    if (q < s) {
      const uint32_t neg = (uint32_t)((w >> q) & 1ull);
      const int64_t e = k * s + q;
      if (col_rows) col_rows[e] = (int32_t)acc[q];
      if (col_signs) col_signs[e] = neg ? (int8_t)-1 : (int8_t)1;
      ebucket[e] = (int32_t)acc[q];
      ekey[e] = ((uint32_t)k << 1) | neg;
      atomicAdd(&counts[acc[q]], 1);
    }
  }
}

// exclusive scan of counts[0..m) into ptr[0..m] and cursor[0..m), one CTA
__global__ void __launch_bounds__(1024) scan_counts_kernel(const int32_t* __restrict__ counts, int64_t m,
                                                           int32_t* __restrict__ ptr, int32_t* __restrict__ cursor) {
  __shared__ int tot;
  const int64_t per = (m + 1023) / 1024;
  const int64_t lo = (int64_t)threadIdx.x * per;
  int v = 0;
  for (int64_t i = lo; i < lo + per && i < m; ++i) v += counts[i];
  int off = block_excl_scan(v, &tot);
  for (int64_t i = lo; i < lo + per && i < m; ++i) {
    ptr[i] = off;
    cursor[i] = off;
    off += counts[i];
  }
  if (threadIdx.x == 0) ptr[m] = tot;
}

__global__ void fill_kernel(int64_t N, const int32_t* __restrict__ ebucket, const uint32_t* __restrict__ ekey,
                            int32_t* __restrict__ cursor, uint32_t* __restrict__ tmp) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  const int pos = atomicAdd(&cursor[ebucket[e]], 1);
  tmp[pos] = ekey[e];
}

// one warp per bucket: bitonic sort of the bucket's keys in shared memory
__global__ void __launch_bounds__(256) segsort_kernel(int64_t m, const int32_t* __restrict__ ptr,
                                                      const uint32_t* __restrict__ tmp, int32_t* __restrict__ rows,
                                                      int8_t* __restrict__ signs) {
  __shared__ uint32_t buf[8][kSegCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * 8 + w;
  if (b >= m) return;
  const int beg = ptr[b], L = ptr[b + 1] - beg;
  if (L <= kSegCap) {
    int P = 1;
    while (P < L) P <<= 1;
    uint32_t* s = buf[w];
    for (int i = lane; i < P; i += 32) s[i] = i < L ? tmp[beg + i] : 0xFFFFFFFFu;
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1) {
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        for (int i = lane; i < P; i += 32) {
          const int ixj = i ^ jj;
          if (ixj > i) {
            const uint32_t a = s[i], c = s[ixj];
            const bool up = (i & k) == 0;
            if ((a > c) == up) {
              s[i] = c;
              s[ixj] = a;
            }
          }
        }
        __syncwarp();
      }
    }
    for (int i = lane; i < L; i += 32) {
      const uint32_t x = s[i];
      rows[beg + i] = (int32_t)(x >> 1);
      signs[beg + i] = (x & 1u) ? (int8_t)-1 : (int8_t)1;
    }
  } else {
    // oversized bucket (not expected for the shapes that take this path):
    // rank sort straight from global memory, keys are distinct
    for (int i = lane; i < L; i += 32) {
      const uint32_t x = tmp[beg + i];
      int rank = 0;  // equal keys (a variant row drawn twice with one sign) by position
      for (int jx = 0; jx < L; ++jx) rank += tmp[beg + jx] < x || (tmp[beg + jx] == x && jx < i);
      rows[beg + rank] = (int32_t)(x >> 1);
      signs[beg + rank] = (x & 1u) ? (int8_t)-1 : (int8_t)1;
    }
  }
}

bool use_segmented(int64_t N, int64_t m) {
  // measured: faster than the radix path up to ~64 entries per bucket (C1-C3),
  // slower at 192-292 (C4, C5) where the warp bitonic sorts and the per-bucket
  // atomics dominate
  return m >= 64 && m <= (1 << 20) && N <= 96 * m;
}

int launch_hash_seg(uint64_t seed, int64_t m, int s, int64_t nrows, int64_t row0, int64_t blk, int64_t stride,
                    int32_t* col_rows, int8_t* col_signs, int32_t* bucket_ptr, int32_t* bucket_rows,
                    int8_t* bucket_signs, const HashWs& w, int32_t* counts, int variant, cudaStream_t st) {
  const int64_t N = nrows * (int64_t)s;
  int32_t* ebucket = reinterpret_cast<int32_t*>(w.keys_a);
  uint32_t* ekey = reinterpret_cast<uint32_t*>(w.keys_a) + N;
  uint32_t* tmp = reinterpret_cast<uint32_t*>(w.keys_b);
  int32_t* cursor = counts + m;
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)m, st);
  const uint64_t key = key_hash(seed);
  const unsigned hb = (unsigned)((nrows + 255) / 256);
#define SKH_HC(MS)                                                                                               \
  hash_count_kernel<MS><<<hb, 256, 0, st>>>(key, m, s, nrows, row0, blk, stride, col_rows, col_signs, ebucket, \
                                            ekey, counts, w.status, variant)
  if (s <= 1) SKH_HC(1);
  else if (s <= 2) SKH_HC(2);
  else if (s <= 4) SKH_HC(4);
  else if (s <= 8) SKH_HC(8);
  else SKH_HC(64);
#undef SKH_HC
  note_launch();
  scan_counts_kernel<<<1, 1024, 0, st>>>(counts, m, bucket_ptr, cursor);
  note_launch();
  fill_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, ebucket, ekey, cursor, tmp);
  note_launch();
  segsort_kernel<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(m, bucket_ptr, tmp, bucket_rows, bucket_signs);
  note_launch();
  return check_launch("hash_seg");
}

}  // namespace

// Exclusive scan of int32 a[0..len) in place; blocksums needs scan_scratch_ints(len).
int64_t scan_scratch_ints(int64_t len) { return scan_blocks(len) + 1; }
int launch_excl_scan_i32(int32_t* a, int64_t len, int32_t* blocksums, cudaStream_t st) {
  return excl_scan(a, len, blocksums, st);
}

size_t hash_ws_bytes(int64_t nrows, int64_t m, int s) {
  const int64_t N = nrows * (int64_t)s;
  const int64_t nt = ntiles_of(N);
  return 256 + 2 * align_up(sizeof(uint64_t) * (size_t)N) + align_up(sizeof(int32_t) * 256 * (size_t)nt) +
         align_up(sizeof(int32_t) * (size_t)(scan_blocks(256 * nt) + 1)) +
         align_up(sizeof(int32_t) * (size_t)(2 * m + 1));
}

int launch_hash(uint64_t seed, int64_t m, int s, int64_t nrows, int64_t row0, int64_t blk, int64_t stride,
                int32_t* col_rows, int8_t* col_signs, int32_t* bucket_ptr, int32_t* bucket_rows,
                int8_t* bucket_signs, void* ws, size_t ws_bytes, cudaStream_t st) {
  return launch_hash_v(seed, m, s, nrows, row0, blk, stride, col_rows, col_signs, bucket_ptr, bucket_rows,
                       bucket_signs, ws, ws_bytes, 0, st);
}

// variant != 0: the s-hashing variant (Def. def::s-hashing-variant, PAPER.md
// L683-686): the s draws r_t, t = 0..s-1, are all kept (with replacement); a
// row drawn twice appears twice in its bucket, + before - (R18).
int launch_hash_v(uint64_t seed, int64_t m, int s, int64_t nrows, int64_t row0, int64_t blk, int64_t stride,
                  int32_t* col_rows, int8_t* col_signs, int32_t* bucket_ptr, int32_t* bucket_rows,
                  int8_t* bucket_signs, void* ws, size_t ws_bytes, int variant, cudaStream_t st) {
  const int64_t N = nrows * (int64_t)s;
  HashWs w = carve(ws, N);
  int32_t* counts = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + hash_ws_bytes(nrows, m, s) -
                                               align_up(sizeof(int32_t) * (size_t)(2 * m + 1)));
  (void)ws_bytes;
  static const bool force_radix = [] {
    const char* e = getenv("SKH_HASH_RADIX");
    return e && atoi(e) != 0;
  }();
  static const bool force_seg = [] {  // measurement switch: the segmented path at any bucket size
    const char* e = getenv("SKH_HASH_SEG");
    return e && atoi(e) != 0;
  }();
  if (N > 0 && !force_radix && (use_segmented(N, m) || (force_seg && m >= 64 && m <= (1 << 20)))) {
    cudaMemsetAsync(w.status, 0, sizeof(int32_t), st);
    return launch_hash_seg(seed, m, s, nrows, row0, blk, stride, col_rows, col_signs, bucket_ptr, bucket_rows,
                           bucket_signs, w, counts, variant, st);
  }
  cudaMemsetAsync(w.status, 0, sizeof(int32_t), st);
  if (N == 0) {
    fill_i32_kernel<<<(unsigned)((m + 1 + 255) / 256), 256, 0, st>>>(bucket_ptr, m + 1, 0); note_launch();
    return check_launch("hash(empty)");
  }
  const uint64_t key = key_hash(seed);
  const unsigned hb = (unsigned)((nrows + 255) / 256);
#define SKH_HASH_LAUNCH(MS) \
  hash_kernel<MS><<<hb, 256, 0, st>>>(key, m, s, nrows, row0, blk, stride, col_rows, col_signs, w.keys_a, w.status, \
                                      variant)
  if (s <= 1) SKH_HASH_LAUNCH(1);
  else if (s <= 2) SKH_HASH_LAUNCH(2);
  else if (s <= 4) SKH_HASH_LAUNCH(4);
  else if (s <= 8) SKH_HASH_LAUNCH(8);
  else SKH_HASH_LAUNCH(64);
  note_launch();
#undef SKH_HASH_LAUNCH
  int rc = check_launch("hash_kernel");
  if (rc) return rc;
  // number of 8-bit digit passes covering bucket ids 0..m-1
  int bits = 0;
  while (bits < 31 && ((int64_t)1 << bits) < m) ++bits;
  const int passes = (bits + 7) / 8;
  uint64_t* src = w.keys_a;
  uint64_t* dst = w.keys_b;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    upsweep_kernel<<<(unsigned)w.ntiles, kSortThreads, 0, st>>>(src, N, shift, w.hist, w.ntiles); note_launch();
    rc = excl_scan(w.hist, 256 * w.ntiles, w.blocksums, st);
    if (rc) return rc;
    downsweep_kernel<<<(unsigned)w.ntiles, kSortThreads, 0, st>>>(src, dst, N, shift, w.hist, w.ntiles); note_launch();
    rc = check_launch("radix pass");
    if (rc) return rc;
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  finalize_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(src, N, m, bucket_ptr, bucket_rows, bucket_signs); note_launch();
  return check_launch("finalize");
}

int hash_status(const void* ws, cudaStream_t st) {
  int32_t v = 0;
  if (cudaMemcpyAsync(&v, ws, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess) return SKH_ECUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return SKH_ECUDA;
  return v ? SKH_ERETRY : SKH_OK;
}

}  // namespace skh
