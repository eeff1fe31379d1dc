// common.cuh -- device helpers shared by the libskh kernels (product side).
// Independent of oracle/: this is the CUDA implementation of the same
// counter-based generator (R1), written from the definition.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "../../include/skh.h"

namespace skh {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kLabelHash = 0x48415348ull;  // "HASH"
constexpr uint64_t kLabelDiag = 0x44494147ull;  // "DIAG"
constexpr int kMaxAttempts = 0xFFFF;            // attempts t = 0..0xFFFE
constexpr uint64_t kSignSlot = 0xFFFF;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// Output number ctr+1 of splitmix64 started at state `key`.
__host__ __device__ __forceinline__ uint64_t stream_u(uint64_t key, uint64_t ctr) {
  return mix64(key + (ctr + 1) * kGamma);
}

__host__ __device__ __forceinline__ uint64_t key_hash(uint64_t seed) { return mix64(seed ^ kLabelHash); }
__host__ __device__ __forceinline__ uint64_t key_diag(uint64_t seed) { return mix64(seed ^ kLabelDiag); }

// SKH_CHECK: device-side invariant checks of the checked build (SKH_CHECKED=1
// python -m paper_2105_11815_b200.build --force; tools/checked_suite.sh) --
// the stand-in for compute-sanitizer, which is closed on the GPU pool.  A
// failed check prints its location and traps (the launch fails, the caller
// gets SKH_ECUDA); the product build compiles them out.
#ifdef SKH_CHECKED
#define SKH_CHECK(c)                                                                     \
  do {                                                                                   \
    if (!(c)) {                                                                          \
      printf("SKH_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                         \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define SKH_CHECK(c) \
  do {               \
  } while (0)
#endif

// Local column k -> global column of S (see skh_hash_gen).
__host__ __device__ __forceinline__ int64_t row_map(int64_t k, int64_t row0, int64_t blk, int64_t stride) {
  return blk <= 0 ? row0 + k : row0 + (k / blk) * stride + (k % blk);
}

// Thread-local error message (api.cu).
void set_error(const char* fmt, ...);

int check_launch(const char* what);

// Process-wide count of kernels enqueued by libskh (skh_launch_count()).
void note_launch();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Kernel launchers (one per .cu file).
// dht.cu: Y[i * ldy + c] = X[c * ldx + i] (column-major n x d -> row-major), 64 x 64 tiles
void transpose_cm_to_rm(int64_t n, int64_t d, const double* X, int64_t ldx, double* Y, int64_t ldy, cudaStream_t st);

// hash.cu
size_t hash_ws_bytes(int64_t nrows, int64_t m, int s);
int launch_hash(uint64_t seed, int64_t m, int s, int64_t nrows, int64_t row0, int64_t blk,
                int64_t stride, int32_t* col_rows, int8_t* col_signs, int32_t* bucket_ptr,
                int32_t* bucket_rows, int8_t* bucket_signs, void* ws, size_t ws_bytes,
                cudaStream_t st);
int launch_hash_v(uint64_t seed, int64_t m, int s, int64_t nrows, int64_t row0, int64_t blk, int64_t stride,
                  int32_t* col_rows, int8_t* col_signs, int32_t* bucket_ptr, int32_t* bucket_rows,
                  int8_t* bucket_signs, void* ws, size_t ws_bytes, int variant, cudaStream_t st);
int hash_status(const void* ws, cudaStream_t st);
int64_t scan_scratch_ints(int64_t len);
int launch_excl_scan_i32(int32_t* a, int64_t len, int32_t* blocksums, cudaStream_t st);
// gather.cu
// s = nonzeros per row of S (the number of reads of each row): s > 1 takes the
// L2-slice lane-group kernel, s = 1 the 128-column wide kernel
int launch_gather_dense(int64_t m, const int32_t* ptr, const int32_t* rows, const int8_t* sg,
                        int64_t d, const double* A, int64_t lda, double* SA, int64_t ldsa,
                        double alpha, cudaStream_t st, int s = 2);
int launch_gather_vec(int64_t m, const int32_t* ptr, const int32_t* rows, const int8_t* sg,
                      const double* b, double* Sb, double alpha, cudaStream_t st);
// csr.cu
size_t csr_ws_bytes(int64_t nrows, int s, int64_t nnz);
int launch_gather_csr(int64_t m, int s, const int32_t* ptr, const int32_t* rows, const int8_t* sg,
                      int64_t nrows, int64_t d, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                      const double* val, double* SA, int64_t ldsa, double alpha, void* ws, cudaStream_t st);
// fwht.cu
size_t fwht_ws_bytes(int64_t nrows, int64_t nvalid, int64_t row0, int64_t d);
int launch_fwht(uint64_t seed, int64_t nrows, int64_t nvalid, int64_t row0, int64_t d,
                const double* X, int64_t ldx, double* Y, int64_t ldy, int bit_lo, int bit_hi,
                int apply_diag, double alpha, void* ws, cudaStream_t st);
// util (api.cu)
int launch_scale(double* X, int64_t rows, int64_t cols, int64_t ldx, double alpha, cudaStream_t st);

// api_cm.cu: stage trace (skh_trace_set) -- records the caller's event after a stage
void skh_trace_mark(cudaStream_t st, const char* name);
void skh_trace_start(cudaStream_t st);
// api.cu: library-owned copy stream of the current device (host-buffer variants)
cudaStream_t skh_copy_stream();
// api.cu: per-thread side stream; fork = it waits for `st`, join = `st` waits for it
cudaStream_t skh_side_fork(cudaStream_t st);
int skh_side_join(cudaStream_t st, cudaStream_t side);

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

}  // namespace skh
