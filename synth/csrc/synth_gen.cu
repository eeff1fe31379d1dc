// synth_gen.cu -- device implementation of the seeded input recipe of
// synth/gen.py (harness code, not part of libskh).  Integer-exact: values are
// bit-identical to the NumPy generator (tests/test_synth_device.py).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t LABEL_A = 0x41, LABEL_B = 0x42, LABEL_DIAGU = 0x55, LABEL_CSR_COL = 0x43, LABEL_CSR_VAL = 0x56,
                   LABEL_INT = 0x49;

__host__ __device__ __forceinline__ uint64_t mixS(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t label) { return mixS(seed ^ (label << 32)); }
__device__ __forceinline__ uint64_t word(uint64_t key, uint64_t ctr) { return mixS(key + (ctr + 1) * kGamma); }

__device__ __forceinline__ double normal_at(uint64_t key, uint64_t idx) {
  uint64_t acc = 0;
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    const uint64_t w = word(key, idx * 6 + t);
    acc += (w & 0xFFFFFFFFull) + (w >> 32);
  }
  const int64_t v = (int64_t)acc - (int64_t)(6ull << 32);
  return __dmul_rn((double)v, 2.3283064365386963e-10);  // 2^-32, exact
}

__device__ __forceinline__ double uniform01_at(uint64_t key, uint64_t idx) {
  return __dmul_rn((double)(word(key, idx) >> 11), 1.1102230246251565e-16);  // 2^-53
}

// kind 0: iid normal; kind 1: coherent (1e-8 normal + U(1,10) on the diagonal i < min(n, d))
__global__ void dense_kernel(int kind, uint64_t seed, int64_t n_total, int64_t d, int64_t row0, int64_t nrows,
                             double* __restrict__ out, int64_t ld) {
  const uint64_t ka = stream_key(seed, LABEL_A), ku = stream_key(seed, LABEL_DIAGU);
  const int64_t total = nrows * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d, c = e % d, gi = row0 + i;
    double v = normal_at(ka, (uint64_t)(gi * d + c));
    if (kind == 1) {
      v = __dmul_rn(1e-8, v);
      if (gi == c && gi < (n_total < d ? n_total : d)) {
        const double dv = __dadd_rn(1.0, __dmul_rn(9.0, uniform01_at(ku, (uint64_t)gi)));
        v = __dadd_rn(dv, v);
      }
    }
    out[i * ld + c] = v;
  }
}

// Same values, column-major: out[c * ld + i] (i fastest, coalesced writes).
__global__ void dense_cm_kernel(int kind, uint64_t seed, int64_t n_total, int64_t d, int64_t row0, int64_t nrows,
                                double* __restrict__ out, int64_t ld) {
  const uint64_t ka = stream_key(seed, LABEL_A), ku = stream_key(seed, LABEL_DIAGU);
  const int64_t total = nrows * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / nrows, i = e % nrows, gi = row0 + i;
    double v = normal_at(ka, (uint64_t)(gi * d + c));
    if (kind == 1) {
      v = __dmul_rn(1e-8, v);
      if (gi == c && gi < (n_total < d ? n_total : d)) {
        const double dv = __dadd_rn(1.0, __dmul_rn(9.0, uniform01_at(ku, (uint64_t)gi)));
        v = __dadd_rn(dv, v);
      }
    }
    out[c * ld + i] = v;
  }
}

__global__ void rhs_kernel(uint64_t seed, int64_t row0, int64_t n, double* __restrict__ out) {
  const uint64_t kb = stream_key(seed, LABEL_B);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = normal_at(kb, (uint64_t)(row0 + i));
}

__global__ void csr_kernel(uint64_t seed, int64_t d, int k, int64_t row0, int64_t nrows, int64_t* __restrict__ row_ptr,
                           int32_t* __restrict__ col_idx, double* __restrict__ val, int* __restrict__ fail) {
  const uint64_t kc = stream_key(seed, LABEL_CSR_COL), kv = stream_key(seed, LABEL_CSR_VAL);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > nrows) return;
  row_ptr[i] = i * k;
  if (i == nrows) return;
  const uint64_t gi = (uint64_t)(row0 + i);
  int cols[64];
  int na = 0;
  for (int t = 0; na < k; ++t) {
    if (t >= 256) {
      atomicOr(fail, 1);
      break;
    }
    const uint64_t w = word(kc, (gi << 8) + (uint64_t)t);
    const int c = (int)(((w >> 32) * (uint64_t)d) >> 32);
    bool dup = false;
    for (int q = 0; q < na; ++q) dup |= cols[q] == c;
    if (!dup) cols[na++] = c;
  }
  for (int a = 1; a < na; ++a) {  // insertion sort
    const int x = cols[a];
    int b = a - 1;
    while (b >= 0 && cols[b] > x) {
      cols[b + 1] = cols[b];
      --b;
    }
    cols[b + 1] = x;
  }
  for (int q = 0; q < k; ++q) {
    col_idx[i * k + q] = q < na ? cols[q] : 0;
    val[i * k + q] = normal_at(kv, gi * (uint64_t)k + (uint64_t)q);
  }
}

__global__ void small_int_kernel(uint64_t seed, int64_t n, int64_t d, int lo, int hi, double* __restrict__ out) {
  const uint64_t key = stream_key(seed, LABEL_INT);
  const uint64_t span = (uint64_t)(hi - lo + 1);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * d; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t w = word(key, (uint64_t)e);
    out[e] = (double)((int64_t)(((w >> 32) * span) >> 32) + lo);
  }
}

unsigned grid_for(int64_t work) {
  int64_t g = (work + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace

extern "C" {

int synth_dense(int kind, uint64_t seed, int64_t n_total, int64_t d, int64_t row0, int64_t nrows, double* out,
                int64_t ld, void* stream) {
  if (nrows <= 0) return 0;
  dense_kernel<<<grid_for(nrows * d), 256, 0, (cudaStream_t)stream>>>(kind, seed, n_total, d, row0, nrows, out, ld);
  return cudaGetLastError() == cudaSuccess ? 0 : 7;
}

int synth_dense_cm(int kind, uint64_t seed, int64_t n_total, int64_t d, int64_t row0, int64_t nrows, double* out,
                   int64_t ld, void* stream) {
  if (nrows <= 0) return 0;
  dense_cm_kernel<<<grid_for(nrows * d), 256, 0, (cudaStream_t)stream>>>(kind, seed, n_total, d, row0, nrows, out,
                                                                          ld);
  return cudaGetLastError() == cudaSuccess ? 0 : 7;
}

int synth_rhs(uint64_t seed, int64_t row0, int64_t n, double* out, void* stream) {
  if (n <= 0) return 0;
  rhs_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(seed, row0, n, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 7;
}

int synth_csr(uint64_t seed, int64_t d, int k, int64_t row0, int64_t nrows, int64_t* row_ptr, int32_t* col_idx,
              double* val, int* fail, void* stream) {
  if (k > 64 || k > d) return 1;
  csr_kernel<<<(unsigned)((nrows + 1 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(seed, d, k, row0, nrows, row_ptr,
                                                                                    col_idx, val, fail);
  return cudaGetLastError() == cudaSuccess ? 0 : 7;
}

int synth_small_int(uint64_t seed, int64_t n, int64_t d, int lo, int hi, double* out, void* stream) {
  if (n * d <= 0) return 0;
  small_int_kernel<<<grid_for(n * d), 256, 0, (cudaStream_t)stream>>>(seed, n, d, lo, hi, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 7;
}

}  // extern "C"
