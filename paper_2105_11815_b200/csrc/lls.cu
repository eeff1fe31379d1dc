// lls.cu -- Algorithm 1 Steps 2-5: the sketch-preconditioned
// least-squares solve that consumes SA and Sb.
//
//  Step 2  SA = Q R (full-rank Householder QR, the Blendenpik/DGEQRF mode the
//          paper allows, L1077; reading R19): cuSOLVER dgeqrf on a
//          column-major copy of SA -- a small dense factorisation (m x d).
//          Rank-revealing mode (skh_lls_solve_rr; the paper's default R-CPQR
//          with p = max{q : |r~_qq| >= rcond}, L1076-1077, L1109-1112; reading
//          R22): SA = Q0 R0 as above, then a column-pivoted Householder QR of
//          the d x d factor, R0 P = Q1 R~ (cpqr_kernel, ours), so SA P = (Q0 Q1) R~
//          -- the pivots of a CPQR of SA itself, since Q0 preserves column norms.
//          W = A V1 R11^{-1} is applied through N = P [R11^{-1} 0; 0 0] as a
//          d x d GEMV (the R^{-1}-as-matrix path below).
//  Step 3  x_s = R^{-1} Q^T Sb (cuSOLVER dormqr + cuBLAS dtrsv, a back-solve,
//          L1081); stop if ||A x_s - b|| <= tau_a.
//  Step 4  LSQR (Paige & Saunders) on W = A R^{-1} from y = 0, stopped by the
//          (7.1) estimate ||W^T r|| / (||W|| ||r||) <= tau_r (L1085-1089) or
//          it_max.  Every iteration streams A twice -- u <- A (R^{-1} v) - alpha u
//          and v <- R^{-T} (A^T u) - beta v -- through the two HBM-bound kernels
//          below; the d x d triangular solves are cuBLAS dtrsv; the whole loop
//          is one CUDA-graph launch (WHILE conditional node, scalar recurrence
//          on the device), with a host-driven loop as fallback.
//  Step 5  x = R^{-1} y.
//
// Kernels (ours, deterministic: every reduction has a fixed order):
//  gemv_n_kernel   out[i] = A[i,:] . t + beta * yin[i] for row-major A, one warp
//                  per row (512-byte coalesced row segments, t staged in shared
//                  memory), plus per-CTA partial sums of out[i]^2;
//  gemv_t_kernel   partial[g][c] = sum_{i in row block g} A[i,c] u[i]: a CTA owns
//                  a row block x 512-column tile, each thread two columns, rows
//                  streamed 8 at a time; colsum_kernel adds the partials in g
//                  order;
//  cm_av_kernel / cm_atu_kernel  the same two products for column-major A
//                  (skh_lls_solve_colmajor): one thread per row over the
//                  columns in order; per-column dot products over 4096-row
//                  blocks (u staged in shared memory) + colsum;
//  norm / vector kernels on n- and d-vectors.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cusolverDn.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace skh {
namespace {

constexpr int kRowsPerCta = 8;   // gemv_n: one warp per row, 8 warps
constexpr int kTCols = 512;      // gemv_t column tile (256 threads x 2 columns)
constexpr int kTRows = 8;        // gemv_t rows in flight per thread
constexpr int kMaxSmemX = 12288; // gemv_n stages t in shared memory up to this d

// out[i] = dot(A[i,:], t) + beta * yin[i]; sq[blockIdx] = sum over the CTA's rows of out^2
template <bool SMEM>
__global__ void __launch_bounds__(256) gemv_n_kernel(int64_t n, int64_t d, const double* __restrict__ A, int64_t lda,
                                                     const double* __restrict__ t, double beta,
                                                     const double* yin, double* out, double* __restrict__ sq,
                                                     int64_t rows_per_cta, const double* bdev) {
  extern __shared__ double ts[];
  if (bdev) beta = *bdev;  // device-resident coefficient (graph-captured LSQR)
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  if (SMEM) {
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) ts[c] = t[c];
    __syncthreads();
  }
  const double* tv = SMEM ? ts : t;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(n, r0 + rows_per_cta);
  const bool vec = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 2 == 0) && (d % 2 == 0);
  double wsq = 0.0;
  for (int64_t i = r0 + wp; i < r1; i += kRowsPerCta) {
    const double* a = A + i * lda;
    double acc0 = 0.0, acc1 = 0.0;
    if (vec) {
      const double2* a2 = reinterpret_cast<const double2*>(a);
      for (int64_t c2 = lane; c2 < d / 2; c2 += 32) {
        const double2 v = __ldg(a2 + c2);
        acc0 = fma(v.x, tv[2 * c2], acc0);
        acc1 = fma(v.y, tv[2 * c2 + 1], acc1);
      }
    } else {
      for (int64_t c = lane; c < d; c += 32) acc0 = fma(__ldg(a + c), tv[c], acc0);
    }
    double acc = acc0 + acc1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const double o = yin ? fma(beta, yin[i], acc) : acc;
      out[i] = o;
      wsq = fma(o, o, wsq);
    }
  }
  __shared__ double part[kRowsPerCta];
  if (lane == 0) part[wp] = wsq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kRowsPerCta; ++w) s += part[w];
    sq[blockIdx.x] = s;
  }
}

// partial[g * d + c] = sum_{i in block g} A[i, c] * u[i]   (grid: nblk x ntc)
__global__ void __launch_bounds__(256) gemv_t_kernel(int64_t n, int64_t d, const double* __restrict__ A, int64_t lda,
                                                     const double* __restrict__ u, double* __restrict__ partial,
                                                     int64_t rows_per_blk, int64_t ntc) {
  const int64_t g = blockIdx.x / ntc, tc = blockIdx.x % ntc;
  const int64_t c = tc * kTCols + 2 * threadIdx.x;
  const int64_t r0 = g * rows_per_blk, r1 = min(n, r0 + rows_per_blk);
  const bool vec = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 2 == 0);
  double acc0 = 0.0, acc1 = 0.0;
  if (c < d) {
    const bool two = c + 1 < d;
    for (int64_t i0 = r0; i0 < r1; i0 += kTRows) {
      double x0[kTRows], x1[kTRows], uu[kTRows];
#pragma unroll
      for (int k = 0; k < kTRows; ++k) {
        const int64_t i = i0 + k;
        x0[k] = 0.0;
        x1[k] = 0.0;
        uu[k] = 0.0;
        if (i < r1) {
          const double* a = A + i * lda + c;
          uu[k] = __ldg(u + i);
          if (vec && two) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(a));
            x0[k] = v.x;
            x1[k] = v.y;
          } else {
            x0[k] = __ldg(a);
            if (two) x1[k] = __ldg(a + 1);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kTRows; ++k) {
        acc0 = fma(x0[k], uu[k], acc0);
        acc1 = fma(x1[k], uu[k], acc1);
      }
    }
    partial[g * d + c] = acc0;
    if (two) partial[g * d + c + 1] = acc1;
  }
}

// out[c] = alpha * (sum_g partial[g][c]) + beta * yin[c]   (g ascending)
__global__ void colsum_kernel(int64_t nblk, int64_t d, const double* __restrict__ partial, double alpha, double beta,
                              const double* yin, double* out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  double s = 0.0;
  for (int64_t g = 0; g < nblk; ++g) s += partial[g * d + c];
  out[c] = yin ? fma(beta, yin[c], alpha * s) : alpha * s;
}

// ---- column-major A (n x d, A[c * lda + i]): the same two products
// out[i] = sum_c A[i, c] t[c] + beta yin[i]: one thread per row, columns in
// order (8 loads in flight), a warp reads 256 contiguous bytes of a column;
// sq[blockIdx] = sum over the CTA's rows of out^2 (fixed order)
template <bool SMEM>
__global__ void __launch_bounds__(256) cm_av_kernel(int64_t n, int64_t d, const double* __restrict__ A, int64_t lda,
                                                    const double* __restrict__ t, double beta, const double* yin,
                                                    double* out, double* __restrict__ sq, const double* bdev) {
  extern __shared__ double ts[];
  if (bdev) beta = *bdev;
  if (SMEM) {
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) ts[c] = t[c];
    __syncthreads();
  }
  const double* tv = SMEM ? ts : t;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (i < n) {
    const double* a = A + i;
    int64_t c = 0;
    for (; c + 8 <= d; c += 8) {
      double x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = __ldg(a + (c + k) * lda);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = fma(x[k], tv[c + k], acc);
    }
    for (; c < d; ++c) acc = fma(__ldg(a + c * lda), tv[c], acc);
    if (yin) acc = fma(beta, yin[i], acc);
    out[i] = acc;
  }
  __shared__ double part[256];
  part[threadIdx.x] = acc * acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) sq[blockIdx.x] = part[0];
}

// The same product, two adjacent rows per thread (16-byte loads: a warp reads
// 512 contiguous bytes of each column, twice the DRAM burst of cm_av_kernel).
// Requires A 16-byte aligned and lda even.  Same per-row order of additions.
template <bool SMEM>
__global__ void __launch_bounds__(256) cm_av2_kernel(int64_t n, int64_t d, const double* __restrict__ A, int64_t lda,
                                                     const double* __restrict__ t, double beta, const double* yin,
                                                     double* out, double* __restrict__ sq, const double* bdev) {
  extern __shared__ double ts[];
  if (bdev) beta = *bdev;
  if (SMEM) {
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) ts[c] = t[c];
    __syncthreads();
  }
  const double* tv = SMEM ? ts : t;
  const int64_t i = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  double acc0 = 0.0, acc1 = 0.0;
  if (i + 1 < n) {
    const double2* a = reinterpret_cast<const double2*>(A + i);
    const int64_t ld2 = lda / 2;
    int64_t c = 0;
    for (; c + 8 <= d; c += 8) {
      double2 x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = __ldg(a + (c + k) * ld2);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc0 = fma(x[k].x, tv[c + k], acc0);
        acc1 = fma(x[k].y, tv[c + k], acc1);
      }
    }
    for (; c < d; ++c) {
      const double2 x = __ldg(a + c * ld2);
      acc0 = fma(x.x, tv[c], acc0);
      acc1 = fma(x.y, tv[c], acc1);
    }
    if (yin) {
      acc0 = fma(beta, yin[i], acc0);
      acc1 = fma(beta, yin[i + 1], acc1);
    }
    out[i] = acc0;
    out[i + 1] = acc1;
  } else if (i < n) {  // odd n: the last row alone
    const double* a = A + i;
    for (int64_t c = 0; c < d; ++c) acc0 = fma(__ldg(a + c * lda), tv[c], acc0);
    if (yin) acc0 = fma(beta, yin[i], acc0);
    out[i] = acc0;
  }
  __shared__ double part[256];
  part[threadIdx.x] = acc0 * acc0 + acc1 * acc1;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) sq[blockIdx.x] = part[0];
}

// partial[g * d + c] = sum over rows i of block g (kCmRows rows) of A[i, c] u[i]:
// the block's u staged in shared memory, one warp per column (lanes stride the
// contiguous rows, warp-tree reduction)
constexpr int kCmRows = 4096;
__global__ void __launch_bounds__(256) cm_atu_kernel(int64_t n, int64_t d, const double* __restrict__ A, int64_t lda,
                                                     const double* __restrict__ u, double* __restrict__ partial,
                                                     int64_t ncg) {
  __shared__ double us[kCmRows];
  const int64_t g = blockIdx.x / ncg, cg = blockIdx.x % ncg;
  const int64_t r0 = g * kCmRows;
  const int nr = (int)min((int64_t)kCmRows, n - r0);
  for (int i = threadIdx.x; i < nr; i += blockDim.x) us[i] = u[r0 + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t cpg = (d + ncg - 1) / ncg;  // columns of this group
  const int64_t cbeg = cg * cpg, cend = min(d, cbeg + cpg);
  for (int64_t c = cbeg + wp; c < cend; c += 8) {
    const double* a = A + c * lda + r0;
    double acc0 = 0.0, acc1 = 0.0;
    int i = lane;
    for (; i + 32 < nr; i += 64) {
      acc0 = fma(__ldg(a + i), us[i], acc0);
      acc1 = fma(__ldg(a + i + 32), us[i + 32], acc1);
    }
    for (; i < nr; i += 32) acc0 = fma(__ldg(a + i), us[i], acc0);
    double acc = acc0 + acc1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) partial[g * d + c] = acc;
  }
}

// sq[blockIdx] = sum of x[i]^2 over a 4096-element chunk, fixed tree order
__global__ void sqsum_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ sq) {
  __shared__ double sh[256];
  const int64_t base = (int64_t)blockIdx.x * 4096;
  double s = 0.0;
  for (int k = 0; k < 16; ++k) {
    const int64_t i = base + threadIdx.x + 256 * k;
    if (i < n) s = fma(x[i], x[i], s);
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) sq[blockIdx.x] = sh[0];
}

// *out = sum of parts[0..np) (one thread, ascending) -- the final deterministic reduction
__global__ void sum_parts_kernel(int64_t np, const double* __restrict__ parts, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int64_t i = 0; i < np; ++i) s += parts[i];
    *out = s;
  }
}

__global__ void scale_vec_kernel(int64_t n, double* x, double a, const double* adev = nullptr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (adev) a = *adev;
  if (i < n) x[i] *= a;
}

// y += p * w;  w = v + q * w
__global__ void lsqr_update_kernel(int64_t d, double* y, double* w, const double* v, double p, double q,
                                   const double* pq = nullptr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pq) {
    p = pq[0];
    q = pq[1];
  }
  if (i < d) {
    const double wi = w[i];
    y[i] = fma(p, wi, y[i]);
    w[i] = fma(q, wi, v[i]);
  }
}

// out = a * x + b * y
__global__ void axpby_kernel(int64_t n, double a, const double* x, double b, const double* y, double* out,
                             const double* bdev = nullptr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (bdev) b = *bdev;
  if (i < n) out[i] = y ? fma(b, y[i], a * x[i]) : a * x[i];
}

// ---- device-resident LSQR scalars (slots of LlsWs::scal)
enum : int {
  kSqBeta = 0, kSqAlpha = 1, kAlpha = 2, kBeta = 3, kRhobar = 4, kPhibar = 5, kAnorm2 = 6, kTest2 = 7,
  kIters = 8, kP = 9, kQ = 10, kInvBeta = 11, kInvAlpha = 12, kNegAlpha = 13, kNegBeta = 14, kTau = 15,
  kItMax = 16, kNumScal = 24
};

// The scalar recurrence in the host loop's exact IEEE operations: explicit
// round-to-nearest intrinsics, so nvcc cannot contract a*b + c into an FMA
// (the host code has none), and the graph and the host loop stay bit-identical.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

// beta = ||u||; u /= beta (when > 0); anorm2 += alpha^2 + beta^2 -- the host loop's order
__global__ void lsqr_beta_kernel(double* sc) {
  const double beta = sqrt(sc[kSqBeta]);
  const double alpha = sc[kAlpha];
  sc[kBeta] = beta;
  sc[kInvBeta] = beta > 0.0 ? 1.0 / beta : 1.0;
  sc[kNegBeta] = -beta;
  sc[kAnorm2] = add(add(sc[kAnorm2], mul(alpha, alpha)), mul(beta, beta));
}

// alpha = ||v||; the plane rotation; the (7.1) estimate; the loop condition
__global__ void lsqr_alpha_kernel(double* sc, cudaGraphConditionalHandle cond) {
  const double alpha = sqrt(sc[kSqAlpha]);
  const double beta = sc[kBeta];
  sc[kAlpha] = alpha;
  sc[kInvAlpha] = alpha > 0.0 ? 1.0 / alpha : 1.0;
  sc[kNegAlpha] = -alpha;
  const double rhobar = sc[kRhobar], phibar = sc[kPhibar];
  const double rho = sqrt(add(mul(rhobar, rhobar), mul(beta, beta)));
  const double c = rhobar / rho, s = beta / rho;
  const double theta = mul(s, alpha);
  sc[kRhobar] = mul(-c, alpha);
  const double phi = mul(c, phibar);
  const double nphibar = mul(s, phibar);
  sc[kPhibar] = nphibar;
  sc[kP] = phi / rho;
  sc[kQ] = -theta / rho;
  const double arnorm = mul(alpha, fabs(mul(s, phi)));
  const double it = sc[kIters] + 1.0;
  sc[kIters] = it;
  bool done;
  if (nphibar == 0.0) {
    sc[kTest2] = 0.0;
    done = true;
  } else {
    const double t2 = arnorm / mul(sqrt(sc[kAnorm2]), nphibar);
    sc[kTest2] = t2;
    done = t2 <= sc[kTau];
  }
  done = done || it >= sc[kItMax];
  cudaGraphSetConditional(cond, done ? 0u : 1u);
}

// row-major m x d (ld ldsa) -> column-major m x d (ld m)
__global__ void to_colmajor_kernel(int64_t m, int64_t d, const double* __restrict__ S, int64_t ld,
                                   double* __restrict__ F) {
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < m && c < d) ? S[r * ld + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < m && c < d) F[c * m + r] = tile[threadIdx.x][k];
  }
}

inline unsigned nblocks(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// ---------------------------------------------------------------- library handles (per thread, per device)
struct Handles {
  cusolverDnHandle_t sol = nullptr;
  cublasHandle_t blas = nullptr;
  int dev = -1;
};
thread_local Handles g_h;

int handles(cudaStream_t st, Handles** out) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_h.dev != dev) {
    if (g_h.sol) cusolverDnDestroy(g_h.sol);
    if (g_h.blas) cublasDestroy(g_h.blas);
    g_h = Handles{};
    if (cusolverDnCreate(&g_h.sol) != CUSOLVER_STATUS_SUCCESS || cublasCreate(&g_h.blas) != CUBLAS_STATUS_SUCCESS) {
      set_error("lls: cannot create cuSOLVER/cuBLAS handles");
      return SKH_ECUDA;
    }
    cublasSetPointerMode(g_h.blas, CUBLAS_POINTER_MODE_HOST);
    g_h.dev = dev;
  }
  cusolverDnSetStream(g_h.sol, st);
  cublasSetStream(g_h.blas, st);
  *out = &g_h;
  return SKH_OK;
}

struct LlsWs {
  double* F;       // SA column-major, factored in place [m x d]
  double* tau;     // Householder scalars [d]
  double* qtb;     // Q^T Sb [m]
  double* u;       // [n]
  double* v;       // [d]
  double* w;       // [d]
  double* y;       // [d]
  double* t;       // [d]
  double* xs;      // [d]
  double* part;    // gemv_t partials [nblk x d]
  double* sq;      // norm partials [max(nrb, nsq)]
  double* scal;    // [kNumScal] device scalars
  int* devinfo;
  double* lwork;   // cuSOLVER workspace
  int lwork_n;
  double* Ri;      // SKH_LLS_RINV=1: M = R^{-1} column-major [d x d] (= M^T row-major)
  double* Rr;      // M row-major
  double* tmp;     // [d]
  // rank-revealing mode (R-CPQR): the d x d factor being pivoted, R11, X = R11^{-1}
  double* Rp;      // [d x d] column-major
  double* Rc;      // [d x d] R11 gathered (column-major, ld d)
  int* perm;       // [d] position -> physical column
  int* pos_of;     // [d] physical column -> position (-1 while unpivoted)
  double* tau1;    // [d] reflector scalars of the pivoted QR
  double* nrm;     // [d] partial column norms^2
  double* nrm0;    // [d] norms^2 at the last recompute
  double* red_val; // [grid] argmax partials
  int* red_idx;    // [grid]
  double* diag;    // [d] |r~_qq|
  int64_t nblk, nrb;
  size_t total;
};

int64_t gemv_t_blocks(int64_t n, int64_t d) {
  const int64_t ntc = (d + kTCols - 1) / kTCols;
  const int64_t want = std::max<int64_t>(1, (148 * 8) / ntc);
  return std::min<int64_t>(want, std::max<int64_t>(1, (n + 255) / 256));
}

// SKH_LLS_RINV=1 (opt-in): form R^{-1} once (cuBLAS dtrsm against I) and apply it
// with dense GEMVs instead of two back-solves per LSQR iteration.  LSQR then
// runs on A M with M = fl(R^{-1}) and returns x = M y: the same minimiser
// whatever M's rounding (M is invertible), a different rounding path from the
// paper's back-solve (L1081), which stays the default.
bool rinv_mode() {
  static const bool v = [] {
    const char* e = getenv("SKH_LLS_RINV");
    return e && e[0] == '1';
  }();
  return v;
}

LlsWs lls_layout(void* base, int64_t n, int64_t d, int64_t m, int lwork_n, bool rr = false) {
  LlsWs w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align_up(bytes);
    return q;
  };
  w.nblk = gemv_t_blocks(n, d);
  const int64_t nblk_cm = (n + kCmRows - 1) / kCmRows;  // column-major A^T u row blocks
  w.nrb = (n + 255) / 256;  // gemv_n CTAs (rows_per_cta = 256)
  const int64_t nsq = std::max<int64_t>(std::max<int64_t>(w.nrb, (n + 4095) / 4096 + 1), d / 8 + 1) + 1;
  w.F = (double*)take(sizeof(double) * (size_t)m * d);
  w.tau = (double*)take(sizeof(double) * (size_t)d);
  w.qtb = (double*)take(sizeof(double) * (size_t)m);
  w.u = (double*)take(sizeof(double) * (size_t)n);
  w.v = (double*)take(sizeof(double) * (size_t)d);
  w.w = (double*)take(sizeof(double) * (size_t)d);
  w.y = (double*)take(sizeof(double) * (size_t)d);
  w.t = (double*)take(sizeof(double) * (size_t)d);
  w.xs = (double*)take(sizeof(double) * (size_t)d);
  w.part = (double*)take(sizeof(double) * (size_t)std::max(w.nblk, nblk_cm) * d);
  w.sq = (double*)take(sizeof(double) * (size_t)nsq);
  w.scal = (double*)take(sizeof(double) * kNumScal);
  w.devinfo = (int*)take(sizeof(int) * 4);
  w.lwork = (double*)take(sizeof(double) * (size_t)std::max(lwork_n, 1));
  w.lwork_n = lwork_n;
  if (rinv_mode() || rr) {
    w.Ri = (double*)take(sizeof(double) * (size_t)d * d);
    w.Rr = (double*)take(sizeof(double) * (size_t)d * d);
    w.tmp = (double*)take(sizeof(double) * (size_t)d);
  }
  if (rr) {
    w.Rp = (double*)take(sizeof(double) * (size_t)d * d);
    w.Rc = (double*)take(sizeof(double) * (size_t)d * d);
    w.perm = (int*)take(sizeof(int) * (size_t)d);
    w.pos_of = (int*)take(sizeof(int) * (size_t)d);
    w.tau1 = (double*)take(sizeof(double) * (size_t)d);
    w.nrm = (double*)take(sizeof(double) * (size_t)d);
    w.nrm0 = (double*)take(sizeof(double) * (size_t)d);
    w.red_val = (double*)take(sizeof(double) * 1024);
    w.red_idx = (int*)take(sizeof(int) * 1024);
    w.diag = (double*)take(sizeof(double) * (size_t)d);
  }
  w.total = off;
  return w;
}

int query_lwork(int64_t m, int64_t d, int* lw) {
  Handles* h = nullptr;
  int rc = handles(nullptr, &h);
  if (rc) return rc;
  int a = 0, b = 0;
  if (cusolverDnDgeqrf_bufferSize(h->sol, (int)m, (int)d, nullptr, (int)m, &a) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDormqr_bufferSize(h->sol, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, (int)m, 1, (int)d, nullptr, (int)m, nullptr,
                                  nullptr, (int)m, &b) != CUSOLVER_STATUS_SUCCESS) {
    set_error("lls: cuSOLVER workspace query failed");
    return SKH_ECUDA;
  }
  *lw = std::max(a, b);
  return SKH_OK;
}

// out = A t + beta yin (row-major A); returns ||out||^2 through w.scal[slot] (device)
int gemv_n(int64_t n, int64_t d, const double* A, int64_t lda, const double* t, double beta, const double* yin,
           double* out, const LlsWs& w, int slot, cudaStream_t st, const double* bdev = nullptr,
           int64_t rows = 256) {
  const int64_t grid = (n + rows - 1) / rows;
  if (d <= kMaxSmemX) {
    const size_t smem = sizeof(double) * (size_t)d;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(gemv_n_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    gemv_n_kernel<true><<<(unsigned)grid, 256, smem, st>>>(n, d, A, lda, t, beta, yin, out, w.sq, rows, bdev);
  } else {
    gemv_n_kernel<false><<<(unsigned)grid, 256, 0, st>>>(n, d, A, lda, t, beta, yin, out, w.sq, rows, bdev);
  }
  note_launch();
  sum_parts_kernel<<<1, 32, 0, st>>>(grid, w.sq, w.scal + slot);
  note_launch();
  return check_launch("gemv_n");
}

// out = alpha (A^T u) + beta yin
int gemv_t(int64_t n, int64_t d, const double* A, int64_t lda, const double* u, double alpha, double beta,
           const double* yin, double* out, const LlsWs& w, cudaStream_t st) {
  const int64_t ntc = (d + kTCols - 1) / kTCols;
  const int64_t rpb = (n + w.nblk - 1) / w.nblk;
  gemv_t_kernel<<<(unsigned)(w.nblk * ntc), 256, 0, st>>>(n, d, A, lda, u, w.part, rpb, ntc);
  note_launch();
  colsum_kernel<<<nblocks(d), 256, 0, st>>>(w.nblk, d, w.part, alpha, beta, yin, out);
  note_launch();
  return check_launch("gemv_t");
}

int sqnorm(int64_t n, const double* x, const LlsWs& w, int slot, cudaStream_t st);

// out = A t + beta yin and ||out||^2 -> scal[slot], for either layout
int apply_A(bool cm, int64_t n, int64_t d, const double* A, int64_t lda, const double* t, double beta,
            const double* yin, double* out, const LlsWs& w, int slot, cudaStream_t st,
            const double* bdev = nullptr) {
  if (!cm) return gemv_n(n, d, A, lda, t, beta, yin, out, w, slot, st, bdev);
  // two rows per thread (16-byte column segments) when there are rows enough to
  // fill the GPU: C5 col 24.0 -> 22.1 ms per LSQR iteration; C2 (2^16 rows,
  // 128 CTAs) was slower, so short A keeps one row per thread
  const bool two = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (lda % 2 == 0) && n >= (1ll << 19);
  if (two) {
    const int64_t grid = (n + 511) / 512;
    const size_t smem = d <= kMaxSmemX ? sizeof(double) * (size_t)d : 0;
    if (smem) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(cm_av2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cm_av2_kernel<true><<<(unsigned)grid, 256, smem, st>>>(n, d, A, lda, t, beta, yin, out, w.sq, bdev);
    } else {
      cm_av2_kernel<false><<<(unsigned)grid, 256, 0, st>>>(n, d, A, lda, t, beta, yin, out, w.sq, bdev);
    }
    note_launch();
    sum_parts_kernel<<<1, 32, 0, st>>>(grid, w.sq, w.scal + slot);
    note_launch();
    return check_launch("cm_av2");
  }
  const int64_t grid = (n + 255) / 256;
  if (d <= kMaxSmemX) {
    const size_t smem = sizeof(double) * (size_t)d;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(cm_av_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cm_av_kernel<true><<<(unsigned)grid, 256, smem, st>>>(n, d, A, lda, t, beta, yin, out, w.sq, bdev);
  } else {
    cm_av_kernel<false><<<(unsigned)grid, 256, 0, st>>>(n, d, A, lda, t, beta, yin, out, w.sq, bdev);
  }
  note_launch();
  sum_parts_kernel<<<1, 32, 0, st>>>(grid, w.sq, w.scal + slot);
  note_launch();
  return check_launch("cm_av");
}

// out = A^T u + beta yin, for either layout
int apply_AT(bool cm, int64_t n, int64_t d, const double* A, int64_t lda, const double* u, double beta,
             const double* yin, double* out, const LlsWs& w, cudaStream_t st) {
  if (!cm) return gemv_t(n, d, A, lda, u, 1.0, beta, yin, out, w, st);
  const int64_t nblk = (n + kCmRows - 1) / kCmRows;
  const int64_t ncg = std::max<int64_t>(1, std::min<int64_t>((d + 7) / 8, (148 * 8 + nblk - 1) / nblk));
  cm_atu_kernel<<<(unsigned)(nblk * ncg), 256, 0, st>>>(n, d, A, lda, u, w.part, ncg);
  note_launch();
  colsum_kernel<<<nblocks(d), 256, 0, st>>>(nblk, d, w.part, 1.0, beta, yin, out);
  note_launch();
  return check_launch("cm_atu");
}

int sqnorm(int64_t n, const double* x, const LlsWs& w, int slot, cudaStream_t st) {
  const int64_t nb = (n + 4095) / 4096;
  sqsum_kernel<<<(unsigned)nb, 256, 0, st>>>(n, x, w.sq);
  note_launch();
  sum_parts_kernel<<<1, 32, 0, st>>>(nb, w.sq, w.scal + slot);
  note_launch();
  return check_launch("sqnorm");
}

int read_scal(const LlsWs& w, int slot, double* out, cudaStream_t st) {
  if (cudaMemcpyAsync(out, w.scal + slot, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return check_launch("lls scalar read-back");
  return SKH_OK;
}

__global__ void identity_kernel(int64_t d, double* __restrict__ X) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < d * d) X[e] = (e / d == e % d) ? 1.0 : 0.0;
}

// M = R^{-1}: cuBLAS dtrsm of R X = I, then the row-major copy Rr
// ------------------------------------------------------------------ Step 2, rank-revealing mode
namespace cg = cooperative_groups;

// Column-pivoted Householder QR (Businger-Golub, LAPACK dgeqp3's rule: pivot
// = the largest remaining partial column norm, ties to the lower column;
// norms downdated with dlaqp2's cancellation safeguard) of the d x d matrix
// Rp (column-major, ld d), in place: R~ in the upper triangle of the pivoted
// positions (entry (i, q) of R~ is Rp[i + perm[q] d] for i <= q), reflector q
// below the diagonal of physical column perm[q] (unit leading entry implied),
// tau1[q].  One cooperative grid: CTA bid owns physical columns bid, bid + G,
// ...; per pivot two grid syncs (argmax partials; the new reflector), and each
// warp applies the reflector to one owned column at a time.
__global__ void __launch_bounds__(256) cpqr_kernel(int d, double* __restrict__ Rp, int* __restrict__ perm,
                                                   int* __restrict__ pos_of, double* __restrict__ tau1,
                                                   double* __restrict__ nrm, double* __restrict__ nrm0,
                                                   double* __restrict__ red_val, int* __restrict__ red_idx) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double vsh[];  // [d] the current reflector
  __shared__ double wv[8];
  __shared__ int wi[8];
  __shared__ double hs[2];
  const int G = gridDim.x, bid = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const double tol3z = 1.4901161193847656e-08;  // sqrt(DBL_EPSILON), dlaqp2
  auto col = [&](int c) { return Rp + (int64_t)c * d; };
  // initial norms of the owned columns (one warp per column)
  for (int c = bid + G * wp; c < d; c += 8 * G) {
    const double* a = col(c);
    double s = 0.0;
    for (int i = lane; i < d; i += 32) s += a[i] * a[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      nrm[c] = s;
      nrm0[c] = s;
      pos_of[c] = -1;
    }
  }
  grid.sync();
  for (int k = 0; k < d; ++k) {
    // (a) argmax of the remaining partial norms over the owned columns
    double best = -1.0;
    int bc = 0x7fffffff;
    for (int c = bid + G * tid; c < d; c += G * 256) {
      if (pos_of[c] >= 0) continue;
      const double v = nrm[c];
      if (v > best || (v == best && c < bc)) {
        best = v;
        bc = c;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ov > best || (ov == best && oc < bc)) {
        best = ov;
        bc = oc;
      }
    }
    if (lane == 0) {
      wv[wp] = best;
      wi[wp] = bc;
    }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < 8; ++q)
        if (wv[q] > best || (wv[q] == best && wi[q] < bc)) {
          best = wv[q];
          bc = wi[q];
        }
      red_val[bid] = best;
      red_idx[bid] = bc;
    }
    grid.sync();
    // (b) the global pivot (every CTA computes the same), its reflector by the owner
    best = -1.0;
    bc = 0x7fffffff;
    for (int q = tid; q < G; q += 256) {
      const double v = red_val[q];
      const int c = red_idx[q];
      if (v > best || (v == best && c < bc)) {
        best = v;
        bc = c;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ov > best || (ov == best && oc < bc)) {
        best = ov;
        bc = oc;
      }
    }
    __syncthreads();  // wv/wi reuse
    if (lane == 0) {
      wv[wp] = best;
      wi[wp] = bc;
    }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < 8; ++q)
        if (wv[q] > best || (wv[q] == best && wi[q] < bc)) {
          best = wv[q];
          bc = wi[q];
        }
      wi[0] = bc;
    }
    __syncthreads();
    const int cs = wi[0];
    if (cs % G == bid) {
      double* a = col(cs);
      double s = 0.0;  // ||x(k+1:)||^2
      for (int i = k + 1 + tid; i < d; i += 256) s += a[i] * a[i];
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      __syncthreads();
      if (lane == 0) wv[wp] = s;
      __syncthreads();
      if (tid == 0) {
        double xn2 = 0.0;
        for (int q = 0; q < 8; ++q) xn2 += wv[q];
        const double alpha = a[k];
        double tau = 0.0, beta = alpha, scal = 0.0;
        if (xn2 > 0.0) {  // dlarfg: beta = -sign(alpha) ||x||, tau = (beta - alpha) / beta, v = x / (alpha - beta)
          beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
          tau = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        hs[0] = scal;
        hs[1] = beta;
        tau1[k] = tau;
        perm[k] = cs;
        pos_of[cs] = k;
      }
      __syncthreads();
      const double scal = hs[0];
      for (int i = k + 1 + tid; i < d; i += 256) a[i] *= scal;
      if (tid == 0) a[k] = hs[1];
    }
    grid.sync();
    // (c) apply H_k = I - tau v v^T to the owned unpivoted columns, downdate their norms
    const double* v = col(cs);
    for (int i = k + 1 + tid; i < d; i += 256) vsh[i] = v[i];
    if (tid == 0) vsh[k] = 1.0;
    __syncthreads();
    const double tau = tau1[k];
    for (int c = bid + G * wp; c < d; c += 8 * G) {
      if (pos_of[c] >= 0) continue;
      double* a = col(c);
      double s = 0.0;
      for (int i = k + lane; i < d; i += 32) s += vsh[i] * a[i];
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const double tw = tau * s;
      if (tw != 0.0)
        for (int i = k + lane; i < d; i += 32) a[i] -= tw * vsh[i];
      __syncwarp();
      // dlaqp2 norm downdate
      double nv = nrm[c];
      if (nv != 0.0) {
        const double rk = a[k];
        double temp = 1.0 - rk * rk / nv;
        temp = temp < 0.0 ? 0.0 : temp;
        if (temp * (nv / nrm0[c]) <= tol3z) {
          double r2 = 0.0;
          for (int i = k + 1 + lane; i < d; i += 32) r2 += a[i] * a[i];
          for (int o = 16; o; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
          nv = r2;
          if (lane == 0) nrm0[c] = r2;
        } else {
          nv *= temp;
        }
        if (lane == 0) nrm[c] = nv;
      }
      __syncwarp();
    }
    __syncthreads();  // vsh is rewritten next step
  }
}

// |r~_qq| per position
__global__ void cpqr_diag_kernel(int d, const double* __restrict__ Rp, const int* __restrict__ perm,
                                 double* __restrict__ diag) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < d) diag[q] = fabs(Rp[q + (int64_t)perm[q] * d]);
}

// R11 (p x p, upper) gathered into Rc (column-major, ld d); Xb = I_p (ld d) in Ri
__global__ void cpqr_r11_kernel(int d, int p, const double* __restrict__ Rp, const int* __restrict__ perm,
                                double* __restrict__ Rc, double* __restrict__ X) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)p * p) return;
  const int i = (int)(t % p), j = (int)(t / p);
  Rc[i + (int64_t)j * d] = i <= j ? Rp[i + (int64_t)perm[j] * d] : 0.0;
  X[i + (int64_t)j * d] = i == j ? 1.0 : 0.0;
}

// the upper triangle of F (m x d, ld m) into Rp (d x d, ld d), zeros below
__global__ void upper_copy_kernel(int64_t d, const double* __restrict__ F, int64_t m, double* __restrict__ Rp) {
  const int64_t j = (int64_t)blockIdx.x * 32 + threadIdx.x;  // column
  for (int64_t i = (int64_t)blockIdx.y * 32 + threadIdx.y; i < (int64_t)blockIdx.y * 32 + 32; i += 8)
    if (i < d && j < d) Rp[i + j * d] = i <= j ? F[i + j * m] : 0.0;
}

// N = P [X 0; 0 0] (column-major d x d, zeroed first): N[perm[i], j] = X[i, j] for i, j < p
__global__ void cpqr_scatter_kernel(int d, int p, const double* __restrict__ X, const int* __restrict__ perm,
                                     double* __restrict__ N) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)p * p) return;
  const int i = (int)(t % p), j = (int)(t / p);
  N[perm[i] + (int64_t)j * d] = X[i + (int64_t)j * d];
}

// z <- Q1^T z = H_{d-1} ... H_0 z (z: first d entries of Q0^T Sb), one CTA
__global__ void __launch_bounds__(256) cpqr_qt_kernel(int d, const double* __restrict__ Rp,
                                                      const int* __restrict__ perm, const double* __restrict__ tau1,
                                                      double* __restrict__ z) {
  __shared__ double ws[8];
  __shared__ double tw;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  for (int k = 0; k < d; ++k) {
    const double* v = Rp + (int64_t)perm[k] * d;
    double s = 0.0;
    for (int i = k + tid; i < d; i += 256) s += (i == k ? 1.0 : v[i]) * z[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) ws[wp] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < 8; ++q) t += ws[q];
      tw = tau1[k] * t;
    }
    __syncthreads();
    const double c = tw;
    for (int i = k + tid; i < d; i += 256) z[i] -= c * (i == k ? 1.0 : v[i]);
    __syncthreads();
  }
}

// Rank-revealing Step 2 on the dgeqrf factor in w.F: returns p (host) and
// leaves N (Ri, column-major) and N^T (Rr, row-major view) for trsv's GEMV path.
int cpqr_step2(Handles* h, int64_t d, int64_t m, const LlsWs& w, double rcond, cudaStream_t st, int64_t* p_out) {
  const int di = (int)d;
  // R0: the upper triangle of F (ld m) -> Rp (ld d), zeros below
  dim3 grid((unsigned)((d + 31) / 32), (unsigned)((d + 31) / 32));
  upper_copy_kernel<<<grid, dim3(32, 8), 0, st>>>(d, w.F, m, w.Rp);
  note_launch();
  int nsm = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = sizeof(double) * (size_t)d;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(cpqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    set_error("lls cpqr: d = %lld too large for the on-chip reflector", (long long)d);
    return SKH_EINVAL;
  }
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cpqr_kernel, 256, smem);
  int G = std::min(nsm * std::max(per, 1), std::min(1024, std::max(1, di)));
  G = std::min(G, nsm);  // one CTA per SM: enough columns per CTA, cheap grid syncs
  void* args[] = {(void*)&di, (void*)&w.Rp, (void*)&w.perm, (void*)&w.pos_of, (void*)&w.tau1,
                  (void*)&w.nrm, (void*)&w.nrm0, (void*)&w.red_val, (void*)&w.red_idx};
  if (cudaLaunchCooperativeKernel((const void*)cpqr_kernel, dim3(G), dim3(256), args, smem, st) != cudaSuccess)
    return check_launch("lls: cpqr");
  note_launch();
  cpqr_diag_kernel<<<(unsigned)((d + 255) / 256), 256, 0, st>>>(di, w.Rp, w.perm, w.diag);
  note_launch();
  std::vector<double> dg((size_t)d);
  if (cudaMemcpyAsync(dg.data(), w.diag, sizeof(double) * (size_t)d, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return check_launch("lls: cpqr diagonal");
  int64_t p = 0;  // p = max{q : |r~_qq| >= rcond} (1-based q), L1109-1112
  for (int64_t q = 0; q < d; ++q)
    if (dg[q] >= rcond) p = q + 1;
  *p_out = p;
  // N = P [R11^{-1} 0; 0 0]
  const int pi = (int)p;
  cudaMemsetAsync(w.Ri, 0, sizeof(double) * (size_t)d * d, st);
  if (p > 0) {
    cpqr_r11_kernel<<<(unsigned)((p * p + 255) / 256), 256, 0, st>>>(di, pi, w.Rp, w.perm, w.Rc, w.Rr);
    note_launch();
    const double one = 1.0;
    if (cublasDtrsm(h->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, pi, pi, &one,
                    w.Rc, di, w.Rr, di) != CUBLAS_STATUS_SUCCESS) {
      set_error("lls: cublasDtrsm (R11^{-1}) failed");
      return SKH_ECUDA;
    }
    cpqr_scatter_kernel<<<(unsigned)((p * p + 255) / 256), 256, 0, st>>>(di, pi, w.Rr, w.perm, w.Ri);
    note_launch();
  }
  to_colmajor_kernel<<<grid, dim3(32, 8), 0, st>>>(d, d, w.Ri, d, w.Rr);  // Rr = row-major N
  note_launch();
  return check_launch("lls: cpqr N");
}

int form_rinv(Handles* h, int64_t d, const LlsWs& w, int64_t m, cudaStream_t st) {
  identity_kernel<<<(unsigned)((d * d + 255) / 256), 256, 0, st>>>(d, w.Ri);
  note_launch();
  const double one = 1.0;
  if (cublasDtrsm(h->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)d,
                  (int)d, &one, w.F, (int)m, w.Ri, (int)d) != CUBLAS_STATUS_SUCCESS) {
    set_error("lls: cublasDtrsm (R^{-1}) failed");
    return SKH_ECUDA;
  }
  dim3 grid((unsigned)((d + 31) / 32), (unsigned)((d + 31) / 32));
  to_colmajor_kernel<<<grid, dim3(32, 8), 0, st>>>(d, d, w.Ri, d, w.Rr);  // Rr = transpose of Ri's storage
  note_launch();
  return check_launch("lls: R^{-1}");
}

// Certified full rank (R22b).  Column pivoting makes the pivoted
// diagonals non-increasing, |r~_11| >= ... >= |r~_dd|, and for any triangular
// factor the last row of R^{-1} is e_d^T / r_dd, so |r~_dd| >= sigma_min(R0) >=
// 1 / ||R0^{-1}||_F.  ||R0^{-1}||_F rcond <= 1/2 (a factor 2 for the rounding of
// the computed inverse) therefore proves p = max{q : |r~_qq| >= rcond} = d
// without pivoting: V1 = I, R11 = R0, N = R0^{-1} -- the same
// least-squares solution as the pivoted factor (R0 = Q1 R~ P^T differs from it
// by an orthogonal factor).  Leaves N in Ri / Rr when it returns *ok = true.
// SKH_LLS_CPQR=1 skips the certificate (always pivot).
int rr_certify(Handles* h, int64_t d, int64_t m, const LlsWs& w, double rcond, cudaStream_t st, bool* ok) {
  *ok = false;
  static const bool force = [] {
    const char* e = getenv("SKH_LLS_CPQR");
    return e && atoi(e) != 0;
  }();
  if (force || d * d >= (1ll << 31)) return SKH_OK;
  int rc = form_rinv(h, d, w, m, st);
  if (rc) return rc;
  double nrm = 0.0;  // host pointer mode: the call returns when the norm is ready
  if (cublasDnrm2(h->blas, (int)(d * d), w.Ri, 1, &nrm) != CUBLAS_STATUS_SUCCESS) {
    set_error("lls: cublasDnrm2 (||R^{-1}||_F) failed");
    return SKH_ECUDA;
  }
  *ok = std::isfinite(nrm) && nrm * rcond * 2.0 <= 1.0;
  return SKH_OK;
}

int trsv(Handles* h, int64_t d, const LlsWs& w, int64_t m, bool trans, double* x) {
  if (w.Ri) {  // x = M x or M^T x, M = R^{-1}: one warp per row of a row-major matrix (rinv_mode)
    cudaStream_t st = nullptr;
    cublasGetStream(h->blas, &st);
    int rc = gemv_n(d, d, trans ? w.Ri : w.Rr, d, x, 0.0, nullptr, w.tmp, w, kNumScal - 1, st, nullptr, 8);
    if (rc) return rc;
    if (cudaMemcpyAsync(x, w.tmp, sizeof(double) * (size_t)d, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return check_launch("lls: R^{-1} copy");
    return SKH_OK;
  }
  if (cublasDtrsv(h->blas, CUBLAS_FILL_MODE_UPPER, trans ? CUBLAS_OP_T : CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)d,
                  w.F, (int)m, x, 1) != CUBLAS_STATUS_SUCCESS) {
    set_error("lls: cublasDtrsv failed");
    return SKH_ECUDA;
  }
  return SKH_OK;
}

// Step 4 as ONE graph launch: a WHILE conditional node whose body is one LSQR
// iteration (the two HBM passes over A, the two triangular solves, the vector
// updates and the scalar recurrence, all on the device); lsqr_alpha_kernel
// clears the condition when (7.1) holds or it_max is reached.  No host round
// trips inside the loop; the arithmetic is the host loop's, operation for
// operation (IEEE sqrt and division on the device), so both give the same bits.
// Returns SKH_OK with *ex instantiated, or an error (the caller then runs the
// host loop; nothing has been enqueued on st).
int lsqr_graph_build(Handles* h, bool cm, int64_t n, int64_t d, int64_t m, const double* A, int64_t lda,
                     const LlsWs& w, cudaStream_t st, cudaGraphExec_t* ex) {
  double* sc = w.scal;
  cudaStream_t cs = nullptr;
  cudaGraph_t g = nullptr;
  *ex = nullptr;
  auto fail = [&]() {
    if (g) cudaGraphDestroy(g);
    if (cs) cudaStreamDestroy(cs);
    cublasSetStream(h->blas, st);
    cudaGetLastError();
    return SKH_ECUDA;
  };
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess || cudaGraphCreate(&g, 0) != cudaSuccess)
    return fail();
  cudaGraphConditionalHandle cond;
  if (cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) return fail();
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = cond;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &np) != cudaSuccess) return fail();
  cudaGraph_t body = np.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return fail();
  cublasSetStream(h->blas, cs);
  int erc = SKH_OK;
  {  // one iteration, exactly the host loop's operations
    axpby_kernel<<<nblocks(d), 256, 0, cs>>>(d, 1.0, w.v, 0.0, nullptr, w.t);  // t = v
    if (!erc) erc = trsv(h, d, w, m, false, w.t);
    if (!erc) erc = apply_A(cm, n, d, A, lda, w.t, 0.0, w.u, w.u, w, kSqBeta, cs, sc + kNegAlpha);
    lsqr_beta_kernel<<<1, 1, 0, cs>>>(sc);
    scale_vec_kernel<<<nblocks(n), 256, 0, cs>>>(n, w.u, 1.0, sc + kInvBeta);
    if (!erc) erc = apply_AT(cm, n, d, A, lda, w.u, 0.0, nullptr, w.t, w, cs);
    if (!erc) erc = trsv(h, d, w, m, true, w.t);
    axpby_kernel<<<nblocks(d), 256, 0, cs>>>(d, 1.0, w.t, 0.0, w.v, w.v, sc + kNegBeta);
    if (!erc) erc = sqnorm(d, w.v, w, kSqAlpha, cs);
    lsqr_alpha_kernel<<<1, 1, 0, cs>>>(sc, cond);
    scale_vec_kernel<<<nblocks(d), 256, 0, cs>>>(d, w.v, 1.0, sc + kInvAlpha);
    lsqr_update_kernel<<<nblocks(d), 256, 0, cs>>>(d, w.y, w.w, w.v, 0.0, 0.0, sc + kP);
  }
  cudaGraph_t captured = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(cs, &captured);
  cublasSetStream(h->blas, st);
  if (erc || ce != cudaSuccess || cudaGraphInstantiate(ex, g, 0) != cudaSuccess) {
    *ex = nullptr;
    return fail();
  }
  cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  return SKH_OK;
}

int lsqr_graph_run(cudaGraphExec_t ex, const LlsWs& w, double alpha, double beta, double tau_r, int64_t it_max,
                   cudaStream_t st, int64_t* it_out, double* test2_out, double* phibar_out) {
  double init[kNumScal] = {};
  init[kAlpha] = alpha;
  init[kBeta] = beta;
  init[kRhobar] = alpha;
  init[kPhibar] = beta;
  init[kAnorm2] = 0.0;
  init[kTest2] = INFINITY;
  init[kIters] = 0.0;
  init[kNegAlpha] = -alpha;
  init[kTau] = tau_r;
  init[kItMax] = (double)it_max;
  double* sc = w.scal;
  if (cudaMemcpyAsync(sc, init, sizeof(init), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return check_launch("lsqr graph: init");
  if (cudaGraphLaunch(ex, st) != cudaSuccess) return check_launch("lsqr graph launch");
  // kernels of the body, counted once per iteration after the fact
  double out[kNumScal];
  if (cudaMemcpyAsync(out, sc, sizeof(out), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return check_launch("lsqr graph: read-back");
  *it_out = (int64_t)out[kIters];
  *test2_out = out[kTest2];
  *phibar_out = out[kPhibar];
  for (int64_t i = 0; i < *it_out * 13; ++i) note_launch();
  return SKH_OK;
}

}  // namespace
}  // namespace skh

using namespace skh;

extern "C" {

size_t skh_lls_workspace_bytes(int64_t n, int64_t d, int64_t m) {
  if (n < 1 || d < 1 || m < d || m >= (1ll << 31)) return 0;
  int lw = 0;
  if (query_lwork(m, d, &lw)) return 0;
  return lls_layout(nullptr, n, d, m, lw).total;
}

size_t skh_lls_rr_workspace_bytes(int64_t n, int64_t d, int64_t m) {
  if (n < 1 || d < 1 || m < d || m >= (1ll << 31) || d >= (1ll << 31)) return 0;
  int lw = 0;
  if (query_lwork(m, d, &lw)) return 0;
  return lls_layout(nullptr, n, d, m, lw, true).total;
}

static int lls_solve_impl(bool cm, int64_t n, int64_t d, const double* A, int64_t lda, const double* b, int64_t m,
                          const double* SA, int64_t ldsa, const double* Sb, double tau_a, double tau_r,
                          int64_t it_max, double* x, double* x_s, int64_t* info, double* stats, void* ws,
                          size_t ws_bytes, void* stream, bool rr = false, double rcond = 0.0) {
  if (n < 1 || d < 1 || m < d || !A || !b || !SA || !Sb || !x || !info || !stats || it_max < 0 || tau_r < 0 ||
      m >= (1ll << 31)) {
    set_error("lls_solve: need n, d >= 1, m >= d, A, b, SA, Sb, x, info, stats, it_max >= 0");
    return SKH_EINVAL;
  }
  if ((!cm && (lda < d || ldsa < d)) || (cm && (lda < n || ldsa < m))) {
    set_error(cm ? "lls_solve_colmajor: lda < n or ldsa < m" : "lls_solve: lda/ldsa < d");
    return SKH_EDIM;
  }
  if (rr && !(rcond >= 0.0)) {
    set_error("lls_solve_rr: rcond must be >= 0");
    return SKH_EINVAL;
  }
  int lw = 0;
  int rc = query_lwork(m, d, &lw);
  if (rc) return rc;
  const LlsWs w = lls_layout(ws, n, d, m, lw, rr);
  if (!ws || ws_bytes < w.total) {
    set_error("lls_solve workspace too small: need %zu bytes", w.total);
    return SKH_EWORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  Handles* h = nullptr;
  rc = handles(st, &h);
  if (rc) return rc;
  skh_trace_start(st);
  // ---- Step 2: SA = Q R
  {
    if (cm) {
      if (cudaMemcpy2DAsync(w.F, sizeof(double) * (size_t)m, SA, sizeof(double) * (size_t)ldsa,
                            sizeof(double) * (size_t)m, d, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return check_launch("lls: copy SA");
    } else {
      dim3 grid((unsigned)((d + 31) / 32), (unsigned)((m + 31) / 32));
      to_colmajor_kernel<<<grid, dim3(32, 8), 0, st>>>(m, d, SA, ldsa, w.F);
      note_launch();
    }
    if (cusolverDnDgeqrf(h->sol, (int)m, (int)d, w.F, (int)m, w.tau, w.lwork, w.lwork_n, w.devinfo) !=
        CUSOLVER_STATUS_SUCCESS) {
      set_error("lls: cusolverDnDgeqrf failed");
      return SKH_ECUDA;
    }
  }
  int64_t p = d;
  bool pivoted = false;
  if (rr) {
    // rank-revealing mode: p = d certified from ||R0^{-1}||_F (N = R0^{-1}), else
    // the pivoted QR of R0, p from rcond, N = P [R11^{-1} 0; 0 0]
    bool cert = false;
    if ((rc = rr_certify(h, d, m, w, rcond, st, &cert))) return rc;
    if (!cert) {
      if ((rc = cpqr_step2(h, d, m, w, rcond, st, &p))) return rc;
      pivoted = true;
    }
    info[2] = p;
  } else {
    // full-rank QR mode (R19): reject a rank-deficient SA -- a diagonal entry
    // |r_qq| < 1e-12 max|r_jj| (relative: the unpivoted QR is not rank
    // revealing, the rank-revealing mode is skh_lls_solve_rr)
    std::vector<double> diag((size_t)d);
    if (cudaMemcpy2DAsync(diag.data(), sizeof(double), w.F, sizeof(double) * (size_t)(m + 1), sizeof(double), d,
                          cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return check_launch("lls: R diagonal");
    double rmax = 0.0;
    for (int64_t q = 0; q < d; ++q) rmax = std::max(rmax, fabs(diag[q]));
    for (int64_t q = 0; q < d; ++q) {
      if (!(fabs(diag[q]) > 1e-12 * rmax)) {
        set_error("lls: SA is numerically rank deficient (|r_%lld,%lld| = %g <= 1e-12 max|r_jj|); the full-rank QR "
                  "mode needs rank d -- use skh_lls_solve_rr", (long long)q, (long long)q, diag[q]);
        return SKH_EINVAL;
      }
    }
    if (w.Ri && (rc = form_rinv(h, d, w, m, st))) return rc;
  }
  skh_trace_mark(st, "qr");
  // ---- Step 3: x_s = R^{-1} Q^T Sb
  cudaMemcpyAsync(w.qtb, Sb, sizeof(double) * (size_t)m, cudaMemcpyDeviceToDevice, st);
  if (cusolverDnDormqr(h->sol, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, (int)m, 1, (int)d, w.F, (int)m, w.tau, w.qtb, (int)m,
                       w.lwork, w.lwork_n, w.devinfo) != CUSOLVER_STATUS_SUCCESS) {
    set_error("lls: cusolverDnDormqr failed");
    return SKH_ECUDA;
  }
  if (pivoted) {  // Q^T Sb = Q1^T (Q0^T Sb): the pivoted QR's reflectors on the first d entries
    cpqr_qt_kernel<<<1, 256, 0, st>>>((int)d, w.Rp, w.perm, w.tau1, w.qtb);
    note_launch();
  }
  cudaMemcpyAsync(w.xs, w.qtb, sizeof(double) * (size_t)d, cudaMemcpyDeviceToDevice, st);
  if ((rc = trsv(h, d, w, m, false, w.xs))) return rc;  // R^{-1} z, or N z = V1 R11^{-1} z_1..p
  if (x_s) cudaMemcpyAsync(x_s, w.xs, sizeof(double) * (size_t)d, cudaMemcpyDeviceToDevice, st);
  if ((rc = apply_A(cm, n, d, A, lda, w.xs, -1.0, b, w.u, w, 0, st))) return rc;  // u = A x_s - b
  double res2 = 0.0;
  if ((rc = read_scal(w, 0, &res2, st))) return rc;
  const double res_s = sqrt(res2);
  stats[2] = res_s;
  skh_trace_mark(st, "step3");
  if (res_s <= tau_a) {
    cudaMemcpyAsync(x, w.xs, sizeof(double) * (size_t)d, cudaMemcpyDeviceToDevice, st);
    info[0] = 3;
    info[1] = 0;
    stats[0] = 0.0;
    stats[1] = res_s;
    return cudaStreamSynchronize(st) == cudaSuccess ? SKH_OK : check_launch("lls");
  }
  // ---- Step 4: LSQR on W = A R^{-1}, y0 = 0
  double beta = 0.0, alpha = 0.0;
  if ((rc = sqnorm(n, b, w, 1, st)) || (rc = read_scal(w, 1, &beta, st))) return rc;
  beta = sqrt(beta);
  cudaMemsetAsync(w.y, 0, sizeof(double) * (size_t)d, st);
  int64_t it = 0;
  double test2 = INFINITY, phibar = beta;
  if (beta > 0.0) {
    axpby_kernel<<<nblocks(n), 256, 0, st>>>(n, 1.0 / beta, b, 0.0, nullptr, w.u);  // u = b / beta
    note_launch();
    // v = R^{-T} A^T u
    if ((rc = apply_AT(cm, n, d, A, lda, w.u, 0.0, nullptr, w.v, w, st))) return rc;
    if ((rc = trsv(h, d, w, m, true, w.v))) return rc;
    if ((rc = sqnorm(d, w.v, w, 1, st)) || (rc = read_scal(w, 1, &alpha, st))) return rc;
    alpha = sqrt(alpha);
  }
  const char* hl = getenv("SKH_LLS_HOSTLOOP");  // 1: the host-driven loop (reference for the graph's bits)
  const bool host_loop = hl && atoi(hl) != 0;
  bool graph_done = false;
  if (beta > 0.0 && alpha > 0.0 && it_max > 0 && !host_loop) {
    cudaGraphExec_t ex = nullptr;
    if (lsqr_graph_build(h, cm, n, d, m, A, lda, w, st, &ex) == SKH_OK) {
      scale_vec_kernel<<<nblocks(d), 256, 0, st>>>(d, w.v, 1.0 / alpha);
      note_launch();
      cudaMemcpyAsync(w.w, w.v, sizeof(double) * (size_t)d, cudaMemcpyDeviceToDevice, st);
      rc = lsqr_graph_run(ex, w, alpha, beta, tau_r, it_max, st, &it, &test2, &phibar);
      cudaGraphExecDestroy(ex);
      if (rc) return rc;
      graph_done = true;
    }
  }
  if (graph_done) {
    // LSQR ran entirely on the device (CUDA graph WHILE node)
  } else if (beta > 0.0 && alpha > 0.0) {
    scale_vec_kernel<<<nblocks(d), 256, 0, st>>>(d, w.v, 1.0 / alpha);
    note_launch();
    cudaMemcpyAsync(w.w, w.v, sizeof(double) * (size_t)d, cudaMemcpyDeviceToDevice, st);
    double rhobar = alpha, anorm2 = 0.0;
    while (it < it_max) {
      ++it;
      // beta u = A (R^{-1} v) - alpha u
      cudaMemcpyAsync(w.t, w.v, sizeof(double) * (size_t)d, cudaMemcpyDeviceToDevice, st);
      if ((rc = trsv(h, d, w, m, false, w.t))) return rc;
      if ((rc = apply_A(cm, n, d, A, lda, w.t, -alpha, w.u, w.u, w, 0, st))) return rc;
      if ((rc = read_scal(w, 0, &beta, st))) return rc;
      beta = sqrt(beta);
      if (beta > 0.0) {
        scale_vec_kernel<<<nblocks(n), 256, 0, st>>>(n, w.u, 1.0 / beta);
        note_launch();
      }
      anorm2 = anorm2 + alpha * alpha + beta * beta;
      // alpha v = R^{-T} (A^T u) - beta v
      if ((rc = apply_AT(cm, n, d, A, lda, w.u, 0.0, nullptr, w.t, w, st))) return rc;
      if ((rc = trsv(h, d, w, m, true, w.t))) return rc;
      axpby_kernel<<<nblocks(d), 256, 0, st>>>(d, 1.0, w.t, -beta, w.v, w.v);
      note_launch();
      if ((rc = sqnorm(d, w.v, w, 1, st)) || (rc = read_scal(w, 1, &alpha, st))) return rc;
      alpha = sqrt(alpha);
      if (alpha > 0.0) {
        scale_vec_kernel<<<nblocks(d), 256, 0, st>>>(d, w.v, 1.0 / alpha);
        note_launch();
      }
      const double rho = sqrt(rhobar * rhobar + beta * beta);
      const double c = rhobar / rho, s = beta / rho;
      const double theta = s * alpha;
      rhobar = -c * alpha;
      const double phi = c * phibar;
      phibar = s * phibar;
      lsqr_update_kernel<<<nblocks(d), 256, 0, st>>>(d, w.y, w.w, w.v, phi / rho, -theta / rho);
      note_launch();
      const double arnorm = alpha * fabs(s * phi);
      if (phibar == 0.0) {
        test2 = 0.0;
        break;
      }
      test2 = arnorm / (sqrt(anorm2) * phibar);
      if (test2 <= tau_r) break;
    }
  } else {
    test2 = 0.0;
  }
  skh_trace_mark(st, "lsqr");
  // ---- Step 5: x = R^{-1} y
  cudaMemcpyAsync(x, w.y, sizeof(double) * (size_t)d, cudaMemcpyDeviceToDevice, st);
  if ((rc = trsv(h, d, w, m, false, x))) return rc;
  info[0] = 4;
  info[1] = it;
  stats[0] = test2;
  stats[1] = phibar;
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("lls");
  skh_trace_mark(st, "step5");
  return SKH_OK;
}

int skh_lls_solve(int64_t n, int64_t d, const double* A, int64_t lda, const double* b, int64_t m, const double* SA,
                  int64_t ldsa, const double* Sb, double tau_a, double tau_r, int64_t it_max, double* x,
                  double* x_s, int64_t* info, double* stats, void* ws, size_t ws_bytes, void* stream) {
  return lls_solve_impl(false, n, d, A, lda, b, m, SA, ldsa, Sb, tau_a, tau_r, it_max, x, x_s, info, stats, ws,
                        ws_bytes, stream);
}

int skh_lls_solve_rr(int64_t n, int64_t d, const double* A, int64_t lda, const double* b, int64_t m,
                     const double* SA, int64_t ldsa, const double* Sb, double rcond, double tau_a, double tau_r,
                     int64_t it_max, double* x, double* x_s, int64_t* info, double* stats, void* ws,
                     size_t ws_bytes, void* stream) {
  return lls_solve_impl(false, n, d, A, lda, b, m, SA, ldsa, Sb, tau_a, tau_r, it_max, x, x_s, info, stats, ws,
                        ws_bytes, stream, true, rcond);
}

int skh_lls_solve_rr_colmajor(int64_t n, int64_t d, const double* A, int64_t lda, const double* b, int64_t m,
                              const double* SA, int64_t ldsa, const double* Sb, double rcond, double tau_a,
                              double tau_r, int64_t it_max, double* x, double* x_s, int64_t* info, double* stats,
                              void* ws, size_t ws_bytes, void* stream) {
  return lls_solve_impl(true, n, d, A, lda, b, m, SA, ldsa, Sb, tau_a, tau_r, it_max, x, x_s, info, stats, ws,
                        ws_bytes, stream, true, rcond);
}

int skh_lls_solve_colmajor(int64_t n, int64_t d, const double* A, int64_t lda, const double* b, int64_t m,
                           const double* SA, int64_t ldsa, const double* Sb, double tau_a, double tau_r,
                           int64_t it_max, double* x, double* x_s, int64_t* info, double* stats, void* ws,
                           size_t ws_bytes, void* stream) {
  return lls_solve_impl(true, n, d, A, lda, b, m, SA, ldsa, Sb, tau_a, tau_r, it_max, x, x_s, info, stats, ws,
                        ws_bytes, stream);
}

}  // extern "C"
