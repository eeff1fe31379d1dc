/*
 * skh.h -- C ABI of libskh.so: the s-hashing sketch hot path of Ski-LLS
 * (Cartis, Fiala & Shao, "Hashing embeddings of optimal dimension, with
 * applications to linear least squares", arXiv 2105.11815) on NVIDIA B200
 * (sm_100a).
 *
 * The operation is Step 1 of the paper's Algorithm 1:
 *   "Randomly draw a sketching matrix S in R^{m x n} ..., compute the
 *    matrix-matrix product SA in R^{m x d} and the matrix-vector product
 *    Sb in R^m",
 * with S an s-hashing matrix (Def. def::sampling_and_hashing, L269-272:
 * "independently for each j in [n], we sample without replacement
 * i_1..i_s in [m] uniformly at random and let S_{i_k j} = +-1/sqrt(s)"), or the
 * hashed randomised Hadamard transform S = S_h H D (Def. def::HRHT, L790-801:
 * D random +-1 diagonal, H_ij = n^{-1/2} (-1)^{<(i-1)_2,(j-1)_2>}).
 * Line numbers are PAPER.md lines; DESIGN.md §3 lists the readings (R1...)
 * where the paper is silent (the random generator, index base, rounding order).
 *
 * Conventions for every entry point
 *  - Pointers named *_host are HOST pointers (pinned memory recommended); every
 *    other array pointer is a DEVICE pointer of the current CUDA device.  All
 *    buffers are owned by the caller.  The library never allocates device
 *    memory: scratch space is the caller-supplied workspace `ws` of at least the
 *    size returned by the matching *_workspace_bytes query, 256-byte aligned.
 *  - Matrices are row-major fp64 with a leading dimension (elements between the
 *    starts of consecutive rows) >= the row length.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Device-pointer calls only enqueue work on `stream` and never synchronise;
 *    outputs are valid once the stream reaches that point.  The *_host calls
 *    enqueue their copies on `stream` too and return immediately; the caller
 *    synchronises `stream` before reading the host outputs.
 *  - Outputs are a pure function of the inputs and are bitwise reproducible run
 *    to run (no floating-point atomics; every sum has a fixed order).
 *  - Return value: SKH_OK (0) or one of the error codes below; on error nothing
 *    has been enqueued, except SKH_ECUDA which reports a failed launch.
 *    skh_last_error() returns a thread-local message for the last failure.
 *  - Safe to call concurrently from several host threads on different streams
 *    with different workspaces.
 */
#ifndef SKH_H_
#define SKH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SKH_OK = 0,
  SKH_EINVAL = 1,      /* n < 0, m < 1, d < 1, s < 1, s > m, s > 64, NULL required pointer */
  SKH_ENOTPOW2 = 2,    /* skh_rht_stages: nrows not a multiple of 2^bit_hi            */
  SKH_EDIM = 3,        /* lda/ldsa/ldx/ldy < d, Sb NULL while b given, bad row map      */
  SKH_ERETRY = 4,      /* reserved: rejection-attempt cap reached (see skh_hash_gen)   */
  SKH_EOVERFLOW = 5,   /* nrows * s >= 2^31 or m >= 2^31 (int32 indices)              */
  SKH_EWORKSPACE = 6,  /* ws NULL or smaller than the *_workspace_bytes query         */
  SKH_ECUDA = 7        /* a CUDA launch or copy failed (detail in skh_last_error())    */
};

/* Static description of an error code. */
const char* skh_strerror(int code);
/* Thread-local message describing the last failing call on this thread. */
const char* skh_last_error(void);
/* ABI version, currently 1. */
int skh_abi_version(void);
/* Number of CUDA kernels this process has enqueued through libskh so far
 * (monotonic, all threads and devices); lets a caller count its launches. */
uint64_t skh_launch_count(void);

/* ------------------------------------------------------------------------ *
 * Scale constants (R5, R9, R10).  Each is one IEEE sqrt followed by
 * one IEEE divide in double precision, exactly as the CPU oracle computes it.
 *   skh_c_s(s)        = 1 / sqrt(s)          entry magnitude of S  (L270)
 *   skh_c_n(n_pad)    = 1 / sqrt(n_pad)      normalisation of H     (L796)
 *   skh_c_ns(n_pad,s) = 1 / sqrt(n_pad * s)  S_h H applied once at the end
 * ------------------------------------------------------------------------ */
double skh_c_s(int32_t s);
double skh_c_n(int64_t n_pad);
double skh_c_ns(int64_t n_pad, int32_t s);

/* ------------------------------------------------------------------------ *
 * R1 + R2: draw S_h and transpose it into bucket lists.
 *
 * Draws the columns of S (= rows of A) held by this caller and builds the
 * bucket lists, i.e. the CSR form of S restricted to those columns.  Local
 * column k in [0, nrows) is global column
 *     j(k) = row0 + (k / blk) * stride + (k % blk)      (blk <= 0: j(k) = row0 + k)
 * which must be strictly increasing in k (stride >= blk); it covers contiguous
 * row shards and the strided layout after a butterfly all-to-all.
 *
 * Column j's s rows are drawn by rejection (R1-R4): attempt
 * t = 0, 1, ... draws r_t = floor(u(key, j*2^16 + t) * m / 2^64) with
 * u = splitmix64 output stream keyed by mix64(seed ^ 0x48415348), accepted if
 * not already drawn for j; the k-th accepted row has sign -1 iff bit k of
 * u(key, j*2^16 + 0xFFFF) is set.
 *
 * Outputs (device, caller-owned):
 *   col_rows  [nrows*s] int32  (nullable) bucket of the k-th draw of local col
 *   col_signs [nrows*s] int8   (nullable) its sign (+1/-1), acceptance order
 *   bucket_ptr  [m+1]   int32  bucket b's entries are [bucket_ptr[b], bucket_ptr[b+1])
 *   bucket_rows [nrows*s] int32  LOCAL column k of each entry, ascending in each bucket
 *   bucket_signs[nrows*s] int8   its sign
 * The bucket lists are unique (a column hits a bucket at most once), so they are
 * compared bit-exactly with the oracle.  nrows == 0 gives bucket_ptr = 0.
 * ATTEMPT CAP (read this if you never call skh_hash_status): attempts are capped
 * at 2^16 - 1 per column.  The hardest column is s = m = 64 (s <= 64 is
 * enforced): a coupon collector that misses one of 64 rows in 65535 attempts
 * has probability <= 64 (63/64)^65535 < 1e-440, so the cap is unreachable for
 * every legal (m, s).  If it were ever reached, the kernel would NOT stop
 * short: it completes the column with the smallest unused rows (a
 * deterministic fill that is NOT the canonical draw of R3, so S would differ
 * from the oracle's) and raises a device flag; skh_hash_gen itself returns
 * SKH_OK because the library never synchronises, and only skh_hash_status()
 * (which synchronises) reports SKH_ERETRY.
 * ------------------------------------------------------------------------ */
size_t skh_hash_workspace_bytes(int64_t nrows, int64_t m, int32_t s);
int skh_hash_gen(uint64_t seed, int64_t m, int32_t s,
                 int64_t nrows, int64_t row0, int64_t blk, int64_t stride,
                 int32_t* col_rows, int8_t* col_signs,
                 int32_t* bucket_ptr, int32_t* bucket_rows, int8_t* bucket_signs,
                 void* ws, size_t ws_bytes, void* stream);
/* The s-hashing VARIANT T (Def. def::s-hashing-variant, L683-686: "sample
 * with replacement i_1..i_s in [m] uniformly at random and add +-1/sqrt(s) to
 * T_{i_k j}"; Lemma 8: T = s^{-1/2} (S^(1) + ... + S^(s)) for
 * independent 1-hashings).  Same arguments, outputs and workspace as
 * skh_hash_gen; draw k = 0..s-1 of column j is r_k = floor(u(key, j*2^16 + k)
 * * m / 2^64) with NO rejection (so with s = 1 it equals skh_hash_gen), sign bit
 * k of the sign word.  A row drawn twice for one column appears twice in that
 * bucket (adjacent, + before -; R18); every consumer of bucket lists
 * (skh_sketch_dense, skh_sketch_csr, ...) then computes T A, T b.  Never
 * reports SKH_ERETRY. */
int skh_hash_gen_variant(uint64_t seed, int64_t m, int32_t s,
                         int64_t nrows, int64_t row0, int64_t blk, int64_t stride,
                         int32_t* col_rows, int8_t* col_signs,
                         int32_t* bucket_ptr, int32_t* bucket_rows, int8_t* bucket_signs,
                         void* ws, size_t ws_bytes, void* stream);
/* Synchronises `stream` and returns SKH_OK or SKH_ERETRY for the last
 * skh_hash_gen that used workspace `ws`. */
int skh_hash_status(const void* ws, void* stream);

/* ------------------------------------------------------------------------ *
 * R5, dense: SA = alpha * S A,  Sb = alpha * S b  (Alg. 1 Step 1, L871).
 *
 *   SA[bk, c] = alpha * ( ... ((0 + sg_1 A[r_1, c]) + sg_2 A[r_2, c]) + ... )
 * over bucket bk's list in ascending local row (R10: the order of the
 * oracle, so results are bit-identical to it).  alpha = skh_c_s(s) gives S A;
 * alpha = 1 gives the unscaled signed sums used for sharded partials.
 *   A  [nrows x d], lda >= d;  b [nrows] (nullable);  SA [m x d], ldsa >= d;
 *   Sb [m] (required iff b != NULL).  SA/Sb must not alias A/b.
 * `s` is only validated (1 <= s <= m); the lists define S.
 * ------------------------------------------------------------------------ */
int skh_sketch_dense(int64_t m, int32_t s,
                     const int32_t* bucket_ptr, const int32_t* bucket_rows,
                     const int8_t* bucket_signs,
                     int64_t nrows, int64_t d, const double* A, int64_t lda,
                     const double* b, double* SA, int64_t ldsa, double* Sb,
                     double alpha, void* stream);

/* ------------------------------------------------------------------------ *
 * R5, sparse: SA (dense m x d) and Sb for A in CSR form, same
 * summation order as skh_sketch_dense applied to the rows of A.
 *   row_ptr [nrows+1] int64, col_idx [nnz] int32 (distinct within a row, each
 *   < d), val [nnz] f64, nnz = row_ptr[nrows] (passed by the caller, so the
 *   library needs no device read).  Column indices need not be sorted.
 *   The bucket lists must be complete lists over all nrows rows (each row in
 *   exactly s buckets); bucket_ptr may be an offset view of m consecutive
 *   buckets of them (a bucket strip).  ws: skh_sketch_csr_workspace_bytes
 *   (the expanded (column, value) list of S.A, 12 * s * nnz bytes + 16 * nrows * s).
 *   Errors: SKH_EOVERFLOW if s * nnz >= 2^31.
 * ------------------------------------------------------------------------ */
size_t skh_sketch_csr_workspace_bytes(int64_t nrows, int32_t s, int64_t nnz);
int skh_sketch_csr(int64_t m, int32_t s,
                   const int32_t* bucket_ptr, const int32_t* bucket_rows,
                   const int8_t* bucket_signs,
                   int64_t nrows, int64_t d, int64_t nnz, const int64_t* row_ptr,
                   const int32_t* col_idx, const double* val,
                   const double* b, double* SA, int64_t ldsa, double* Sb,
                   double alpha, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * R3 + R4: Y = alpha * Hhat_[bit_lo,bit_hi) (D?) X along the row index.
 *
 * For every column, the unnormalised radix-2 Walsh-Hadamard butterflies
 * (x_i, x_{i+h}) <- (x_i + x_{i+h}, x_i - x_{i+h}), h = 2^bit, are applied for
 * bit = bit_lo, ..., bit_hi - 1 in that order (R9) to the local row
 * index i in [0, nrows).  With bit_lo = 0, bit_hi = log2(nrows), apply_diag = 1
 * and alpha = skh_c_n(nrows) this is H D X of Def. def::HRHT (L790-801).
 *   apply_diag: multiply local row i by D_{row0+i} before the first stage,
 *     D_g = -1 iff bit (g & 63) of u(mix64(seed ^ 0x44494147), g >> 6) is set
 *     (R7); rows i >= nvalid are read as zero (zero padding, R8).
 *   X [nvalid x d] (ldx >= d), Y [nrows x d] (ldy >= d); Y may alias X
 *   (then nvalid must equal nrows).  nrows must be a multiple of 2^bit_hi.
 *   ws: scratch of skh_rht_stages_workspace_bytes(nrows, nvalid, row0, d) bytes
 *   (task counters of the fused passes, the D bitmap of the generic pass).
 * ------------------------------------------------------------------------ */
size_t skh_rht_stages_workspace_bytes(int64_t nrows, int64_t nvalid, int64_t row0, int64_t d);
/* The HBM-pass split skh_rht_stages uses for `nbits` stages on rows of length d
 * (aligned != 0: X, Y 16-byte aligned with even leading dimensions).  Writes
 * the stage count of each pass (low bits first) into bits_out[0..] and returns
 * the number of passes (at most max_out are written).  One skh_rht_stages call
 * per returned range launches exactly one transform kernel. */
int skh_rht_pass_plan(int nbits, int64_t d, int aligned, int* bits_out, int max_out);
int skh_rht_stages(uint64_t seed, int64_t nrows, int64_t nvalid, int64_t row0,
                   int64_t d, const double* X, int64_t ldx, double* Y, int64_t ldy,
                   int bit_lo, int bit_hi, int apply_diag, double alpha,
                   void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * R1-R5 on one GPU: SA = S_h H D A, Sb = S_h H D b (HRHT, Def. def::HRHT).
 * n is padded to n_pad = 2^ceil(log2 n) with zero rows; S_h hashes all n_pad
 * columns (R8).  SA[bk, :] = skh_c_ns(n_pad, s) * (ascending-row
 * signed sum of the rows of Hhat D [A; 0]) -- bit-identical to the oracle.
 *   A [n x d] (lda >= d), b [n] nullable, SA [m x d] (ldsa >= d), Sb [m].
 * ------------------------------------------------------------------------ */
size_t skh_rht_dense_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d);
int skh_rht_dense(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d,
                  const double* A, int64_t lda, const double* b,
                  double* SA, int64_t ldsa, double* Sb,
                  void* ws, size_t ws_bytes, void* stream);

/* Same computation from HOST buffers: A_host/b_host (pinned recommended) are
 * copied to the device in row chunks whose transfer overlaps the first
 * transform pass; SA_host/Sb_host receive the result.  Enqueued on `stream`;
 * synchronise it before reading SA_host.  Workspace: the same query. */
int skh_rht_dense_host(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d,
                       const double* A_host, int64_t lda, const double* b_host,
                       double* SA_host, int64_t ldsa, double* Sb_host,
                       void* ws, size_t ws_bytes, void* stream);

/* Plain s-hashing from HOST buffers (dense A): hash, copy A in chunks
 * overlapped with nothing else to do, gather, copy SA/Sb back. */
size_t skh_sketch_dense_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d);
int skh_sketch_dense_host(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d,
                          const double* A_host, int64_t lda, const double* b_host,
                          double* SA_host, int64_t ldsa, double* Sb_host,
                          void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * Elementwise helper for sharded use: X[r, c] *= alpha for r < rows, c < cols.
 * ------------------------------------------------------------------------ */
int skh_scale(double* X, int64_t rows, int64_t cols, int64_t ldx, double alpha,
              void* stream);

/* Exchange-free sharded H D A: with
 * H_n = H_G (x) H_L (L = n / G, row i = g L + l), rank r's contribution is
 * T_r Z_r with Z_r = H_L D A_r (its local rows, all local stages) and
 * T_r = sum_g (-1)^popcount(g & r) S_g (S_g: columns g L .. g L + L - 1 of S).
 * Given bucket lists of all n columns of S (skh_hash_gen, row0 = 0, nrows =
 * n, rows = global j), this rewrites them in place into T_r's lists: row
 * j -> j mod L, sign times (-1)^popcount((j / L) & r).  Entries keep their
 * ascending-j order (a fixed summation order). */
int skh_fold_lists(int64_t nentries, int32_t* bucket_rows, int8_t* bucket_signs,
                   int64_t L, int64_t rank, void* stream);

/* The same fold in COLUMN-list form, for the column-major M3 path (the
 * on-chip fan-out of SURVEY §8(e) M3): given the column lists of all n = G L
 * columns of S (skh_hash_gen col_rows / col_signs, nrows = n, row0 = 0;
 * [n][s] row-major), writes T_r's column lists over the L local rows:
 *   fold_rows[l (G s) + g s + q]  = col_rows[(g L + l) s + q]
 *   fold_signs[l (G s) + g s + q] = col_signs[(g L + l) s + q] * (-1)^popcount(g & rank)
 * for l < L, g < G, q < s (device arrays, caller-owned; fold_* hold L G s
 * entries).  A bucket may appear twice in one local row (two blocks g hit it):
 * the sum keeps both terms.  Errors: SKH_EINVAL (L < 1, G < 1, s < 1, rank
 * outside [0, G), null pointers). */
int skh_fold_cols(int64_t L, int64_t G, int32_t s, int64_t rank, const int32_t* col_rows,
                  const int8_t* col_signs, int32_t* fold_rows, int8_t* fold_signs, void* stream);

/* Deterministic ordered sum of G partial blocks laid out consecutively:
 * out[r, c] = (((P_0[r,c] + P_1[r,c]) + P_2[r,c]) + ...) * alpha, where
 * P_g = parts + g * part_stride (elements), each [rows x cols] with ld `ldp`.
 * Used after an all-to-all of SA strips (rank-order reduction). */
int skh_ordered_sum(const double* parts, int64_t G, int64_t part_stride,
                    int64_t rows, int64_t cols, int64_t ldp,
                    double* out, int64_t ldo, double alpha, void* stream);

/* ======================================================================== *
 * Column-major A (the paper's own LAPACK/FFTW storage, L1073-1081): column c
 * of A is A[c*lda .. c*lda + n), lda >= n; SA is column-major m x d,
 * SA[c*ldsa + bucket], ldsa >= m.  Restrictions: s <= 8, m <= 65536.
 * ======================================================================== */

/* R1-R5: SA = S_h H D A, Sb = S_h H D b (Def. def::HRHT, L790-801), n padded
 * to n_pad = 2^L with zero rows.  Two HBM passes: D and the butterflies of
 * row bits 0..12 on contiguous 2^13-row chunks, then the bits 13..L-1 on
 * 2^(L-13)-row groups fused with the sketch (the transformed rows are never
 * written back; each SA column accumulates in on-chip memory).  Bits beyond 21
 * take extra in-place passes of <= 8 bits before the fused one.
 * Summation order (R17): a bucket receives the rows of each 4096-row
 * gather tile in ascending order, tile after tile -- fixed, so the result is
 * bitwise reproducible, but not the oracle's order: SA agrees with the oracle
 * to rounding (relative Frobenius 1e-12) and exactly on integer data.
 *   A [n x d] col-major (lda >= n), b [n] nullable, SA [m x d] col-major
 *   (ldsa >= m), Sb [m] (required iff b).  ws: the workspace query (it holds
 *   the transformed copy of A, (d + 1) * n_pad doubles). */
size_t skh_rht_dense_colmajor_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d);
int skh_rht_dense_colmajor(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d,
                           const double* A, int64_t lda, const double* b,
                           double* SA, int64_t ldsa, double* Sb,
                           void* ws, size_t ws_bytes, void* stream);

/* Column-major H_L D A_r and its sketch with CALLER-GIVEN column lists (the
 * M3 rank step; P:L790-801 for H D, L871 for S_h): A is the
 * rank's L local rows (column-major, column c at A + c lda, lda >= L), D uses
 * global ids row0 + l, H_L is the unnormalised transform over the L rows
 * (padded with zero rows to n_pad, the next power of two >= L), and the
 * sketch takes s_eff entries per row of the transformed (padded) block from
 * col_rows / col_signs ([n_pad][s_eff]: H mixes the padding rows in, so they
 * need lists too; bucket ids in [0, m), signs +-1; e.g. skh_fold_cols' T_r
 * lists, L a power of two, s_eff = G s <= 8).  Output
 * column-major like skh_rht_dense_colmajor: SAt[c ldsa + k] = alpha * (the
 * signed sum of bucket k over the transformed column c), ldsa >= m; Sb[k]
 * likewise for b (optional, L doubles).  alpha = 1 gives the unscaled partial
 * of the deterministic strip reduction.  Workspace:
 * skh_rht_colmajor_lists_workspace_bytes (device, caller-owned).  Errors:
 * SKH_EINVAL (bad sizes, s_eff > 8, null A/SAt/lists, b without Sb),
 * SKH_EWORKSPACE, SKH_ECUDA. */
size_t skh_rht_colmajor_lists_workspace_bytes(int64_t L, int64_t m, int32_t s_eff, int64_t d);
int skh_rht_colmajor_lists(uint64_t seed, int64_t L, int64_t row0, int64_t m, int32_t s_eff, int64_t d,
                           const double* A, int64_t lda, const double* b, const int32_t* col_rows,
                           const int8_t* col_signs, double alpha, double* SAt, int64_t ldsa, double* Sb,
                           void* ws, size_t ws_bytes, void* stream);
/* Same from HOST buffers (pinned recommended): A_host is copied in groups of
 * columns on a library copy stream, each group transformed (pass 1) as soon as
 * it lands; SA_host/Sb_host receive the result.  Synchronise `stream` before
 * reading them.  Workspace: skh_rht_dense_colmajor_workspace_bytes. */
int skh_rht_dense_colmajor_host(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d,
                                const double* A_host, int64_t lda, const double* b_host,
                                double* SA_host, int64_t ldsa, double* Sb_host,
                                void* ws, size_t ws_bytes, void* stream);

/* R1, R2, R5: plain s-hashing SA = S A, Sb = S b of a column-major A.  Two
 * ways, chosen by the workspace the caller passes:
 *  - ws_bytes >= skh_sketch_dense_colmajor_fast_workspace_bytes(n, m, s, d)
 *    (room for a row-major copy of A and of SA): A is transposed (64 x 64
 *    tiles), gathered by rows and SA transposed back -- 3 |A| of traffic at
 *    near copy rate (C3: 2.5x faster than the walk);
 *  - else (skh_sketch_dense_colmajor_workspace_bytes(n, m, s) suffices): one
 *    HBM read of A, gather tiles of consecutive 4096-row blocks walked on chip.
 * Either way every bucket sums its rows in ascending order from +0.0 and scales
 * once by c_s: the result is bit-identical to skh_sketch_dense and to the
 * oracle. */
size_t skh_sketch_dense_colmajor_workspace_bytes(int64_t n, int64_t m, int32_t s);
size_t skh_sketch_dense_colmajor_fast_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d);
int skh_sketch_dense_colmajor(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d,
                              const double* A, int64_t lda, const double* b,
                              double* SA, int64_t ldsa, double* Sb,
                              void* ws, size_t ws_bytes, void* stream);

/* R3 + R4 on column-major data: Y = Hhat D? X along the row index of every
 * column, unnormalised, all log2(nrows) stages low bit to high bit (bit-exact
 * with the oracle's radix-2 order).  nrows = 2^L (else SKH_ENOTPOW2); rows
 * >= nvalid of X read as zero; D uses global rows row0 + i.  Y may alias X
 * when nvalid == nrows.  X [ncols][ldx >= nvalid], Y [ncols][ldy >= nrows]. */
int skh_rht_colmajor(uint64_t seed, int64_t nrows, int64_t nvalid, int64_t row0, int64_t ncols,
                     const double* X, int64_t ldx, double* Y, int64_t ldy, int apply_diag,
                     void* stream);

/* ======================================================================== *
 * HR-DHT (eq. eqn::HR-DHT, "(6.1)", L1066-1075): SA = S_h F D A, Sb = S_h F D b
 * with F the normalised Discrete Hartley Transform, F_ij = n^{-1/2}
 * [cos + sin](2 pi (i-1)(j-1)/n) -- the sketch of the paper's Ski-LLS-dense.
 * Any n (no padding): S_h hashes the n rows.  Fhat y = Re X - Im X of the DFT
 * X of each column: for n = 2^L <= 2^18 the library's own two-pass four-step
 * transform (column-major A is transposed into the workspace first; DESIGN.md
 * §5d), otherwise cuFFT's D2Z with its work area taken from `ws`.  SA = c *
 * (ascending-row signed sums of Fhat D A rows), c = 1/sqrt(n s) (R20).
 * FFT rounding differs from the oracle's: compared to 1e-12 relative Frobenius.
 *   skh_hrdht_dense:          A row-major [n x d] (lda >= d), SA [m x d] (ldsa >= d), s <= 64
 *   skh_hrdht_dense_colmajor: A column-major (lda >= n), SA column-major (ldsa >= m),
 *                             s <= 8, m <= 65536
 * b nullable, Sb required iff b.  ws: the matching query (about two transformed
 * copies of [A b]; for the cuFFT sizes creating the plan needs the device).
 * cuFFT plans are cached per host thread, device, n and batch for the life of
 * the process. */
size_t skh_hrdht_dense_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d);
int skh_hrdht_dense(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d,
                    const double* A, int64_t lda, const double* b,
                    double* SA, int64_t ldsa, double* Sb,
                    void* ws, size_t ws_bytes, void* stream);
size_t skh_hrdht_dense_colmajor_workspace_bytes(int64_t n, int64_t m, int32_t s, int64_t d);
int skh_hrdht_dense_colmajor(uint64_t seed, int64_t n, int64_t m, int32_t s, int64_t d,
                             const double* A, int64_t lda, const double* b,
                             double* SA, int64_t ldsa, double* Sb,
                             void* ws, size_t ws_bytes, void* stream);

/* SR-DHT (eq. eq::SR-DHT, "(7.2)", L1285-1289; Blendenpik's sketch, the
 * paper's comparison in Fig. 1): SA = S_s F D A, Sb = S_s F D b, where row r of
 * the sampling matrix S_s selects column j_r = floor(u(mix64(seed ^
 * 0x53414D50), r) * n / 2^64) with value 1 (independent draws, with
 * replacement; R21).  Same transform as skh_hrdht_dense; SA[r, :] =
 * n^{-1/2} (Fhat D A)[j_r, :].  Row-major A and SA.  No m limit but m >= 1;
 * m < d is allowed (an underdetermined sketch). */
size_t skh_srdht_dense_workspace_bytes(int64_t n, int64_t m, int64_t d);
int skh_srdht_dense(uint64_t seed, int64_t n, int64_t m, int64_t d,
                    const double* A, int64_t lda, const double* b,
                    double* SA, int64_t ldsa, double* Sb,
                    void* ws, size_t ws_bytes, void* stream);

/* ======================================================================== *
 * Algorithm 1 Steps 2-5 (L868-905): the least-squares solve preconditioned by
 * the sketch.  Given Step 1's SA (m x d, row-major, ldsa >= d) and Sb for the
 * row-major A (n x d, lda >= d) and b (n):
 *   Step 2  SA = Q R, Householder QR (the full-rank DGEQRF mode the paper
 *           allows, L1077; R19); SKH_EINVAL if some r_qq == 0;
 *   Step 3  x_s = R^{-1} Q^T Sb; if ||A x_s - b|| <= tau_a: x = x_s, info[0] = 3;
 *   Step 4  LSQR on W = A R^{-1} from y = 0 until the (7.1) estimate
 *           ||W^T r|| / (||W|| ||r||) <= tau_r (L1085-1089) or it_max steps;
 *   Step 5  x = R^{-1} y, info[0] = 4.
 * Paper defaults (L1100-1102): tau_a = 1e-8, tau_r = 1e-6, it_max = 1e4.
 * Outputs: x [d] (device), x_s [d] (device, nullable), info[2] (host:
 * step, LSQR iterations), stats[3] (host: final (7.1) estimate, ||r|| estimate,
 * ||A x_s - b||).  m >= d.  Each LSQR iteration streams A twice through the
 * library's HBM kernels; the loop runs as one CUDA-graph launch with the scalar
 * recurrence on the device (a host-driven loop is the fallback).  This call
 * SYNCHRONISES `stream` and returns when x is ready.
 * Deterministic: fixed-order reductions.  ws: skh_lls_workspace_bytes (it
 * creates the per-thread cuSOLVER/cuBLAS handles, so it needs the device).
 * Errors: argument errors as usual (nothing enqueued); a numerically
 * rank-deficient SA (some |r_qq| <= 1e-12 max|r_jj| in the unpivoted QR) is
 * detected after Step 2 and returns SKH_EINVAL with the workspace already
 * written and x untouched -- skh_lls_solve_rr solves such problems.
 * Environment (read once per process, workspace query and solve alike):
 * SKH_LLS_HOSTLOOP=1 drives Step 4 from the host (bit-identical to the graph);
 * SKH_LLS_RINV=1 forms M = R^{-1} once (dtrsm against I, 2 d^2 doubles more
 * workspace) and applies it as GEMVs instead of the paper's back-solves (L1081):
 * the same minimiser (x = M y for the LSQR solution y of min ||A M y - b||),
 * a different rounding path. */
size_t skh_lls_workspace_bytes(int64_t n, int64_t d, int64_t m);
int skh_lls_solve(int64_t n, int64_t d, const double* A, int64_t lda, const double* b,
                  int64_t m, const double* SA, int64_t ldsa, const double* Sb,
                  double tau_a, double tau_r, int64_t it_max,
                  double* x, double* x_s, int64_t* info, double* stats,
                  void* ws, size_t ws_bytes, void* stream);
/* Same for column-major A (A[c*lda + i], lda >= n) and column-major SA
 * (ldsa >= m) -- the output layout of skh_rht_dense_colmajor; same workspace
 * query.  A x is one thread per row over the columns in order, A^T u partial
 * dot products over 4096-row blocks summed in block order. */
int skh_lls_solve_colmajor(int64_t n, int64_t d, const double* A, int64_t lda, const double* b,
                           int64_t m, const double* SA, int64_t ldsa, const double* Sb,
                           double tau_a, double tau_r, int64_t it_max,
                           double* x, double* x_s, int64_t* info, double* stats,
                           void* ws, size_t ws_bytes, void* stream);

/* Algorithm 1 with the paper's DEFAULT Step 2 (L1076-1077, L1109-1112): a
 * column-pivoted, rank-revealing factorisation SA = Q R~ V^T (V = P) and
 *     p = max{q : |r~_qq| >= rcond}     (1-based q; rcond absolute, default 1e-12),
 * R11 = R~[:p, :p], Q1, V1 its first p columns (L873-886).  Computed as the
 * Householder QR SA = Q0 R0 (cuSOLVER dgeqrf) followed by a column-pivoted
 * Householder QR of the d x d factor, R0 P = Q1 R~ (the library's cooperative
 * kernel, pivot = largest remaining column norm, LAPACK dgeqp3's norm
 * downdating): SA P = (Q0 Q1) R~, the pivots of a CPQR of SA itself (Q0 keeps
 * column norms).  Then Step 3 x_s = V1 R11^{-1} Q1^T Sb, Step 4 LSQR on
 * W = A V1 R11^{-1} (applied as A (N y) and N^T (A^T u) with the d x d matrix
 * N = P [R11^{-1} 0; 0 0]), Step 5 x = V1 R11^{-1} y: x has zeros outside the
 * p pivoted coordinates; for rank-deficient A it attains the minimum residual
 * (the objective, not x, is unique).  info[3] (host): step, LSQR iterations,
 * p.  Workspace: skh_lls_rr_workspace_bytes (4 d^2 doubles more than
 * skh_lls_workspace_bytes).  SKH_EINVAL for rcond < 0 and for d beyond the
 * on-chip reflector of the pivoting kernel (d <= 27000).  Synchronises `stream`
 * (Step 2 reads the d diagonal entries back to choose p). */
size_t skh_lls_rr_workspace_bytes(int64_t n, int64_t d, int64_t m);
int skh_lls_solve_rr(int64_t n, int64_t d, const double* A, int64_t lda, const double* b,
                     int64_t m, const double* SA, int64_t ldsa, const double* Sb, double rcond,
                     double tau_a, double tau_r, int64_t it_max,
                     double* x, double* x_s, int64_t* info, double* stats,
                     void* ws, size_t ws_bytes, void* stream);
int skh_lls_solve_rr_colmajor(int64_t n, int64_t d, const double* A, int64_t lda, const double* b,
                              int64_t m, const double* SA, int64_t ldsa, const double* Sb, double rcond,
                              double tau_a, double tau_r, int64_t it_max,
                              double* x, double* x_s, int64_t* info, double* stats,
                              void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * Stage trace (thread-local).  After skh_trace_set(events, n) with n
 * caller-created cudaEvent_t handles (as void*), every composite entry point
 * (skh_*_colmajor*) records events[0] on its stream when it starts and
 * events[i] after stage i, up to n events; skh_trace_count() returns the number
 * recorded by the last call and skh_trace_name(i) the stage that events[i]
 * closes ("begin" for 0).  skh_trace_set(NULL, 0) disables tracing.
 * ------------------------------------------------------------------------ */
int skh_trace_set(void* const* events, int nevents);
int skh_trace_count(void);
const char* skh_trace_name(int i);

#ifdef __cplusplus
}
#endif
#endif /* SKH_H_ */
