/*
 * skp.h -- C ABI of the B200-native sketched power method (libskp.so).
 *
 * Drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/skpower, a pure NumPy/SciPy package with no FFI of
 * its own; its boundary is the Python call surface re-exported at
 * pkg/src/skpower/__init__.py:25-86).  Each entry point below names the
 * reference operation it replaces.  The Python facade
 * (paper_2605_09755_b200/) binds these with ctypes; INTEGRATION.md shows the
 * binding a maintainer of the reference would add.
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes, no torch types; every array argument is a
 *     DEVICE pointer on the current CUDA device; matrices are row-major with
 *     an explicit leading dimension (elements);
 *   - no allocation inside: scratch comes from the caller (`ws`, sized by the
 *     matching *_ws_bytes query);
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); every call is
 *     asynchronous on it; no host synchronisation unless stated;
 *   - return 0 (SKP_OK) or a status code; skp_last_error() returns the
 *     calling thread's last message.  Thread-safe, stateless.
 */
#ifndef SKP_H_
#define SKP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SKP_OK = 0,
    SKP_ERR_ARG = 1,          /* -> ValueError in the facade */
    SKP_ERR_CUDA = 2,         /* -> RuntimeError */
    SKP_ERR_UNSUPPORTED = 3,  /* -> ValueError ("unsupported") */
    SKP_ERR_NUMERIC = 4
};

const char* skp_last_error(void);
int skp_abi_version(void);
/* Number of kernels this process has launched through libskp (all threads). */
int64_t skp_launch_count(void);
/* 1 if the tcgen05 (sm_100a) GEMM path is compiled in and the device is sm_100. */
int skp_has_tcgen05(void);

/* ---------------------------------------------------------------- K1 ----
 * CountSketch draw, bit-exact with numpy 2.3.5 PCG64.
 * Replaces SketchOperator.__init__ countsketch branch + _draw_countsketch
 * (reference sketching.py:114-124, :141-150).  (st, inc) is the 128-bit PCG64
 * state of _rng(seed) (sketching.py:57-58), split in 64-bit halves.
 * Rows [j0, j1) of the n x s arrays are written to cols[(j-j0)*s + t]
 * (int32 column index, ascending-key order) and signs[...] (+1 / -1).
 * Supported: 1 <= s <= 32, r < 2^31 (s == 1: r <= 2^31 - 1).
 * s == 1 needs `ws` (skp_countsketch_ws_bytes) and synchronises the stream
 * once if Lemire rejections exhaust the first candidate window.            */
int64_t skp_countsketch_ws_bytes(int64_t n, int64_t r, int32_t s);
int skp_countsketch_gen(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                        int64_t n, int64_t r, int32_t s, int64_t j0, int64_t j1,
                        int32_t* cols, int8_t* signs, void* ws, int64_t ws_bytes,
                        void* stream);

/* Column-compressed (CSC) view of S for the gather kernels: colptr[r+1],
 * entries[n*s] = j | (sign < 0) << 31, each column's entries ascending in j
 * (deterministic).  ws: skp_countsketch_csc_ws_bytes.                       */
int64_t skp_countsketch_csc_ws_bytes(int64_t n, int32_t s, int64_t r);
int skp_countsketch_csc(const int32_t* cols, const int8_t* signs, int64_t n, int32_t s,
                        int64_t r, int32_t* colptr, int32_t* entries, void* ws,
                        int64_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- K2 ----
 * out (m x r) = A (m x n) . S, i.e. SketchOperator.apply_right for a
 * countsketch (reference sketching.py:158-164: `a @ self._sparse`).  Fused:
 * fro2 += ||A||_F^2 (double) and nonfinite += #non-finite entries of A (the
 * as_matrix finiteness contract, linalg.py:30-39).  fro2 / nonfinite may be
 * NULL.  With ws (skp_sketch_right_ws_bytes) and 16-byte aligned rows the
 * rows-in-lanes kernel runs (32 rows per warp, chunked CSC in smem); without
 * it a slab kernel gathers per output column.                              */
int64_t skp_sketch_right_ws_bytes(int64_t n, int32_t s, int64_t r, int32_t elem_bytes);
int skp_sketch_right_f32(const float* A, int64_t lda, int64_t m, int64_t n,
                         const int32_t* colptr, const int32_t* entries, int32_t s, int64_t r,
                         float* out, int64_t ldo, double* fro2, int64_t* nonfinite, void* ws,
                         int64_t ws_bytes, void* stream);
int skp_sketch_right_f64(const double* A, int64_t lda, int64_t m, int64_t n,
                         const int32_t* colptr, const int32_t* entries, int32_t s, int64_t r,
                         double* out, int64_t ldo, double* fro2, int64_t* nonfinite, void* ws,
                         int64_t ws_bytes, void* stream);

/* K2 v2 (fp32, range-finder path): the same product written with PERMUTED
 * output columns, out = (A . S) P, by a row gather with a register-resident,
 * bank-conflict-free schedule.  The r columns are cut into ceil(r/800)
 * equal slices (rounded up to an even count; one or two per CTA); P sorts the columns of each slice by entry
 * count; its table is plan[0 .. r) (int32 column of S at each output
 * position; -1 from r to slices*768).  Build the plan once per sketch
 * (skp_sketch_gather_plan, from the
 * CSC view); it is usable iff the int32 at byte offset
 * skp_sketch_gather_plan_fail_offset(r) is 0 after the build -- or, without a
 * host check, run skp_sketch_gather_f32 anyway: with a failed plan it writes
 * nothing and adds 2^40 to *nonfinite (the caller then uses skp_sketch_right).
 * Requires n <= 98304 (rows wider than one 24576-column shared-memory buffer
 * run as up to 4 column passes, each adding to the previous) and 16-byte
 * aligned rows padded to a multiple of 4 floats;
 * returns SKP_ERR_UNSUPPORTED otherwise (callers keep skp_sketch_right).
 * amax (may be NULL): atomicMax of the bits of max |out| (for the 3xFP16
 * split of the output, skp_split_h2_f32 with have_amax = 1).
 * nonfinite (may be NULL) += #non-finite outputs: > 0 iff A has a non-finite
 * entry (every column of A feeds nonzero entries), barring fp32 overflow of a
 * finite sum; fro2 (may be NULL) += ||A||_F^2 by a separate pass.
 * Replaces the same `a @ self._sparse` (sketching.py:158-164) inside
 * range_finder_sketched (power.py:141-154): Y = (A S) Omega = (A S P)(P^T Omega). */
int64_t skp_sketch_gather_plan_bytes(int64_t n, int64_t r);
int64_t skp_sketch_gather_plan_fail_offset(int64_t r);
int skp_sketch_gather_plan(const int32_t* colptr, const int32_t* entries, int64_t n, int64_t r,
                           void* plan, int64_t plan_bytes, void* stream);
int skp_sketch_gather_f32(const float* A, int64_t lda, int64_t m, int64_t n, int64_t r,
                          const void* plan, float scale, float* out, int64_t ldo, double* fro2,
                          int64_t* nonfinite, uint32_t* amax, void* stream);
/* skp_sketch_gather_variant: which gather kernel skp_sketch_gather_f32 runs
 * for (n, r) on the current device -- 3: two slices per CTA on a 16-bit
 * schedule (an even slice count, column passes of <= 16384 words); 2: one
 * slice per CTA.  Diagnostic only (same results either way).                 */
int skp_sketch_gather_variant(int64_t n, int64_t r);
/* skp_sketch_gather_f32_acc64: the same gather of fp32 A with fp64
 * accumulation and an fp64 output (the entries and their signs are exact in
 * fp64): the sketch C~ = K S of the psd Nystrom core (power.py:272-275),
 * whose literal power amplifies an fp32 sketch's rounding.                   */
int skp_sketch_gather_f32_acc64(const float* A, int64_t lda, int64_t m, int64_t n, int64_t r,
                                const void* plan, double scale, double* out, int64_t ldo,
                                double* fro2, int64_t* nonfinite, void* stream);

/* ----------------------------------------------------------- Omega ----
 * out (rows x cols) = Generator(PCG64 (state, inc)).standard_normal((rows,
 * cols)) / divisor, computed on the device, cast to fp32 for _f32 -- the
 * reference's Gaussian start block (power.py:137-138: divisor = sqrt(cols)).
 * numpy's ziggurat is reproduced draw for draw (the wedge test's exp and the
 * tail's log1p are CUDA's: ~2^-52 chance per wedge test of a different accept
 * decision, rare 1-ulp differences in tail values).  A generation that cannot
 * complete (a tail beyond the tracked window: astronomically rare) writes
 * nothing and adds 2^50 to *fail_counter (may be NULL).
 * ws: skp_gaussian_ws_bytes(rows*cols).                                    */
int64_t skp_gaussian_ws_bytes(int64_t count);
int skp_gaussian_f32(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                     int64_t rows, int64_t cols, double divisor, float* out, int64_t ldo,
                     int64_t* fail_counter, void* ws, int64_t ws_bytes, void* stream);
int skp_gaussian_f64(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                     int64_t rows, int64_t cols, double divisor, double* out, int64_t ldo,
                     int64_t* fail_counter, void* ws, int64_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- K3 ----
 * out (r x c) = S^T . X (X n x c); SketchOperator.apply_left_transpose
 * (reference sketching.py:176-182: `self._sparse.T @ a`).                   */
int skp_sketch_left_t_f32(const float* X, int64_t ldx, int64_t n, int64_t c,
                          const int32_t* colptr, const int32_t* entries, int32_t s, int64_t r,
                          float* out, int64_t ldo, void* stream);
int skp_sketch_left_t_f64(const double* X, int64_t ldx, int64_t n, int64_t c,
                          const int32_t* colptr, const int32_t* entries, int32_t s, int64_t r,
                          double* out, int64_t ldo, void* stream);

/* ---------------------------------------------------------------- K4 ----
 * C (M x N) = alpha * op(A) . op(B) + beta * C, row-major.
 * op(A) is M x K: transA == 0 -> A is M x K (lda >= K); 1 -> A is K x M.
 * op(B) is K x N: transB == 0 -> B is K x N (ldb >= N); 1 -> B is N x K.
 * Replaces the dense products of power_iterate (power.py:129-133), randsvd
 * (power.py:194-199) and nystrom_psd (power.py:280-287), which the reference
 * runs through OpenBLAS dgemm.
 * f32 mode: 0 = auto (3xTF32 on tcgen05 when available, else SIMT fp32),
 *           1 = 3xTF32 tcgen05 (error if unavailable), 2 = SIMT fp32 FFMA.
 * f64: SIMT FP64 (mode ignored).
 * ws: skp_gemm_ws_bytes (split-K partials; 0 bytes is always accepted and
 * disables split-K).                                                        */
int64_t skp_gemm_ws_bytes(int transA, int transB, int64_t M, int64_t N, int64_t K,
                          int32_t elem_bytes, int32_t mode);
int skp_gemm_f32(int transA, int transB, int64_t M, int64_t N, int64_t K, float alpha,
                 const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
                 float* C, int64_t ldc, int32_t mode, void* ws, int64_t ws_bytes,
                 void* stream);
int skp_gemm_f64(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                 const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                 double* C, int64_t ldc, int32_t mode, void* ws, int64_t ws_bytes,
                 void* stream);

/* ---------------------------------------------------------------- K5 ----
 * CholeskyQR2 building blocks (replace orthonormalize's pivoted QR,
 * reference linalg.py:57-81).  All fp64, n <= 4096.
 * cholesky: G (n x n, ld) -> lower L in place (strict upper clobbered);
 *   *info (device int) = 0 or the 1-based index of the first non-positive
 *   pivot.                                                                  */
int skp_cholesky_f64(double* G, int64_t n, int64_t ld, int32_t* info, void* stream);
/* Rank check after skp_cholesky_f64: if *info == 0 and
 * min_i L_ii < rel_tol * max_i L_ii, sets *info = -1 (numerically rank
 * deficient; the facade then takes the eigen-based truncating path, matching
 * orthonormalize's column dropping, linalg.py:75-81).                       */
int skp_chol_pivot_check_f64(const double* L, int64_t n, int64_t ld, double rel_tol,
                             int32_t* info, void* stream);
/* Fused K5: G + shift = L L^T, rank check and X = L^{-1} in one cooperative
 * kernel (32-wide panels), shift = shift_rel * max_i G_ii * I (0: plain
 * Cholesky; > 0: the first pass of shifted CholeskyQR3, which replaces the
 * pivoted QR of orthonormalize, linalg.py:57-81, without losing columns to
 * the Gram's rounding floor).  X dense n x n (strict upper zero).  *info
 * (device) is only written on failure: k+1 first non-positive pivot, -1 if
 * min L_ii < rel_tol * max L_ii; callers zero it (failures accumulate).     */
int64_t skp_cholinv_ws_bytes(int64_t n);
int skp_cholinv_f64(const double* G, int64_t n, int64_t ld, double rel_tol, double shift_rel,
                    double* X, int32_t* info, void* ws, int64_t ws_bytes, void* stream);
/* X (n x n, dense, row-major) = L^{-1} (lower; strict upper zeroed). */
int skp_trinv_lower_f64(const double* L, int64_t ldl, int64_t n, double* X, void* stream);

/* ---------------------------------------------------------------- K6 ----
 * Symmetric eigensolver (fp64) for the small cores -- one-CTA cyclic Jacobi
 * for n <= 112, tridiagonal reduction (cluster sytrd) + bisection + inverse
 * iteration + back-transform above (eig_tri.cu):
 * the Gram B B^T of randsvd's B = Q^T A (replaces thin_svd / gesdd,
 * linalg.py:84-88) and the Nystrom W.  A (n x n) is destroyed.  On return
 * W[n] holds eigenvalues DESCENDING and V (n x n) the matching eigenvectors
 * as columns.  *sweeps (device int) = sweeps used.                          */
int64_t skp_syevj_ws_bytes(int64_t n);
int skp_syevj_f64(double* A, int64_t n, double* W, double* V, int32_t max_sweeps,
                  void* ws, int64_t ws_bytes, int32_t* sweeps, void* stream);

/* G (C x C, fp64) = X^T X for fp32 X (K x C): exact fp32 products, fp64
 * accumulation (randsvd's B B^T from B^T, reference power.py:196-197 /
 * linalg.py:84-88 in fp64).  ws: skp_gram_f32_f64_ws_bytes.                 */
int64_t skp_gram_f32_f64_ws_bytes(int64_t K, int64_t C);
int skp_gram_f32_f64(const float* X, int64_t K, int64_t C, int64_t ldx, double* G, int64_t ldg,
                     void* ws, int64_t ws_bytes, void* stream);

/* ----------------------------------------------------------- utilities -- */
int skp_cast_f32_f64(const float* x, double* y, int64_t count, void* stream);
int skp_cast_f64_f32(const double* x, float* y, int64_t count, void* stream);
/* 2-D strided casts: y[i*ldy + j] = x[i*ldx + j] for i < rows, j < cols */
int skp_cast2d_f32_f64(const float* x, int64_t ldx, double* y, int64_t ldy, int64_t rows,
                       int64_t cols, void* stream);
/* skp_gesvj_{f64,f32}: thin SVD A = U diag(S) V^T of A (m x n, m >= n,
 * row-major, lda) by one-sided Jacobi in fp64 (replaces LAPACK gesdd behind
 * thin_svd / pinv, reference linalg.py:84-106): every sigma_i to an absolute
 * ~eps sigma_1, so ill-conditioned inputs keep their small singular values.
 * S descending (n), U (m x n, ldu), V (n x n, ldv), fp64; *sweeps = sweeps
 * run (<= max_sweeps).  ws: skp_gesvj_ws_bytes(m, n).                      */
int64_t skp_gesvj_ws_bytes(int64_t m, int64_t n);
int skp_gesvj_f64(const double* A, int64_t m, int64_t n, int64_t lda, double* S, double* U,
                  int64_t ldu, double* V, int64_t ldv, int32_t max_sweeps, void* ws,
                  int64_t ws_bytes, int32_t* sweeps, void* stream);
int skp_gesvj_f32(const float* A, int64_t m, int64_t n, int64_t lda, double* S, double* U,
                  int64_t ldu, double* V, int64_t ldv, int32_t max_sweeps, void* ws,
                  int64_t ws_bytes, int32_t* sweeps, void* stream);
/* skp_sym_check_{f32,f64}: out[0] = max_ij |A_ij - A_ji|, out[1] = max |A_ij|
 * (n x n, leading dimension ld; fp64 outputs), reading A once -- the
 * symmetry test of _check_psd (power.py:242-255) at any size.              */
int skp_sym_check_f32(const float* A, int64_t n, int64_t ld, double* out, void* stream);
int skp_sym_check_f64(const double* A, int64_t n, int64_t ld, double* out, void* stream);
int skp_cast2d_f64_f32(const double* x, int64_t ldx, float* y, int64_t ldy, int64_t rows,
                       int64_t cols, void* stream);
/* ------------------------------------------------------------ 3xFP16 ----
 * FP32 GEMM on the kind::f16 tensor cores from PRE-SPLIT operands (K4h,
 * gemm_h3.cu) -- the power-iteration products of power.py:129-133.
 * skp_split_h2_f32: X (rows x cols, ld) -> hi, lo (fp16 planes, ldh) with
 * X 2^e ~= hi + lo, e = e_io[0] = 15 - ceil(log2 max|X|) (written on the
 * device; e_io[1] holds the bits of max|X|: computed here, or -- have_amax
 * = 1 -- already accumulated by the caller, e.g. by skp_sketch_gather_f32's
 * amax output); trans=1 writes X^T (cols x rows).
 * skp_gemm_h3: C = alpha op(A) B^T + beta C, computed as 2^-(ea+eb) times
 * the fp32-accumulated A_lo B_hi + A_hi B_lo + A_hi B_hi, with op(A) = A
 * (M x K, transA=0) or A^T (A stored K x M, transA=1, lda % 64 == 0) and B
 * stored N x K.  Planes 16-byte aligned, ld % 8 == 0.  Accuracy ~2^-22 per
 * product (3xTF32: 2^-20).  B_lo = NULL: two products (A_lo B_hi + A_hi B_hi),
 * i.e. B rounded to fp16 (2^-12), A kept to 22 bits -- for the power
 * iteration, whose products only need to preserve the span.
 * ws: skp_gemm_h3_ws_bytes (wave-pacing slots, then split-K partials).     */
int skp_split_h2_f32(const float* X, int64_t rows, int64_t cols, int64_t ld, int32_t trans,
                     void* hi, void* lo, int64_t ldh, int32_t* e_io, int32_t have_amax,
                     void* stream);
/* In place: row i of X (fp32, ld) becomes the fp16 planes [hi | lo]: hi at
 * (half*)X + i*2ld, lo at (half*)X + ld + i*2ld -- planes with leading
 * dimension 2 ld -- so a buffer that is no longer needed in fp32 (A~) is split
 * without a second allocation.  ld % 8 == 0, rows <= 50K columns.           */
int skp_split_h2_inplace_f32(float* X, int64_t rows, int64_t cols, int64_t ld, int32_t* e_io,
                             int32_t have_amax, void* stream);
int64_t skp_gemm_h3_ws_bytes(int transA, int64_t M, int64_t N, int64_t K);
int skp_gemm_h3(int transA, int64_t M, int64_t N, int64_t K, float alpha, const void* A_hi,
                const void* A_lo, int64_t lda, const int32_t* a_exp, const void* B_hi,
                const void* B_lo, int64_t ldb, const int32_t* b_exp, float beta, float* C,
                int64_t ldc, void* ws, int64_t ws_bytes, void* stream);

/* skp_gemm_h3_emit_t: the product of skp_gemm_h3 (beta = 0), written not as
 * fp32 C but as the fp16 split of C^T: Ct_hi, Ct_lo (N x M planes, ldct),
 * C^T 2^e ~= hi + lo with e = e_fixed (fixed = 1; a caller-known bound, e.g.
 * 14 for an orthonormal basis) or ea + eb - shift (fixed = 0; shift = 15 +
 * ceil(log2 K) bounds every entry), stored to *e_out.  An entry that does
 * not fit fp16 (or NaN) sets *overflow (may be NULL).  The epilogue's rows
 * are consecutive in C^T, so the transposed planes are written coalesced:
 * products feed the next product without an fp32 round trip or split pass.
 * b_lower = 1: B (stored N x K) is lower triangular (Q = Y L^-T with L^-1
 * from the Cholesky kernel), so each N tile stops at its own K extent --
 * half the MMAs of the dense product.  ws (may be NULL): skp_gemm_h3_ws_bytes
 * -- its head holds the wave-pacing slots (the N tiles of an M block stay in
 * step so A is read ~once per wave).                                        */
int skp_gemm_h3_emit_t(int transA, int64_t M, int64_t N, int64_t K, float alpha, const void* A_hi,
                       const void* A_lo, int64_t lda, const int32_t* a_exp, const void* B_hi,
                       const void* B_lo, int64_t ldb, const int32_t* b_exp, void* Ct_hi,
                       void* Ct_lo, int64_t ldct, int32_t shift, int32_t fixed, int32_t e_fixed,
                       int32_t* e_out, int32_t* overflow, int32_t b_lower, void* ws,
                       int64_t ws_bytes, void* stream);

/* skp_syrk_h3: C = alpha A^T A (N x N, fp32, exactly symmetric) from the
 * pre-split planes of A stored K x N (kmajor = 0, lda % 64 == 0, both GEMM
 * operands MN-major) or A^T stored N x K (kmajor = 1: the Gram of the rows,
 * e.g. Y^T Y from the planes of Y^T; split over K when there are fewer
 * lower-triangle tiles than CTA pairs, ws: skp_syrk_h3_ws_bytes).  beta:
 * C = alpha A^T A + beta C (block-wise accumulation of G behind a streamed
 * upload).  Replaces the operator A~^T A~ that power.py:131-133 applies
 * twice per power step (y = atil @ (atil.T @ y)): formed once, the q power
 * steps then run in the l-dimensional sketch space (SKETCH-SPACE power
 * iteration).  Only the tiles meeting the lower triangle run;
 * the strict upper triangle is mirrored.  Same 3xFP16 numerics as
 * skp_gemm_h3 (2^-22 per product, register-promoted accumulation).          */
int64_t skp_syrk_h3_ws_bytes(int64_t N, int64_t K);
int skp_syrk_h3(int32_t kmajor, int64_t N, int64_t K, float alpha, const void* A_hi,
                const void* A_lo, int64_t lda, const int32_t* a_exp, float beta, float* C,
                int64_t ldc, void* ws, int64_t ws_bytes, void* stream);

/* skp_gemm_h3s: C = alpha A^T B + beta C with A (K x M, fp32, lda % 32 == 0)
 * split into fp16 hi/lo INSIDE the kernel with the caller's exponent 2^a_exp
 * (a bound on max|A|: skp_h2_exponent_f32), B pre-split as for skp_gemm_h3.
 * randsvd's B^T = A^T Q (power.py:197), whose A is read once.  If a scaled
 * entry of A does not fit fp16 (|a 2^e| >= 65504, or NaN), *overflow |= 1
 * (may be NULL) and C is invalid: the caller recomputes (skp_gemm_f32).
 * skp_h2_exponent_f32: e_io[0] = 15 - ceil(log2 max|X|) - margin_bits, with
 * max|X| computed here or (have_amax = 1) taken from e_io[1]'s bits.        */
int64_t skp_gemm_h3s_ws_bytes(int64_t M, int64_t N, int64_t K);
int skp_gemm_h3s(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                 const int32_t* a_exp, const void* B_hi, const void* B_lo, int64_t ldb,
                 const int32_t* b_exp, float beta, float* C, int64_t ldc, int32_t* overflow,
                 void* ws, int64_t ws_bytes, void* stream);
int skp_h2_exponent_f32(const float* X, int64_t rows, int64_t cols, int64_t ld, int32_t* e_io,
                        int32_t have_amax, int32_t margin_bits, void* stream);

/* ---------------------------------------------------------------- K7 ----
 * SRHT (sketching.py:125-130, :167-171, :185-189): for each of `fibres`
 * input fibres f (element j at X[f*x_fs + j*x_es], j < n),
 *   out[f*o_fs + c*o_es] = scale * (H D pad(x_f))[subset[c]],  c < r,
 * with D = diag(signs) (int8 +-1, n_pad entries), H the unnormalised
 * Sylvester Hadamard matrix of order n_pad (a power of two), scale normally
 * 1/sqrt(r).  A S: fibres = rows of A (x_fs = lda, x_es = 1); S^T X: fibres
 * = columns of X (x_fs = 1, x_es = ldx).  n_pad * sizeof(T) <= 200 KB.      */
int skp_srht_apply_f32(const float* X, int64_t fibres, int64_t n, int64_t x_fs, int64_t x_es,
                       const int8_t* signs, int64_t n_pad, const int32_t* subset, int64_t r,
                       double scale, float* out, int64_t o_fs, int64_t o_es, void* stream);
int skp_srht_apply_f64(const double* X, int64_t fibres, int64_t n, int64_t x_fs, int64_t x_es,
                       const int8_t* signs, int64_t n_pad, const int32_t* subset, int64_t r,
                       double scale, double* out, int64_t o_fs, int64_t o_es, void* stream);

/* In-place column un-permutation X[i, perm[v]] = X[i, v] (v < cols): the
 * K2 v2 output A S P back in the reference's column order, so that
 * apply_right (sketching.py:158-174) runs on the row gather.  cols <= 25600
 * (fp32) / 17066 (fp64); perm = the first `cols` int32 of a gather plan.      */
int skp_unpermute_cols_f32(float* X, int64_t rows, int64_t cols, int64_t ldx, const int32_t* perm,
                           void* stream);
int skp_unpermute_cols_f64(double* X, int64_t rows, int64_t cols, int64_t ldx,
                           const int32_t* perm, void* stream);
/* Row gather y[v, :] = x[perm[v], :], v < rows (P^T Omega for the K2 v2
 * column permutation; perm = the first `rows` int32 of a gather plan).       */
int skp_permute_rows_f32(const float* x, int64_t ldx, const int32_t* perm, float* y, int64_t ldy,
                         int64_t rows, int64_t cols, void* stream);
int skp_permute_rows_f64(const double* x, int64_t ldx, const int32_t* perm, double* y,
                         int64_t ldy, int64_t rows, int64_t cols, void* stream);
/* out[0] += sum of squares (double), nonfinite[0] += #non-finite (either may be NULL) */
int skp_sumsq_f32(const float* X, int64_t rows, int64_t cols, int64_t ld, double* out,
                  int64_t* nonfinite, void* stream);
int skp_sumsq_f64(const double* X, int64_t rows, int64_t cols, int64_t ld, double* out,
                  int64_t* nonfinite, void* stream);
/* W = (W + W^T) / 2 in place (power.py:276, :287) */
int skp_symmetrize_f32(float* W, int64_t n, int64_t ld, void* stream);
int skp_symmetrize_f64(double* W, int64_t n, int64_t ld, void* stream);
/* X[:, j] *= scale[j] */
int skp_scale_cols_f32(float* X, int64_t rows, int64_t cols, int64_t ld, const double* scale,
                       void* stream);
int skp_scale_cols_f64(double* X, int64_t rows, int64_t cols, int64_t ld, const double* scale,
                       void* stream);
/* out[0] = max_ij |G_ij - delta_ij|  (randsvd's orthonormality check, power.py:194-196) */
int skp_orth_dev_f64(const double* G, int64_t n, int64_t ld, double* out, void* stream);
/* Eigen-based orthonormaliser (rank-revealing fallback for orthonormalize):
 * given eigen-decomposition (W desc, V) of G = Y^T Y, writes T (n x n, ld n)
 * = V[:, :k] diag(W[:k]^{-1/2}) padded with zero columns and *k_out = number
 * of eigenvalues > rel_tol * W[0] (device int).                              */
int skp_eig_orth_f64(const double* W, const double* V, int64_t n, double rel_tol, double* T,
                     int32_t* k_out, void* stream);
/* sigma[i] = sqrt(max(W[i], 0)); inv[i] = sigma[i] > 0 ? 1/sigma[i] : 0 */
int skp_sqrt_eigs_f64(const double* W, int64_t n, double* sigma, double* inv, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKP_H_ */
