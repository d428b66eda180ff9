/*
 * libtvk — B200 (sm_100a) kernels for the GPU i-vector hot path (arXiv 1906.08556).
 *
 * C ABI: plain pointers and sizes, no framework types.  Every pointer argument
 * is DEVICE memory owned by the caller unless stated otherwise; `stream` is a
 * cudaStream_t passed as void*.  Every entry point returns a status code
 * (TVK_OK on success); on failure tvk_last_error() holds a message.  Per-item
 * numeric failures (non-SPD covariance, singular accumulator, ...) are reported
 * through caller-provided int32 status arrays so the host layer can raise or
 * warn exactly like the reference.  No entry point synchronizes the stream and
 * the library keeps no global state (kernel attributes aside).
 *
 * Reference interface replaced by each call (paths relative to the reference
 * package root pkg/src/tvkit/):
 *   tvk_diag_table          GmmDiag.log_likelihoods            gmm.py:56-67   (coefficient table)
 *   tvk_full_table          GmmFull.log_likelihoods            gmm.py:106-119 (coefficient table)
 *   tvk_align_frames        align_frames / select_top_k        gmm.py:376-439
 *   tvk_bw_stats            accumulate_bw_stats                gmm.py:442-492
 *   tvk_spd_small           PosteriorWorkspace per-component   tvm.py:163-171 (chol, inverse, logdet)
 *   tvk_dgemm               every dense contraction            tvm.py:169,190-193,298-302,347,436-444
 *   tvk_dgemm_i8            E-step contractions (FP64 on int8) tvm.py:183-200, 283-302
 *   tvk_posterior           _posterior_terms                   tvm.py:183-215 (chol, Phi, phi, logdet)
 *   tvk_spd_solve_rows      update_T                           tvm.py:317-334
 *   tvk_sigma_floor         update_sigma + floor_eigenvalues   tvm.py:337-358, _linalg.py:15-24
 *   tvk_row_softmax         UBM EM responsibilities            gmm.py:284-287, 345-348
 *   tvk_seed_dist2          _seed_means distance update        gmm.py:228-243
 *   tvk_seed_means          _seed_means draw loop              gmm.py:228-243
 *   tvk_full_moments        train_gmm_full M-step moments      gmm.py:350-366
 */
#ifndef TVK_H_
#define TVK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TVK_OK 0
#define TVK_ERR_INVALID 1 /* bad argument / unsupported shape */
#define TVK_ERR_CUDA 2    /* CUDA launch or runtime error */
#define TVK_ERR_NUMERIC 3 /* reserved: numeric failures are reported per item */

#define TVK_OUT_DENSE 0
#define TVK_OUT_PACKED_LOWER 1 /* row-major lower triangle: (i,j), j<=i at i*(i+1)/2+j */

#define TVK_ITEM_OK 0
#define TVK_ITEM_NOT_SPD 1  /* Cholesky failed (non-SPD covariance / precision / accumulator) */
#define TVK_ITEM_CLAMPED 2  /* eigenvalue floor was applied */
#define TVK_ITEM_SKIPPED 4  /* zero occupancy: item left unchanged */

/* Library version (major*10000 + minor*100 + patch). */
int tvk_version(void);
/* Copies the calling thread's last error message into buf (NUL-terminated); returns its length. */
int tvk_last_error(char* buf, int64_t n);

/* Host-side ALN1 alignment-cache decoder walk (io_formats.py:154-227, read_alignment): for one
 * utterance's u32 frame stream, starts[t] / counts[t] = word offset and entry count of frame t, *end =
 * words consumed.  TVK_ERR_INVALID with the reference's message when the stream is short.  No device. */
int tvk_aln1_scan(const uint32_t* words, int64_t n_words, int64_t n_frames, int64_t* starts, int64_t* counts,
                  int64_t* end);

/* ---------------------------------------------------------------- dense algebra */

/* Batched FP64 GEMM on the DMMA tensor pipe, row-major:
 *   C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b],  op(A) is m x k, op(B) is k x n.
 * trans_a: A stored k x m (lda >= m); else m x k (lda >= k).  trans_b likewise.
 * out_mode TVK_OUT_PACKED_LOWER writes only the lower triangle of the (square) result
 * into packed storage (ldc ignored).  splits > 1 (batch 1 only) splits K over CTAs;
 * partial sums go to `work` (splits*m*n doubles) and are summed in fixed order. */
int tvk_dgemm(int trans_a, int trans_b, int m, int n, int k, double alpha, const double* a, int64_t lda,
              int64_t stride_a, const double* b, int64_t ldb, int64_t stride_b, double beta, double* c,
              int64_t ldc, int64_t stride_c, int batch, int out_mode, int splits, double* work, void* stream);

/* C = alpha op(A) op(B) + beta C (row-major, dense, unbatched) in FP64 emulated on the int8 tensor cores
 * (tcgen05 kind::i8): every row of op(A) and column of op(B) is scaled by a power of two and cut into
 * `digits` (6..8) signed 7-bit digits, the digit products are summed exactly in int32 and combined in
 * FP64; |error| <= (2 + digits) 2^(-7 digits) K max_k|op(A)_mk| max_k|op(B)_kn| (digits = 7: 2^-45.8 K
 * max max).  The E-step contractions L = N U, A += N'M, b = F W, B += F' phi (tvm.py:183-200, 283-302)
 * run here; non-finite inputs give NaN rows / columns.  Bit-reproducible.
 * An operand that is reused across calls (U and W within an EM iteration) can be split once with
 * tvk_i8_split into a buffer of tvk_i8_operand_bytes(rows, k, row_tile, digits) bytes -- op(A) as its
 * m rows with row_tile 128, op(B) as its n columns (rows of op(B)^T) with row_tile 64, element (r, kk)
 * at x[r * rs + kk * ks] -- and passed as a_split / b_split (then a / b are not read). */
int64_t tvk_i8_operand_bytes(int rows, int k, int row_tile, int digits);
int tvk_i8_split(const double* x, int rows, int k, int64_t rs, int64_t ks, int row_tile, int digits, void* out,
                 void* stream);
int tvk_dgemm_i8(int trans_a, int trans_b, int m, int n, int k, double alpha, const double* a, int64_t lda,
                 const void* a_split, const double* b, int64_t ldb, const void* b_split, double beta, double* c,
                 int64_t ldc, int digits, void* stream);

/* Fixed-order reductions (bit-reproducible, no atomics):
 *   tvk_colsum: out[j] = beta*out[j] + alpha * sum_r a[r*lda + j]   (rows x cols)
 *   tvk_ddot:   out[0] = beta*out[0] + alpha * sum_i x_i y_i (y may be NULL: plain sum);
 *               workspace of tvk_ddot_workspace_bytes(). */
int tvk_colsum(const double* a, int64_t rows, int64_t cols, int64_t lda, double alpha, double beta, double* out,
               void* stream);
int64_t tvk_ddot_workspace_bytes(void);
/* Row log-sum-exp and softmax in place (GMM E-step responsibilities, gmm.py:284-287, 345-348):
 * norm[r] = logsumexp(a[r, :]), a[r, :] <- exp(a[r, :] - norm[r]); rows x cols row-major. */
int tvk_row_softmax(double* a, int64_t rows, int cols, double* norm, void* stream);
int tvk_ddot(const double* x, const double* y, int64_t n, double alpha, double beta, double* out, double* workspace,
             void* stream);

/* Batched SPD factorization of n x n matrices (n <= 96): lower Cholesky factor (optional),
 * inverse (optional, full symmetric), log-determinant (optional).  status[i] = TVK_ITEM_NOT_SPD
 * when the factorization of matrix i fails (outputs for it are then undefined).
 * Replaces the per-component loop of PosteriorWorkspace (tvm.py:163-171) and the
 * per-component Cholesky in GmmFull.log_likelihoods (gmm.py:111-118). */
int tvk_spd_small(const double* a, int batch, int n, double* chol, double* inv, double* logdet, int32_t* status,
                  void* stream);

/* ---------------------------------------------------------------- frame posteriors */

/* Diagonal-model coefficient table such that for frame x the diagonal log-likelihood is
 * [x*x, x, 1] . table[:, c]  (gmm.py:56-67).  The buffer holds tvk_diag_table_bytes(C, F) bytes:
 * the (2F+1) x C FP64 matrix first, followed by the tensor-core operands of the preselection
 * (3xTF32 hi/lo split of the coefficients in tcgen05 K-major layout, per-row magnitude bounds,
 * and a component-major FP64 copy for exact rescoring). */
int64_t tvk_diag_table_bytes(int C, int F);
int tvk_diag_table(const double* weights, const double* means, const double* variances, int C, int F,
                   double* table, void* stream);

/* Full-covariance coefficient table Q x C, Q = 1 + F + F(F+1)/2, such that the full
 * log-likelihood is phi(x) . table[:, c] with phi(x) = [1, x_i, x_i x_j (i<=j)]
 * (gmm.py:106-119 as a quadratic-feature GEMM).  status[c] = TVK_ITEM_NOT_SPD if Sigma_c
 * is not positive definite. */
int tvk_full_table(const double* weights, const double* means, const double* covariances, int C, int F,
                   double* table, int32_t* status, void* stream);

/* Per-component whitening table for the grouped (default) path, stride tvk_precision_table_stride(F)
 * doubles.  F <= 64: 64*64 + 64 + 4 = [U_c = L_c^-T (Sigma_c = L_c L_c^T; upper triangular, zero
 * padded to 64 x 64) | mu_c (zero padded to 64) | log w_c - (F log 2pi + log|Sigma_c|)/2 | 0 0 0],
 * so that ll_c(x) = const_c - ||(x - mu_c) U_c||^2 / 2 (gmm.py:111-118's Cholesky + triangular
 * solve).  64 < F <= 128: F(F+1)/2 + F + 2 = [L_c^-1 column-packed lower (column m holds rows
 * m..F-1) | mu_c | const_c | 0].  status as above. */
int tvk_precision_table(const double* weights, const double* means, const double* covariances, int C, int F,
                        double* table, int32_t* status, void* stream);
int64_t tvk_precision_table_stride(int F);

#define TVK_ALIGN_DENSE 1 /* full LLs by the dense quadratic-feature GEMM over all C (else grouped) */

/* Scratch bytes tvk_align_frames needs for T frames, top-K K and C components (either mode). */
int64_t tvk_align_workspace_bytes(int64_t T, int K, int C);

/* Shape envelope: 1 <= K <= min(C, 8192), F <= 128, C <= 24576 (TVK_ERR_INVALID outside).  K <= 32
 * with F <= 63 runs the tensor-core preselection and F <= 64 the DMMA whitening; other shapes run
 * the generic kernels of align_wide.cu (same outputs).  TVK_ALIGN_DENSE needs K <= 32, F <= 96.
 * Sparse frame alignment (gmm.py:389-439) of frames x (T x F, f32 or f64 if x_f64): diagonal top-K
 * preselection (stable, lower index wins ties), full-covariance log-likelihoods of the selected
 * components, softmax over the selection, prune (post >= prune), degenerate rule (argmax in
 * selection order), renormalize, entries sorted by component within a frame.
 * Full log-likelihoods: default (grouped) mode evaluates only the T*K selected pairs, bucketed by
 * component, from prec_table; flags & TVK_ALIGN_DENSE evaluates the quadratic-feature GEMM over
 * all C from full_table and gathers the selected ones (the reference's own work, gmm.py:412).
 * Outputs CSR: offsets (T+1, int64, offsets[T] is the entry count E), components/weights with
 * capacity T*K.  Optional debugging outputs: selected (T*K int32, selection order) and sel_ll
 * (T*K f64 full log-likelihoods). */
int tvk_align_frames(const void* x, int x_f64, int64_t T, int F, const double* diag_table, const double* full_table,
                     const double* prec_table, int C, int K, double prune, int flags, void* workspace,
                     int64_t workspace_bytes, int64_t* offsets, int32_t* components, float* weights,
                     int32_t* selected, double* sel_ll, void* stream);

/* Stable top-K of the diagonal log-likelihoods (select_top_k, gmm.py:376-386 and gmm.py:409-410):
 * selected (T*K int32) in descending order, lower index first on ties; values (T*K f64, may be NULL). */
int tvk_select_topk(const void* x, int x_f64, int64_t T, int F, const double* diag_table, int C, int K,
                    int32_t* selected, double* values, void* stream);

/* Full-covariance log-likelihoods of preselected components only (stage 2 of tvk_align_frames,
 * either mode; grouped mode needs tvk_full_loglik_workspace_bytes of scratch).  sel_ll is T*K f64. */
int64_t tvk_full_loglik_workspace_bytes(int64_t T, int K, int C);
int tvk_full_loglik_selected(const void* x, int x_f64, int64_t T, int F, const double* full_table,
                             const double* prec_table, int C, int K, int flags, const int32_t* selected,
                             double* sel_ll, void* workspace, int64_t workspace_bytes, void* stream);

/* Frame feature expansion used by the dense log-likelihood API (GmmDiag/GmmFull.log_likelihoods):
 * kind 0 -> [x*x, x, 1] (T x (2F+1)); kind 1 -> [1, x_i, x_i x_j (i<=j)] (T x Q).  The dense T x C
 * log-likelihoods are then tvk_dgemm(features, table). */
int tvk_frame_features(const void* x, int x_f64, int64_t T, int F, int kind, double* out, void* stream);

/* ---------------------------------------------------------------- Baum-Welch statistics */

/* Scratch bytes for tvk_bw_stats with at most E alignment entries over U utterances and C components. */
int64_t tvk_bw_workspace_bytes(int64_t E, int U, int C);

/* Per-utterance zeroth/first order statistics (gmm.py:442-492) for U utterances whose frames
 * are rows utt_frames[u]..utt_frames[u+1] of x (f32, or f64 if x_f64; row-major F wide) and whose alignment is
 * the frame CSR (ali_offsets over all frames, components, weights f32).  center (C x F, may be
 * NULL) shifts frames by center[c] before accumulation (standard formulation).
 *   n_out: U x C, f_out: U x C x F (dense, zero for absent components)
 *   S_out: U x C x F x F per-utterance second order (NULL to skip; the reference API path)
 *   ssum_acc: C x F x F, ADDED TO (corpus second-order sum for the E-step; NULL to skip)
 * entry_capacity bounds the batch's entry count (the workspace is sized for it).
 * Reductions run in a fixed order (no floating-point atomics): results are bit-reproducible. */
int tvk_bw_stats(const void* x, int x_f64, int F, const int64_t* utt_frames, int U, const int64_t* ali_offsets,
                 const int32_t* components, const float* weights, int C, const double* center, double* n_out,
                 double* f_out, double* S_out, double* ssum_acc, int64_t entry_capacity, void* workspace,
                 int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- i-vector posterior */

/* Scratch doubles tvk_posterior / tvk_spd_solve_rows need for matrices of order D. */
int64_t tvk_posterior_workspace_bytes(int D, int batch);

#define TVK_POST_ADD_IDENTITY 1 /* L_u = Lpk[u] + I */
#define TVK_POST_MOMENT 2       /* Mpk = Phi + phi phi^T (else Phi) */

/* Batched latent posterior (tvm.py:183-215) from packed precisions (factored in place):
 *   L_u = Lpk[u] (+ I);  R R^T = L_u (Cholesky);  phi_u = L_u^-1 b_u;
 *   Mpk[u] = packed(L_u^-1 [+ phi_u phi_u^T]) (may alias Lpk: computed in place);  logdet[u] = log|L_u|;
 *   bphi[u] = b_u . phi_u.   Any output pointer except phi may be NULL.
 * status[u] = TVK_ITEM_NOT_SPD when L_u is not positive definite. */
int tvk_posterior(const double* lpk, const double* b, int U, int D, int flags, double* phi, double* mpk,
                  double* logdet, double* bphi, int32_t* status, void* workspace, int64_t workspace_bytes,
                  void* stream);

/* Batched SPD solve by rows (update_T, tvm.py:317-334): for item c with skip[c] == 0,
 * X_c = B_c A_c^-1 where A_c is packed D x D SPD and B_c is R x D (row-major); the result
 * overwrites X_c (R x D).  Items that fail to factor get status TVK_ITEM_NOT_SPD and X_c is
 * left unchanged; skipped items get TVK_ITEM_SKIPPED. */
int tvk_spd_solve_rows(const double* apk, const double* b, int batch, int D, int R, const int32_t* skip,
                       double* x, int32_t* status, void* workspace, int64_t workspace_bytes, void* stream);

/* Residual covariance floor (update_sigma, tvm.py:337-358 with _linalg.py:15-24):
 *   r_c = sym((Ssum_c - TB_c) / N_c); scale = tr(r_c)/F (or tr(Sigma_old_c)/F if <= 0);
 *   Sigma_c = floor_eigenvalues(r_c, floor_scale*scale).
 * Items with N_c <= 0 keep Sigma_old_c (status TVK_ITEM_SKIPPED).  status bit TVK_ITEM_CLAMPED
 * reports an applied floor; TVK_ITEM_NOT_SPD reports a non-positive floor (collapse). */
int tvk_sigma_floor(const double* ssum, const double* tb, const double* N, const double* sigma_old, int C, int F,
                    double floor_scale, double* sigma_out, int32_t* status, void* stream);

/* ---------------------------------------------------------------- UBM EM training */

/* k-means++ seeding distances (_seed_means, gmm.py:228-243): d_t = sum_i (x_ti - center_i)^2 summed
 * in numpy's pairwise order (bit-identical to np.sum(..., axis=1)); dist2[t] = d_t when init, else
 * min(dist2[t], d_t).  F <= 128. */
int tvk_seed_dist2(const void* x, int x_f64, int64_t T, int F, const double* center, double* dist2, int init,
                   void* stream);

/* Whole k-means++ seeding loop on the device (_seed_means, gmm.py:228-243), no host round trips.
 * idx[0] (set by the caller) is the first seeded frame; u[0..C-2] are the caller's rng.random()
 * draws, one per rng.choice.  Step c folds the distance to frame idx[c-1] into dist2 (as
 * tvk_seed_dist2) and sets idx[c] = first frame whose dist2 prefix sum exceeds u[c-1] * sum(dist2)
 * (rng.choice's inverse-CDF draw).  If the total at step c is <= 0 or non-finite the loop stops:
 * stop[0] = c, stop[1] = 1 (total <= 0) or 2 (non-finite); dist2 then holds the distances the host
 * needs to continue.  Workspace: tvk_seed_workspace_bytes(T).  F <= 128. */
int64_t tvk_seed_workspace_bytes(int64_t T);
int tvk_seed_means(const void* x, int x_f64, int64_t T, int F, int C, const double* u, int64_t* idx, double* dist2,
                   int32_t* stop, void* workspace, int64_t workspace_bytes, void* stream);

/* Full-covariance M-step moments (train_gmm_full, gmm.py:350-366).  stats is C x Q, Q = 1+F+F(F+1)/2,
 * row c = sum_t r_tc [1, x_i, x_i x_j (i<=j)] (responsibilities^T x tvk_frame_features kind 1).
 * Writes mean_c = s1/occ (mean_old_c when starved), s2_c (full F x F), tb_c = s1 s1^T / occ, n_out[c] = occ (0 when
 * occ < occ_min: starved, tvk_sigma_floor keeps the old covariance) and trace[c] =
 * tr(s2_c - tb_c)/occ (NaN when starved), ready for tvk_sigma_floor(s2, tb, n_out, ...). */
int tvk_full_moments(const double* stats, int C, int F, double occ_min, const double* mean_old, double* mean,
                     double* s2, double* tb, double* n_out, double* trace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TVK_H_ */
