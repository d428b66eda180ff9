// Internal (non-exported) interfaces shared between the libtvk translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tvk {

struct GemmArgs {
  int trans_a, trans_b;
  int M, N, K;
  const double* A;
  int64_t lda, strideA;
  const double* B;
  int64_t ldb, strideB;
  double* C;
  int64_t ldc, strideC;
  double alpha, beta;
  int batch;
  int out_mode;
  int splits;
  double* work;
};

int gemm(const GemmArgs& p, cudaStream_t st);
// FP64 GEMM emulated on the int8 tensor cores (ozaki.cu), dense unbatched C = alpha op(A) op(B) + beta C
int ozaki_gemm(const GemmArgs& p, int digits, const void* a_split, const void* b_split, cudaStream_t st);

// small batched SPD factor / inverse / log-determinant (n <= kSmallSpdMax)
constexpr int kSmallSpdMax = 96;
int spd_small(const double* A, int batch, int n, double* chol, double* inv, double* logdet, int* status,
              cudaStream_t st);

}  // namespace tvk

namespace tvk {
// grouped (selected-only) full-covariance log-likelihoods, align_grouped.cu
// whitening table row: F <= 64 [U = L^-T 64x64 | mu 64 | const | pad]; F > 64 (wide path)
// [column-packed L^-1 (F(F+1)/2) | mu F | const | pad]
__host__ __device__ inline int64_t precision_stride(int F) {
  return F <= 64 ? 64 * 64 + 64 + 4 : (int64_t)F * (F + 1) / 2 + F + 2;
}
constexpr int kGroupedMaxC = 24576;  // pair bucketing keeps 2 C counters in shared memory
int64_t grouped_workspace_bytes(int64_t n_pairs, int C);
template <typename XT>
int grouped_full_ll(const XT* x, int64_t T, int F, const double* ptab, int C, int K, const int32_t* sel,
                    double* sel_ll, void* ws_base, int64_t ws_bytes, cudaStream_t st);
}  // namespace tvk

namespace tvk {
// tensor-core diagonal preselection, select_tc.cu
size_t diag_table_bytes(int C, int F);
int diag_table_tc(const double* tab, int C, int F, cudaStream_t st);
bool select_tc_supported(int F, int K, int C);
template <typename XT>
int select_tc(const XT* x, int64_t T, int F, const double* tab, int C, int K, int32_t* sel, double* val,
              cudaStream_t st);
}  // namespace tvk

namespace tvk {
// approximate (tcgen05 3xTF32) + exact (FP64, kept/ambiguous pairs only) stages 2-3 of align_frames
template <typename XT>
int grouped_align_sparse(const XT* x, int64_t T, int F, const double* ptab, int C, int K, double prune,
                         const int32_t* sel, double* sel_ll, int32_t* comp_pad, float* w_pad, int64_t* counts,
                         void* ws_base, int64_t ws_bytes, cudaStream_t st);
}  // namespace tvk

namespace tvk {
// alignment outside the fast path's envelope, align_wide.cu
constexpr int kWideMaxK = 8192;
constexpr int kWideMaxF = 128;
template <typename XT>
int wide_select(const XT* x, int64_t T, int F, const double* tab, int C, int K, int32_t* sel, double* val,
                cudaStream_t st);
int finalize_wide(int64_t T, int K, double prune, const int32_t* sel, const double* sel_ll, int32_t* comp_pad,
                  float* w_pad, int64_t* counts, cudaStream_t st);
int wide_precision_table(const double* w, const double* mu, const double* cov, int C, int F, double* tab,
                         int32_t* status, cudaStream_t st);
template <typename XT>
int wide_whiten(const XT* x, int F, const double* ptab, int K, const int32_t* sorted, const int4* tiles,
                const int* ntile_dev, int64_t max_tiles, double* sel_ll, cudaStream_t st);
}  // namespace tvk
