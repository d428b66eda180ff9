// Batched small SPD kernels (n <= 96, one CTA per matrix, matrix resident in shared memory).
//
// Used for the per-component F x F covariances: PosteriorWorkspace (tvm.py:163-171:
// cho_factor, cho_solve(I), log|Sigma|), the full-covariance alignment table
// (gmm.py:111-118: Cholesky + log|L|), and the predictive-covariance UBM.
#include "common.cuh"
#include "internal.h"
#include "spd_small.cuh"

namespace tvk {

__global__ void spd_small_kernel(const double* A, int n, double* chol, double* inv, double* logdet, int32_t* status) {
  extern __shared__ double sm[];
  double* a = sm;          // n x n working matrix -> lower Cholesky factor
  double* y = sm + n * n;  // n x n scratch (inverse of the factor)
  __shared__ int bad;
  const int64_t b = blockIdx.x;
  const double* src = A + b * (int64_t)n * n;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) a[i] = src[i];
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  block_cholesky(a, n, &bad);
  if (bad) {
    if (threadIdx.x == 0 && status) status[b] = TVK_ITEM_NOT_SPD;
    return;
  }
  if (threadIdx.x == 0 && status) status[b] = TVK_ITEM_OK;
  if (logdet && threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) s += log(a[i * n + i]);
    s = warp_sum(s);
    if (threadIdx.x == 0) logdet[b] = 2.0 * s;
  }
  if (chol) {
    double* dst = chol + b * (int64_t)n * n;
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
      int r = i / n, c = i % n;
      dst[i] = c <= r ? a[i] : 0.0;
    }
  }
  if (inv) {
    block_spd_inverse(a, y, n);
    double* dst = inv + b * (int64_t)n * n;
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) dst[i] = a[i];
  }
}

int spd_small(const double* A, int batch, int n, double* chol, double* inv, double* logdet, int* status,
              cudaStream_t st) {
  TVK_REQUIRE(n >= 1 && n <= kSmallSpdMax, "spd_small: order must be in [1, 96]");
  if (batch <= 0) return TVK_OK;
  size_t smem = 2 * sizeof(double) * n * n;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(spd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(2 * sizeof(double) * kSmallSpdMax * kSmallSpdMax));
    attr = true;
  }
  spd_small_kernel<<<batch, 256, smem, st>>>(A, n, chol, inv, logdet, status);
  TVK_CHECK_LAUNCH("spd_small");
  return TVK_OK;
}

}  // namespace tvk

extern "C" int tvk_spd_small(const double* a, int batch, int n, double* chol, double* inv, double* logdet,
                             int32_t* status, void* stream) {
  return tvk::spd_small(a, batch, n, chol, inv, logdet, status, (cudaStream_t)stream);
}
