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

// small batched SPD factor / inverse / log-determinant (n <= kSmallSpdMax)
constexpr int kSmallSpdMax = 96;
int spd_small(const double* A, int batch, int n, double* chol, double* inv, double* logdet, int* status,
              cudaStream_t st);

}  // namespace tvk
