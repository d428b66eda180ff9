// Block-cooperative dense SPD helpers for small matrices held in shared memory.
#pragma once
#include "common.cuh"

namespace tvk {

// In-place lower Cholesky of the n x n row-major matrix a (shared memory), whole block.
// Sets *bad = 1 (shared) if a pivot is not positive (LAPACK dpotrf failure condition).
// The strict upper triangle is left untouched.
__device__ inline void block_cholesky(double* a, int n, int* bad) {
  for (int k = 0; k < n; k++) {
    if (threadIdx.x == 0) {
      double d = a[k * n + k];
      if (!(d > 0.0)) *bad = 1;
      else a[k * n + k] = sqrt(d);
    }
    __syncthreads();
    if (*bad) return;
    double piv = a[k * n + k];
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) a[i * n + k] /= piv;
    __syncthreads();
    int m = n - k - 1;
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
      int r = idx / m, c = idx % m;
      if (c <= r) {
        int i = k + 1 + r, j = k + 1 + c;
        a[i * n + j] -= a[i * n + k] * a[j * n + k];
      }
    }
    __syncthreads();
  }
}

// Given the lower Cholesky factor L in a, overwrite a with the full symmetric inverse
// (L L^T)^-1 = Y^T Y, Y = L^-1 (computed into y).  Whole block.
__device__ inline void block_spd_inverse(double* a, double* y, int n) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    for (int i = 0; i < j; i++) y[i * n + j] = 0.0;
    y[j * n + j] = 1.0 / a[j * n + j];
    for (int i = j + 1; i < n; i++) {
      double s = 0.0;
      for (int k = j; k < i; k++) s += a[i * n + k] * y[k * n + j];
      y[i * n + j] = -s / a[i * n + i];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int i = idx / n, j = idx % n;
    if (j > i) continue;
    double s = 0.0;
    for (int k = i; k < n; k++) s += y[k * n + i] * y[k * n + j];
    a[i * n + j] = s;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int i = idx / n, j = idx % n;
    if (j > i) a[i * n + j] = a[j * n + i];
  }
  __syncthreads();
}

}  // namespace tvk
