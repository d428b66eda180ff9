// Residual covariance update with eigenvalue floor (update_sigma, tvm.py:337-358 and
// floor_eigenvalues, _linalg.py:15-24).  One CTA per component, matrix in shared memory.
//
// The reference always reconstructs V max(lambda, floor) V^T.  When no eigenvalue is below
// the floor that reconstruction equals the input up to rounding, so the kernel first tests
// "lambda_min > floor" with a Cholesky factorization of r - floor*I and only runs the
// (parallel cyclic Jacobi) eigensolver when the floor actually bites.
#include <math.h>

#include "common.cuh"
#include "internal.h"
#include "spd_small.cuh"

namespace tvk {

constexpr int kSigmaMaxF = 96;  // r, w, v (3 F^2 doubles) in shared memory: 221 KB at F = 96
constexpr int ST = 256;

// Parallel cyclic Jacobi on the symmetric n x n matrix a (shared, row stride n); v <- eigenvectors
// (columns), a's diagonal <- eigenvalues.  Round-robin pair schedule; n padded to even.
__device__ void block_jacobi_eigh(double* a, double* v, int n, int* pairs /* [2*64] */, double* cs /* [2*32] */) {
  const int tid = threadIdx.x;
  const int m = (n + 1) & ~1;  // even player count; index n (if odd) is a dummy
  for (int i = tid; i < n * n; i += ST) v[i] = (i / n == i % n) ? 1.0 : 0.0;
  __shared__ double off_norm, tot_norm;
  for (int sweep = 0; sweep < 40; sweep++) {
    if (tid == 0) {
      double o = 0.0, t = 0.0;
      for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
          double x = a[i * n + j] * a[i * n + j];
          t += x;
          if (i != j) o += x;
        }
      off_norm = o;
      tot_norm = t;
    }
    __syncthreads();
    if (!(off_norm > 1e-30 * tot_norm) || off_norm == 0.0) break;
    for (int round = 0; round < m - 1; round++) {
      // round-robin: player 0 fixed, others rotate
      if (tid < m / 2) {
        // circle method: seat 0 fixed, seats 1..m-1 rotate; seat i plays seat m-1-i
        int i = tid, ib = m - 1 - i;
        int p = (i == 0) ? 0 : ((i - 1 + round) % (m - 1)) + 1;
        int q = ((ib - 1 + round) % (m - 1)) + 1;
        if (p > q) {
          int t = p;
          p = q;
          q = t;
        }
        pairs[2 * i] = p;
        pairs[2 * i + 1] = q;
        double c = 1.0, s = 0.0;
        if (q < n) {
          double apq = a[p * n + q];
          if (apq != 0.0) {
            double tau = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
            double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        cs[2 * i] = c;
        cs[2 * i + 1] = s;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int idx = tid; idx < (m / 2) * n; idx += ST) {
        int i = idx / n, k = idx % n;
        int p = pairs[2 * i], q = pairs[2 * i + 1];
        if (q >= n) continue;
        double c = cs[2 * i], s = cs[2 * i + 1];
        double ap = a[p * n + k], aq = a[q * n + k];
        a[p * n + k] = c * ap - s * aq;
        a[q * n + k] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J, V <- V J
      for (int idx = tid; idx < (m / 2) * n; idx += ST) {
        int i = idx / n, k = idx % n;
        int p = pairs[2 * i], q = pairs[2 * i + 1];
        if (q >= n) continue;
        double c = cs[2 * i], s = cs[2 * i + 1];
        double ap = a[k * n + p], aq = a[k * n + q];
        a[k * n + p] = c * ap - s * aq;
        a[k * n + q] = s * ap + c * aq;
        double vp = v[k * n + p], vq = v[k * n + q];
        v[k * n + p] = c * vp - s * vq;
        v[k * n + q] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(ST) sigma_floor_kernel(const double* ssum, const double* tb, const double* N,
                                                         const double* sigma_old, int F, double floor_scale,
                                                         double* sigma_out, int32_t* status) {
  extern __shared__ double dyn[];
  double* r = dyn;
  double* w = r + F * F;
  double* v = w + F * F;
  __shared__ int pairs[2 * kSigmaMaxF];
  __shared__ double cs[kSigmaMaxF];
  __shared__ double sh_floor;
  __shared__ int bad;
  const int c = blockIdx.x, tid = threadIdx.x;
  const int64_t off = (int64_t)c * F * F;
  const double n = N[c];
  if (!(n > 0.0)) {
    for (int i = tid; i < F * F; i += ST) sigma_out[off + i] = sigma_old[off + i];
    if (tid == 0) status[c] = TVK_ITEM_SKIPPED;
    return;
  }
  for (int i = tid; i < F * F; i += ST) w[i] = (ssum[off + i] - tb[off + i]) / n;
  __syncthreads();
  for (int i = tid; i < F * F; i += ST) {
    int a = i / F, b = i % F;
    r[i] = 0.5 * (w[a * F + b] + w[b * F + a]);
  }
  __syncthreads();
  if (tid == 0) {
    double tr = 0.0;
    for (int i = 0; i < F; i++) tr += r[i * F + i];
    double scale = tr / F;
    if (scale <= 0.0) {
      double to = 0.0;
      for (int i = 0; i < F; i++) to += sigma_old[off + i * F + i];
      scale = to / F;
    }
    sh_floor = floor_scale * scale;
    bad = 0;
  }
  __syncthreads();
  const double fl = sh_floor;
  if (!(fl > 0.0)) {
    if (tid == 0) status[c] = TVK_ITEM_NOT_SPD;  // collapsed: host raises NumericError
    return;
  }
  // lambda_min > floor  <=>  r - floor*I positive definite
  for (int i = tid; i < F * F; i += ST) w[i] = r[i] - ((i / F == i % F) ? fl : 0.0);
  __syncthreads();
  block_cholesky(w, F, &bad);
  __syncthreads();
  if (!bad) {
    for (int i = tid; i < F * F; i += ST) sigma_out[off + i] = r[i];
    if (tid == 0) status[c] = TVK_ITEM_OK;
    return;
  }
  for (int i = tid; i < F * F; i += ST) w[i] = r[i];
  __syncthreads();
  block_jacobi_eigh(w, v, F, pairs, cs);
  // reconstruct V max(lambda, floor) V^T
  for (int i = tid; i < F * F; i += ST) {
    int a = i / F, b = i % F;
    double s = 0.0;
    for (int k = 0; k < F; k++) s += v[a * F + k] * fmax(w[k * F + k], fl) * v[b * F + k];
    sigma_out[off + i] = s;
  }
  if (tid == 0) status[c] = TVK_ITEM_CLAMPED;
}

}  // namespace tvk

extern "C" int tvk_sigma_floor(const double* ssum, const double* tb, const double* N, const double* sigma_old, int C,
                               int F, double floor_scale, double* sigma_out, int32_t* status, void* stream) {
  TVK_REQUIRE(C >= 0 && F >= 1 && F <= tvk::kSigmaMaxF, "sigma_floor: F must be in [1, 96]");
  TVK_REQUIRE(status != nullptr, "sigma_floor: status array required");
  if (C == 0) return TVK_OK;
  size_t smem = 3 * sizeof(double) * F * F;
  cudaFuncSetAttribute(tvk::sigma_floor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tvk::sigma_floor_kernel<<<C, tvk::ST, smem, (cudaStream_t)stream>>>(ssum, tb, N, sigma_old, F, floor_scale,
                                                                      sigma_out, status);
  TVK_CHECK_LAUNCH("sigma_floor");
  return TVK_OK;
}
