// UBM EM training helpers (train_gmm_diag / train_gmm_full, gmm.py:228-373).
//
// The E-step itself is built from the shared primitives (frame features -> DMMA GEMM against the
// coefficient table -> row softmax -> one responsibility^T x features GEMM for all sufficient
// statistics).  This file holds the two pieces that have no shared primitive:
//   * seed_dist2: the squared distance of every frame to a newly seeded mean, min-folded into the
//     running distance (_seed_means, gmm.py:228-243).  The per-frame sum reproduces numpy's
//     pairwise summation order bit for bit, so the host-side rng.choice over the copied-back
//     distances draws exactly the frames the reference draws.
//   * full_moments: per component, unpack the [1, x_i, x_i x_j (i<=j)] moment row into the
//     residual-covariance inputs of tvk_sigma_floor (S2 and s1 s1^T / occ) and the new mean.
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace tvk {

constexpr int kSeedMaxF = 128;

// numpy's pairwise_sum (n <= 128) of (row_i - c_i)^2, streamed: n < 8 sums sequentially from 0;
// otherwise 8 interleaved partial sums over the largest multiple of 8, a fixed combine tree, then
// the tail added sequentially.  Explicit _rn intrinsics keep nvcc from contracting into FMAs.
template <typename XT>
__device__ __forceinline__ double np_pairwise_sq(const XT* row, const double* c, int n) {
  auto sq = [&](int i) {
    double v = __dsub_rn((double)row[i], c[i]);
    return __dmul_rn(v, v);
  };
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; i++) r = __dadd_rn(r, sq(i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = sq(j);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], sq(i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; i++) res = __dadd_rn(res, sq(i));
  return res;
}

template <typename XT>
__global__ void seed_dist2_kernel(const XT* __restrict__ x, int64_t T, int F, const double* __restrict__ center,
                                  double* __restrict__ dist2, int init) {
  __shared__ double c[kSeedMaxF];
  for (int i = threadIdx.x; i < F; i += blockDim.x) c[i] = center[i];
  __syncthreads();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    double s = np_pairwise_sq(x + t * F, c, F);
    dist2[t] = init ? s : fmin(dist2[t], s);
  }
}

// One CTA per component.  stats row c: [occ, s1 (F), s2 packed upper (F(F+1)/2)].
__global__ void full_moments_kernel(const double* __restrict__ stats, int F, double occ_min,
                                    const double* __restrict__ mean_old, double* __restrict__ mean,
                                    double* __restrict__ s2, double* __restrict__ tb, double* __restrict__ n_out,
                                    double* __restrict__ trace) {
  const int c = blockIdx.x;
  const int Q = 1 + F + F * (F + 1) / 2;
  const double* row = stats + (int64_t)c * Q;
  const double occ = row[0];
  const bool keep = occ >= occ_min;
  const int64_t off = (int64_t)c * F * F;
  for (int i = threadIdx.x; i < F; i += blockDim.x)
    mean[(int64_t)c * F + i] = keep ? row[1 + i] / occ : mean_old[(int64_t)c * F + i];
  for (int idx = threadIdx.x; idx < F * F; idx += blockDim.x) {
    int a = idx / F, b = idx % F;
    int i = min(a, b), j = max(a, b);
    int p = i * F - i * (i - 1) / 2 + (j - i);  // packed upper, row-major
    s2[off + idx] = row[1 + F + p];
    tb[off + idx] = row[1 + a] * row[1 + b] / occ;
  }
  if (threadIdx.x == 0) {
    n_out[c] = keep ? occ : 0.0;
    // trace of (S2 - s1 s1^T / occ) / occ, summed in tvk_sigma_floor's order
    double tr = 0.0;
    for (int i = 0; i < F; i++) {
      int p = i * F - i * (i - 1) / 2;
      tr += (row[1 + F + p] - row[1 + i] * row[1 + i] / occ) / occ;
    }
    trace[c] = keep ? tr : NAN;
  }
}

}  // namespace tvk

extern "C" int tvk_seed_dist2(const void* x, int x_f64, int64_t T, int F, const double* center, double* dist2,
                              int init, void* stream) {
  TVK_REQUIRE(T >= 0 && F >= 1 && F <= tvk::kSeedMaxF, "seed_dist2: F must be in [1, 128]");
  if (T == 0) return TVK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t blocks = (T + 127) / 128;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (x_f64)
    tvk::seed_dist2_kernel<double><<<(unsigned)blocks, 128, 0, st>>>((const double*)x, T, F, center, dist2, init);
  else
    tvk::seed_dist2_kernel<float><<<(unsigned)blocks, 128, 0, st>>>((const float*)x, T, F, center, dist2, init);
  TVK_CHECK_LAUNCH("seed_dist2");
  return TVK_OK;
}

extern "C" int tvk_full_moments(const double* stats, int C, int F, double occ_min, const double* mean_old,
                                double* mean, double* s2, double* tb, double* n_out, double* trace,
                                void* stream) {
  TVK_REQUIRE(C >= 0 && F >= 1, "full_moments: bad shape");
  if (C == 0) return TVK_OK;
  tvk::full_moments_kernel<<<C, 256, 0, (cudaStream_t)stream>>>(stats, F, occ_min, mean_old, mean, s2, tb, n_out,
                                                                 trace);
  TVK_CHECK_LAUNCH("full_moments");
  return TVK_OK;
}
