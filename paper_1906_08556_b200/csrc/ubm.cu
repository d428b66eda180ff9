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

// ---------------------------------------------------------------- device-resident seeding loop
//
// All C-1 draws of _seed_means run on the device without a host round trip.  The caller draws the
// C-1 uniforms u_c up front (rng.choice(T, p) consumes exactly one rng.random() per call), so the
// random stream is the reference's.  Step c: (1) fold the distance to mean c-1 (frame idx[c-1]) into
// dist2 (bit-identical to numpy) and write per-block partial sums in a fixed order; (2) one warp
// finds the first frame whose prefix sum of dist2 exceeds u_c * total -- numpy's
// cdf.searchsorted(u, 'right') over cumsum(dist2 / total) / cdf[-1] up to the rounding of the
// prefix sums, i.e. the same frame unless u_c lands within a few ulps of a CDF step.
// A non-positive total (every frame coincides with a chosen mean; the reference then draws with
// rng.integers) or a non-finite one (rng.choice raises) stops the loop and is reported to the
// host, which replays the random stream and finishes the remaining draws itself.

constexpr int kSeedThreads = 256;

template <typename XT>
__global__ void __launch_bounds__(kSeedThreads)
    seed_step_kernel(const XT* __restrict__ x, int64_t T, int F, int64_t per, const int64_t* __restrict__ idx, int c,
                     double* __restrict__ dist2, double* __restrict__ bsum, const int32_t* __restrict__ stop) {
  if (stop[0]) return;
  __shared__ double cen[kSeedMaxF];
  __shared__ double red[kSeedThreads / 32];
  const XT* crow = x + idx[c - 1] * F;
  for (int i = threadIdx.x; i < F; i += blockDim.x) cen[i] = (double)crow[i];
  __syncthreads();
  const int64_t lo = blockIdx.x * per, hi = min(T, lo + per);
  double acc = 0.0;
  for (int64_t t = lo + threadIdx.x; t < hi; t += blockDim.x) {
    double s = np_pairwise_sq(x + t * F, cen, F);
    double v = c == 1 ? s : fmin(dist2[t], s);
    dist2[t] = v;
    acc += v;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < kSeedThreads / 32; w++) b += red[w];
    bsum[blockIdx.x] = b;
  }
}

// Walk v[0..n) from running sum `acc`; first j with acc + v[j] > thr (else the last j with v[j] > 0).
__device__ __forceinline__ int64_t seed_walk(const double* v, int64_t n, double& acc, double thr) {
  int64_t last = -1;
  for (int64_t j = 0; j < n; j++) {
    double nxt = acc + v[j];
    if (v[j] > 0.0) last = j;
    if (nxt > thr && v[j] > 0.0) return j;
    acc = nxt;
  }
  return last;
}

// One warp: lane chunks of the block sums -> crossing block -> lane chunks of that block's
// frames -> crossing frame.
__global__ void seed_draw_kernel(const double* __restrict__ dist2, int64_t T, int64_t per, const double* __restrict__ bsum,
                                 int nb, const double* __restrict__ u, int c, int64_t* __restrict__ idx,
                                 int32_t* __restrict__ stop) {
  if (stop[0]) return;
  const int lane = threadIdx.x;
  // level 1: block sums
  int64_t cb = (nb + 31) / 32, b0 = min((int64_t)nb, lane * cb), b1 = min((int64_t)nb, b0 + cb);
  double ls = 0.0;
  for (int64_t b = b0; b < b1; b++) ls += bsum[b];
  double inc = ls;
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const double total = __shfl_sync(0xffffffffu, inc, 31);
  if (!(total > 0.0) || !isfinite(total)) {
    if (lane == 0) {
      stop[0] = c;
      stop[1] = isfinite(total) ? 1 : 2;
    }
    return;
  }
  const double thr = u[c - 1] * total;
  unsigned hit = __ballot_sync(0xffffffffu, inc > thr && ls > 0.0);
  int l = hit ? __ffs(hit) - 1 : 31 - __clz(__ballot_sync(0xffffffffu, ls > 0.0));
  double acc = __shfl_sync(0xffffffffu, inc - ls, l);
  int64_t blk = 0;
  if (lane == l) {
    int64_t lb0 = min((int64_t)nb, l * cb), lb1 = min((int64_t)nb, lb0 + cb);
    blk = lb0 + seed_walk(bsum + lb0, lb1 - lb0, acc, thr);
  }
  blk = __shfl_sync(0xffffffffu, blk, l);
  acc = __shfl_sync(0xffffffffu, acc, l);
  // level 2: frames of the crossing block; acc = sum of all earlier blocks
  const int64_t f0 = blk * per, f1 = min(T, f0 + per);
  int64_t cf = (f1 - f0 + 31) / 32, e0 = min(f1, f0 + lane * cf), e1 = min(f1, e0 + cf);
  double fs = 0.0;
  for (int64_t t = e0; t < e1; t++) fs += dist2[t];
  double finc = fs;
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, finc, o);
    if (lane >= o) finc += y;
  }
  hit = __ballot_sync(0xffffffffu, acc + finc > thr && fs > 0.0);
  l = hit ? __ffs(hit) - 1 : 31 - __clz(__ballot_sync(0xffffffffu, fs > 0.0));
  if (lane == l) {
    double a2 = acc + (finc - fs);
    int64_t le0 = min(f1, f0 + l * cf), le1 = min(f1, le0 + cf);
    idx[c] = le0 + seed_walk(dist2 + le0, le1 - le0, a2, thr);
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

extern "C" int64_t tvk_seed_workspace_bytes(int64_t T) {
  int64_t nb = (T + tvk::kSeedThreads - 1) / tvk::kSeedThreads;
  if (nb > 148 * 8) nb = 148 * 8;
  return (nb < 1 ? 1 : nb) * (int64_t)sizeof(double);
}

extern "C" int tvk_seed_means(const void* x, int x_f64, int64_t T, int F, int C, const double* u, int64_t* idx,
                              double* dist2, int32_t* stop, void* workspace, int64_t workspace_bytes, void* stream) {
  TVK_REQUIRE(T >= 1 && F >= 1 && F <= tvk::kSeedMaxF && C >= 1, "seed_means: bad shape (F must be <= 128)");
  TVK_REQUIRE(workspace_bytes >= tvk_seed_workspace_bytes(T), "seed_means: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nb = tvk_seed_workspace_bytes(T) / (int64_t)sizeof(double);
  int64_t per = (T + nb - 1) / nb;
  nb = (T + per - 1) / per;
  double* bsum = (double*)workspace;
  cudaMemsetAsync(stop, 0, 2 * sizeof(int32_t), st);
  for (int c = 1; c < C; c++) {
    if (x_f64)
      tvk::seed_step_kernel<double><<<(unsigned)nb, tvk::kSeedThreads, 0, st>>>((const double*)x, T, F, per, idx, c,
                                                                                 dist2, bsum, stop);
    else
      tvk::seed_step_kernel<float><<<(unsigned)nb, tvk::kSeedThreads, 0, st>>>((const float*)x, T, F, per, idx, c,
                                                                                dist2, bsum, stop);
    tvk::seed_draw_kernel<<<1, 32, 0, st>>>(dist2, T, per, bsum, (int)nb, u, c, idx, stop);
  }
  TVK_CHECK_LAUNCH("seed_means");
  return TVK_OK;
}
