// Grouped full-covariance log-likelihoods of the preselected components (default alignment path).
//
// The reference evaluates the full-covariance log-likelihood of all C components and keeps the
// K preselected ones (gmm.py:412-413).  Only those K values reach the output, so this path
// evaluates exactly the T*K (frame, component) pairs:
//   1. pairs are bucketed by component (block-local counting sort, one global atomic per
//      (block, component) to reserve a range);
//   2. grouped_ll_kernel walks the sorted pairs in 128-row tiles; per component run it stages
//      P_c = Sigma_c^-1 (F x F, zero-padded to 64) and Y = x - mu_c in shared memory and forms
//      Z = Y P_c on the FP64 tensor pipe (DMMA.8x8x4); q = rowsum(Z o Y) = (x-mu)' P (x-mu);
//      ll = log w_c - (F log 2pi + log|Sigma_c|)/2 - q/2, scattered to sel_ll[t*K + j].
// Each pair's arithmetic is independent of its position in the sort, so the output is
// bit-reproducible although the bucket order is not.  Work per frame: K*F*64 MACs (2.5% of the
// dense quadratic-feature GEMM at C=2048, K=20).
#include <math.h>

#include "common.cuh"
#include "internal.h"
#include "spd_small.cuh"

namespace tvk {

constexpr int GP = 64;          // padded feature width (F <= 64)
constexpr int GROWS = 128;      // pairs per tile
constexpr int GT = 256;         // threads
constexpr int GS = GP + 4;      // smem row stride (== 4 mod 16: conflict-free fragments)
constexpr int kSortChunk = 4096;
constexpr int64_t kGroupWindowFrames = 131072;  // 31 MB of f32 frames per window



// [P_c (F x F) | mu_c (F) | const_c | pad], const_c = log w_c - (F log 2pi + log|Sigma_c|)/2
__global__ void precision_table_kernel(const double* w, const double* mu, const double* cov, int C, int F,
                                       double* ptab, int32_t* status) {
  extern __shared__ double sm[];
  double* a = sm;
  double* y = sm + F * F;
  __shared__ int bad;
  __shared__ double logdet;
  const int c = blockIdx.x;
  const double* src = cov + (int64_t)c * F * F;
  for (int i = threadIdx.x; i < F * F; i += blockDim.x) a[i] = src[i];
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  block_cholesky(a, F, &bad);
  if (bad) {
    if (threadIdx.x == 0) status[c] = TVK_ITEM_NOT_SPD;
    return;
  }
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < F; i += 32) s += log(a[i * F + i]);
    s = warp_sum(s);
    if (threadIdx.x == 0) logdet = 2.0 * s;
  }
  __syncthreads();
  block_spd_inverse(a, y, F);
  double* dst = ptab + (int64_t)c * precision_stride(F);
  for (int i = threadIdx.x; i < F * F; i += blockDim.x) dst[i] = a[i];
  for (int i = threadIdx.x; i < F; i += blockDim.x) dst[F * F + i] = mu[(int64_t)c * F + i];
  if (threadIdx.x == 0) {
    dst[F * F + F] = log(w[c]) - 0.5 * (F * kLog2Pi + logdet);
    dst[F * F + F + 1] = 0.0;
    status[c] = TVK_ITEM_OK;
  }
}

__global__ void pair_hist_kernel(const int32_t* sel, int64_t n_pairs, int C, int* hist) {
  extern __shared__ int lh[];
  for (int c = threadIdx.x; c < C; c += blockDim.x) lh[c] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortChunk;
  for (int i = threadIdx.x; i < kSortChunk; i += blockDim.x)
    if (base + i < n_pairs) atomicAdd(&lh[sel[base + i]], 1);
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x)
    if (lh[c]) atomicAdd(&hist[c], lh[c]);
}

__global__ void hist_scan_kernel(int* hist, int C, int* start, int* cursor) {
  // single CTA exclusive scan of C counters (C <= 8192)
  __shared__ int part[1024];
  const int per = (C + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(lo + per, C);
  int s = 0;
  for (int c = lo; c < hi; c++) s += hist[c];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < (int)blockDim.x; i++) {
      int v = part[i];
      part[i] = run;
      run += v;
    }
    start[C] = run;
  }
  __syncthreads();
  int run = part[threadIdx.x];
  for (int c = lo; c < hi; c++) {
    start[c] = run;
    cursor[c] = run;
    run += hist[c];
  }
}

__global__ void pair_scatter_kernel(const int32_t* sel, int64_t n_pairs, int C, int* cursor, int32_t* sorted) {
  extern __shared__ int sh[];
  int* lh = sh;       // local counts -> local cursor
  int* lb = sh + C;   // global base per component
  constexpr int PER = kSortChunk / GT;
  for (int c = threadIdx.x; c < C; c += blockDim.x) lh[c] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortChunk;
  int rank[PER], comp[PER];
#pragma unroll
  for (int k = 0; k < PER; k++) {
    int64_t p = base + threadIdx.x + k * GT;
    comp[k] = p < n_pairs ? sel[p] : -1;
    rank[k] = comp[k] >= 0 ? atomicAdd(&lh[comp[k]], 1) : 0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x)
    if (lh[c]) lb[c] = atomicAdd(&cursor[c], lh[c]);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PER; k++) {
    int64_t p = base + threadIdx.x + k * GT;
    if (comp[k] >= 0) sorted[lb[comp[k]] + rank[k]] = (int32_t)p;
  }
}

template <typename XT>
__global__ void __launch_bounds__(GT) grouped_ll_kernel(const XT* x, int F, const double* ptab, const int32_t* sel,
                                                        int K, const int32_t* sorted, int64_t n_pairs,
                                                        double* sel_ll) {
  extern __shared__ __align__(16) double sm[];
  double* sP = sm;                 // [GP][GS]
  double* sY = sP + GP * GS;       // [GROWS][GS]
  double* sMu = sY + GROWS * GS;   // [GP]
  double* part = sMu + GP;         // [GROWS][2]
  int* sPair = reinterpret_cast<int*>(part + 2 * GROWS);  // [GROWS]
  int* sComp = sPair + GROWS;                              // [GROWS]
  __shared__ int loaded_comp;
  __shared__ double sConst;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // 4 x 2 warps of 32x32
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t PS = precision_stride(F);
  if (tid == 0) loaded_comp = -1;
  for (int i = tid; i < GP * GS; i += GT) sP[i] = 0.0;
  for (int i = tid; i < GROWS * GS; i += GT) sY[i] = 0.0;
  __syncthreads();

  // contiguous tile range per CTA: consecutive tiles mostly share a component (P_c stays staged)
  const int64_t ntiles = (n_pairs + GROWS - 1) / GROWS;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t tile_end = min((int64_t)(blockIdx.x + 1) * per, ntiles);
  for (int64_t tile = blockIdx.x * per; tile < tile_end; tile++) {
    const int64_t s0 = tile * GROWS;
    const int nrow = (int)((n_pairs - s0) < GROWS ? (n_pairs - s0) : GROWS);
    for (int r = tid; r < GROWS; r += GT) {
      int p = r < nrow ? sorted[s0 + r] : -1;
      sPair[r] = p;
      sComp[r] = p >= 0 ? sel[p] : -1;
    }
    __syncthreads();
    int r0 = 0;
    while (r0 < nrow) {
      const int c = sComp[r0];
      int r1 = r0 + 1;
      while (r1 < nrow && sComp[r1] == c) r1++;
      // stage P_c and mu_c unless already resident
      if (c != loaded_comp) {
        const double* src = ptab + (int64_t)c * PS;
        for (int i = tid; i < F * F; i += GT) sP[(i / F) * GS + (i % F)] = src[i];
        for (int i = tid; i < F; i += GT) sMu[i] = src[F * F + i];
        if (tid == 0) sConst = src[F * F + F];
      }
      __syncthreads();
      if (tid == 0) loaded_comp = c;
      // Y rows of this run (rows outside the run are zero)
      for (int idx = tid; idx < GROWS * F; idx += GT) {
        int r = idx / F, f = idx % F;
        double v = 0.0;
        if (r >= r0 && r < r1) {
          int64_t tf = sPair[r] / K;
          v = (double)x[tf * F + f] - sMu[f];
        }
        sY[r * GS + f] = v;
      }
      __syncthreads();
      // Z = Y P on the tensor pipe: warp (wm, wn) owns rows wm*32.., cols wn*32..
      double acc[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
      const bool live = (wm * 32 < r1) && (wm * 32 + 32 > r0);
      if (live) {
#pragma unroll 4
        for (int kk = 0; kk < GP; kk += 4) {
          double a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; i++) a[i] = sY[(wm * 32 + i * 8 + g) * GS + kk + t4];
#pragma unroll
          for (int j = 0; j < 4; j++) b[j] = sP[(kk + t4) * GS + wn * 32 + j * 8 + g];
#pragma unroll
          for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
      }
      // q partial = sum over this warp's 32 columns of Z o Y
#pragma unroll
      for (int i = 0; i < 4; i++) {
        int r = wm * 32 + i * 8 + g;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          int col = wn * 32 + j * 8 + 2 * t4;
          s += acc[i][j][0] * sY[r * GS + col] + acc[i][j][1] * sY[r * GS + col + 1];
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (t4 == 0) part[r * 2 + wn] = s;
      }
      __syncthreads();
      for (int r = r0 + tid; r < r1; r += GT) {
        double q = part[r * 2] + part[r * 2 + 1];
        sel_ll[sPair[r]] = sConst - 0.5 * q;
      }
      __syncthreads();
      r0 = r1;
    }
  }
}

struct GroupWs {
  int* hist;
  int* start;
  int* cursor;
  int32_t* sorted;
  size_t bytes;
};

static size_t gup(size_t v) { return (v + 255) & ~size_t(255); }

static GroupWs group_carve(void* base, int64_t n_pairs, int C) {
  GroupWs w{};
  char* b = (char*)base;
  size_t off = 0;
  auto take = [&](size_t n) {
    char* p = b ? b + off : nullptr;
    off += gup(n);
    return p;
  };
  w.hist = (int*)take(sizeof(int) * C);
  w.start = (int*)take(sizeof(int) * (C + 1));
  w.cursor = (int*)take(sizeof(int) * C);
  w.sorted = (int32_t*)take(sizeof(int32_t) * (n_pairs + 1));
  w.bytes = off;
  return w;
}

int64_t grouped_workspace_bytes(int64_t n_pairs, int C) {
  return (int64_t)group_carve(nullptr, std::min<int64_t>(n_pairs, kGroupWindowFrames * 32), C).bytes;
}

template <typename XT>
int grouped_full_ll(const XT* x, int64_t T, int F, const double* ptab, int C, int K, const int32_t* sel,
                    double* sel_ll, void* ws_base, int64_t ws_bytes, cudaStream_t st) {
  TVK_REQUIRE(F <= GP, "grouped full log-likelihood supports F <= 64");
  TVK_REQUIRE(C <= 8192, "grouped full log-likelihood supports C <= 8192");
  const int64_t n_pairs = T * K;
  TVK_REQUIRE(n_pairs < (1ll << 31) - 1, "too many (frame, component) pairs for one call");
  // frame windows sized so the window's frames and the precision table stay L2-resident while the
  // window's pairs (sorted by component, i.e. random in frame order) gather their frame rows
  const int64_t win = std::min<int64_t>(T, kGroupWindowFrames);
  GroupWs w = group_carve(ws_base, win * K, C);
  TVK_REQUIRE(ws_base != nullptr && (int64_t)w.bytes <= ws_bytes, "grouped full log-likelihood: workspace too small");
  size_t sc_smem = sizeof(int) * 2 * C;
  cudaFuncSetAttribute(pair_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc_smem);
  size_t smem = sizeof(double) * (GP * GS + GROWS * GS + GP + 2 * GROWS) + sizeof(int) * 2 * GROWS;
  cudaFuncSetAttribute(grouped_ll_kernel<XT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, grouped_ll_kernel<XT>, GT, smem);
  for (int64_t f0 = 0; f0 < T; f0 += win) {
    const int64_t nf = std::min<int64_t>(win, T - f0);
    const int64_t np = nf * K;
    const int32_t* wsel = sel + f0 * K;
    cudaMemsetAsync(w.hist, 0, sizeof(int) * C, st);
    int nchunks = (int)((np + kSortChunk - 1) / kSortChunk);
    pair_hist_kernel<<<nchunks, GT, sizeof(int) * C, st>>>(wsel, np, C, w.hist);
    hist_scan_kernel<<<1, 1024, 0, st>>>(w.hist, C, w.start, w.cursor);
    pair_scatter_kernel<<<nchunks, GT, sc_smem, st>>>(wsel, np, C, w.cursor, w.sorted);
    TVK_CHECK_LAUNCH("pair sort");
    int64_t ntiles = (np + GROWS - 1) / GROWS;
    int grid = (int)std::min<int64_t>(ntiles, (int64_t)sms * std::max(per, 1));
    grouped_ll_kernel<XT><<<grid, GT, smem, st>>>(x + f0 * F, F, ptab, wsel, K, w.sorted, np, sel_ll + f0 * K);
    TVK_CHECK_LAUNCH("grouped_ll");
  }
  return TVK_OK;
}

template int grouped_full_ll<float>(const float*, int64_t, int, const double*, int, int, const int32_t*, double*,
                                    void*, int64_t, cudaStream_t);
template int grouped_full_ll<double>(const double*, int64_t, int, const double*, int, int, const int32_t*,
                                     double*, void*, int64_t, cudaStream_t);

}  // namespace tvk

extern "C" int tvk_precision_table(const double* weights, const double* means, const double* covariances, int C,
                                   int F, double* table, int32_t* status, void* stream) {
  TVK_REQUIRE(C >= 1 && F >= 1 && F <= tvk::kSmallSpdMax, "precision_table: need 1 <= F <= 96");
  size_t smem = 2 * sizeof(double) * F * F;
  cudaFuncSetAttribute(tvk::precision_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * sizeof(double) * tvk::kSmallSpdMax * tvk::kSmallSpdMax));
  tvk::precision_table_kernel<<<C, 256, smem, (cudaStream_t)stream>>>(weights, means, covariances, C, F, table,
                                                                      status);
  TVK_CHECK_LAUNCH("precision_table");
  return TVK_OK;
}

extern "C" int64_t tvk_precision_table_stride(int F) { return tvk::precision_stride(F); }
