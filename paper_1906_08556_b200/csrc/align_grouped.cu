// Grouped full-covariance log-likelihoods of the preselected components (default alignment path).
//
// The reference evaluates the full-covariance log-likelihood of all C components and keeps the
// K preselected ones (gmm.py:412-413), each by a Cholesky factor and a triangular solve
// (gmm.py:111-118: ll = log w - (F log 2pi + log|Sigma|)/2 - ||L^-1 (x - mu)||^2 / 2).  Only the K
// selected values reach the output, so this path evaluates exactly the T*K (frame, component) pairs:
//   1. pairs are bucketed by component (block-local counting sort, one global atomic per
//      (block, component) to reserve a range) and cut into per-component tiles of <= 128 pairs;
//   2. whiten_ll_kernel (persistent, one CTA per SM) gathers the tile's frame rows with cp.async
//      (double-buffered against the math of the previous tile), forms Z = (X - mu) U with
//      U = L^-T upper triangular on the FP64 tensor pipe (DMMA.8x8x4, the zero blocks of U are
//      skipped: 56% of the dense work), and q = rowsum(Z o Z) = ||L^-1 (x - mu)||^2;
//      ll = log w_c - (F log 2pi + log|Sigma_c|)/2 - q/2, scattered to sel_ll[t*K + j].
// Each pair's arithmetic is independent of its position in the sort, so the output is
// bit-reproducible although the bucket order is not.
#include <math.h>

#include "common.cuh"
#include "internal.h"
#include "spd_small.cuh"

namespace tvk {

constexpr int GP = 64;          // padded feature width (F <= 64)
constexpr int GROWS = 128;      // pairs per tile
constexpr int GT = 256;         // threads (8 warps of 32 rows x 4 column blocks)
constexpr int GS = GP + 4;      // smem row stride of U (doubles) and of the frame rows (elements)
constexpr int kSortChunk = 4096;
constexpr int64_t kGroupWindowFrames = 131072;  // 31 MB of f32 frames per window

// Whitening table row: [U = L^-T (64 x 64, zero padded) | mu (64) | const | pad],
// const = log w_c - (F log 2pi + log|Sigma_c|)/2.
constexpr int64_t kWhitenStride = GP * GP + GP + 4;

__global__ void whiten_table_kernel(const double* w, const double* mu, const double* cov, int C, int F,
                                    double* tab, int32_t* status) {
  extern __shared__ double sm[];
  double* a = sm;
  double* y = sm + F * F;
  __shared__ int bad;
  __shared__ double logdet;
  const int c = blockIdx.x;
  const double* src = cov + (int64_t)c * F * F;
  double* dst = tab + (int64_t)c * kWhitenStride;
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
  // y = L^-1 (lower triangular), column-parallel forward substitution
  for (int j = threadIdx.x; j < F; j += blockDim.x) {
    for (int i = 0; i < j; i++) y[i * F + j] = 0.0;
    y[j * F + j] = 1.0 / a[j * F + j];
    for (int i = j + 1; i < F; i++) {
      double s = 0.0;
      for (int k = j; k < i; k++) s += a[i * F + k] * y[k * F + j];
      y[i * F + j] = -s / a[i * F + i];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < GP * GP; idx += blockDim.x) {  // U[i][j] = y[j][i]
    int i = idx / GP, j = idx % GP;
    dst[idx] = (i < F && j < F && j >= i) ? y[j * F + i] : 0.0;
  }
  for (int i = threadIdx.x; i < GP; i += blockDim.x) dst[GP * GP + i] = i < F ? mu[(int64_t)c * F + i] : 0.0;
  if (threadIdx.x == 0) {
    dst[GP * GP + GP] = log(w[c]) - 0.5 * (F * kLog2Pi + logdet);
    dst[GP * GP + GP + 1] = dst[GP * GP + GP + 2] = dst[GP * GP + GP + 3] = 0.0;
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

// per-component tiles of <= GROWS sorted pairs: tile descriptors (first sorted index, rows, comp)
__global__ void tile_count_kernel(const int* hist, int C, int* ntile) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) ntile[c] = (hist[c] + GROWS - 1) / GROWS;
}
__global__ void tile_build_kernel(const int* hist, const int* start, const int* tile_start, int C, int4* tiles) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  int n = hist[c], t0 = tile_start[c];
  for (int i = 0; i * GROWS < n; i++) tiles[t0 + i] = make_int4(start[c] + i * GROWS, min(GROWS, n - i * GROWS), c, 0);
}

template <typename XT>
struct WhitenSmem {
  double U[GP * GS];        // U of the staged component (single buffer: 2 CTAs fit per SM)
  double mu[GP];
  double cst[2];            // const, pad (one 16-byte copy)
  XT X[2][GROWS * GS];      // raw frame rows (columns F..63 stay zero)
  int pair[2][GROWS];
};

template <int BYTES>  // 4 or 8: one frame element
__device__ __forceinline__ void cp_async_elem(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES));
}

// One warp's 16 rows of Z = Y U (all 8 column blocks of 8): column block n needs k-step kk
// (4 wide) only when 4 kk <= 8 n + 7 (U upper triangular).
template <typename XT>
__device__ __forceinline__ void whiten_mma(const XT* X, const double* U, const double* mu, int w, int g, int t4,
                                           double (&acc)[2][8][2]) {
#pragma unroll
  for (int kk = 0; kk < GP / 4; kk++) {
    const int k = kk * 4 + t4;
    const double m = mu[k];
    double a[2];
#pragma unroll
    for (int i = 0; i < 2; i++) a[i] = (double)X[(w * 16 + i * 8 + g) * GS + k] - m;
#pragma unroll
    for (int n = kk / 2; n < 8; n++) {
      const double b = U[k * GS + n * 8 + g];
#pragma unroll
      for (int i = 0; i < 2; i++) dmma884(acc[i][n][0], acc[i][n][1], a[i], b);
    }
  }
}

template <typename XT, bool VEC>
__global__ void __launch_bounds__(GT, 2)
    whiten_ll_kernel(const XT* __restrict__ x, int F, const double* __restrict__ tab, int K, uint64_t kinv,
                     const int32_t* __restrict__ sorted, const int4* __restrict__ tiles, const int* __restrict__ ntile_p,
                     double* __restrict__ sel_ll) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  WhitenSmem<XT>& S = *reinterpret_cast<WhitenSmem<XT>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int ntiles = *ntile_p;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int tb = blockIdx.x * per, te = min(tb + per, ntiles);
  if (tb >= te) return;
  for (int i = tid; i < 2 * GROWS * GS; i += GT) (&S.X[0][0])[i] = (XT)0;
  __syncthreads();

  // issue the copies of tile ti into buffer b (frame rows always, U/mu/const when ucopy)
  auto stage_U = [&](int c) {  // U, mu, const of component c
    const double* src = tab + (int64_t)c * kWhitenStride;
    for (int i = tid; i < GP * GP / 2; i += GT) {  // 16-byte pieces of U rows
      const int row = i / (GP / 2), c2 = i % (GP / 2);
      cp_async16(&S.U[row * GS + 2 * c2], src + row * GP + 2 * c2, 16);
    }
    for (int i = tid; i < GP / 2 + 1; i += GT) {
      if (i < GP / 2) cp_async16(&S.mu[2 * i], src + GP * GP + 2 * i, 16);
      else cp_async16(&S.cst[0], src + GP * GP + GP, 16);
    }
    cp_async_commit();
  };
  auto issue = [&](int ti, int b) {
    const int4 d = tiles[ti];
    for (int r = tid; r < GROWS; r += GT) S.pair[b][r] = r < d.y ? sorted[d.x + r] : -1;
    // frame rows: row r <- x[sorted / K], F elements; warp w copies rows w, w+8, ... (lanes over
    // 16-byte pieces), lane j first fetches the frame index of the warp's j-th row
    const int per_row = VEC ? (F * (int)sizeof(XT)) / 16 : F;
    // frame = pair / K by a 40-bit reciprocal (exact for pair < 2^31, K <= 32)
    const int myrow = warp + (GT / 32) * lane;
    const int myframe = (lane < GROWS / (GT / 32) && myrow < d.y)
                            ? (int)(((uint64_t)(uint32_t)sorted[d.x + myrow] * kinv) >> 40) : 0;
    if (VEC && per_row <= 16) {  // two rows per warp step: lanes 0-15 and 16-31
      const int sub = lane >> 4, c = lane & 15;
      for (int j = 0; j < GROWS / (GT / 32); j += 2) {
        const int r = warp + (GT / 32) * (j + sub);
        const int fr = __shfl_sync(0xffffffffu, myframe, j + sub);
        if (warp + (GT / 32) * j >= d.y) break;
        if (r < d.y && c < per_row)
          cp_async16(reinterpret_cast<uint8_t*>(&S.X[b][r * GS]) + 16 * c,
                     reinterpret_cast<const uint8_t*>(x + (int64_t)fr * F) + 16 * c, 16);
      }
    } else {
      for (int j = 0; j < GROWS / (GT / 32); j++) {
        const int r = warp + (GT / 32) * j;
        const int fr = __shfl_sync(0xffffffffu, myframe, j);
        if (r >= d.y) break;
        const XT* src = x + (int64_t)fr * F;
        for (int c = lane; c < per_row; c += 32) {
          if (VEC) cp_async16(reinterpret_cast<uint8_t*>(&S.X[b][r * GS]) + 16 * c,
                              reinterpret_cast<const uint8_t*>(src) + 16 * c, 16);
          else cp_async_elem<(int)sizeof(XT)>(&S.X[b][r * GS + c], src + c);
        }
      }
    }
    cp_async_commit();
  };

  int comp = -1;
  issue(tb, 0);
  for (int ti = tb; ti < te; ti++) {
    const int xb = (ti - tb) & 1;
    const int4 d = tiles[ti];
    if (d.z != comp) {  // new component: stage U once every warp is done with the previous tile
      __syncthreads();
      stage_U(d.z);
      comp = d.z;
    }
    cp_async_wait<0>();
    __syncthreads();
    // prefetch the next tile's frame rows into the other buffer (its last readers passed the barrier)
    if (ti + 1 < te) issue(ti + 1, xb ^ 1);
    // warp w owns rows 16w..16w+15 of the tile: Z rows, q = rowsum(Z o Z), ll, store -- no more barriers
    if (warp * 16 < d.y) {
      double acc[2][8][2];
#pragma unroll
      for (int i = 0; i < 2; i++)
#pragma unroll
        for (int n = 0; n < 8; n++) acc[i][n][0] = acc[i][n][1] = 0.0;
      whiten_mma(S.X[xb], S.U, S.mu, warp, g, t4, acc);
#pragma unroll
      for (int i = 0; i < 2; i++) {
        double s = 0.0;
#pragma unroll
        for (int n = 0; n < 8; n++) s += acc[i][n][0] * acc[i][n][0] + acc[i][n][1] * acc[i][n][1];
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        const int r = warp * 16 + i * 8 + g;
        if (t4 == 0 && r < d.y) sel_ll[S.pair[xb][r]] = S.cst[0] - 0.5 * s;
      }
    }
  }
}

struct GroupWs {
  int* hist;
  int* start;
  int* cursor;
  int* ntile;
  int* tile_start;
  int4* tiles;
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
  w.ntile = (int*)take(sizeof(int) * C);
  w.tile_start = (int*)take(sizeof(int) * (C + 1));
  w.tiles = (int4*)take(sizeof(int4) * (n_pairs / GROWS + C + 1));
  w.sorted = (int32_t*)take(sizeof(int32_t) * (n_pairs + 1));
  w.bytes = off;
  return w;
}

int64_t grouped_workspace_bytes(int64_t n_pairs, int C) {
  return (int64_t)group_carve(nullptr, std::min<int64_t>(n_pairs, kGroupWindowFrames * 32), C).bytes;
}

template <typename XT, bool VEC>
static int launch_whiten(const XT* x, int F, const double* tab, int K, const GroupWs& w, double* sel_ll, int sms,
                         cudaStream_t st) {
  const size_t smem = sizeof(WhitenSmem<XT>);
  cudaFuncSetAttribute(whiten_ll_kernel<XT, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const uint64_t kinv = ((1ull << 40) + K - 1) / K;
  whiten_ll_kernel<XT, VEC><<<2 * sms, GT, smem, st>>>(x, F, tab, K, kinv, w.sorted, w.tiles, w.tile_start + 0,
                                                       sel_ll);
  TVK_CHECK_LAUNCH("whiten_ll");
  return TVK_OK;
}

template <typename XT>
int grouped_full_ll(const XT* x, int64_t T, int F, const double* ptab, int C, int K, const int32_t* sel,
                    double* sel_ll, void* ws_base, int64_t ws_bytes, cudaStream_t st) {
  TVK_REQUIRE(F <= GP, "grouped full log-likelihood supports F <= 64");
  TVK_REQUIRE(K >= 1 && K <= 32, "grouped full log-likelihood supports K <= 32");
  TVK_REQUIRE(C <= 8192, "grouped full log-likelihood supports C <= 8192");
  const int64_t n_pairs = T * K;
  TVK_REQUIRE(n_pairs < (1ll << 31) - 1, "too many (frame, component) pairs for one call");
  // frame windows sized so the window's frames and the whitening table stay L2-resident while the
  // window's pairs (sorted by component, i.e. random in frame order) gather their frame rows
  const int64_t win = std::min<int64_t>(T, kGroupWindowFrames);
  GroupWs w = group_carve(ws_base, win * K, C);
  TVK_REQUIRE(ws_base != nullptr && (int64_t)w.bytes <= ws_bytes, "grouped full log-likelihood: workspace too small");
  size_t sc_smem = sizeof(int) * 2 * C;
  cudaFuncSetAttribute(pair_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc_smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool vec = ((F * sizeof(XT)) % 16 == 0) && ((uintptr_t)x % 16 == 0);
  for (int64_t f0 = 0; f0 < T; f0 += win) {
    const int64_t nf = std::min<int64_t>(win, T - f0);
    const int64_t np = nf * K;
    const int32_t* wsel = sel + f0 * K;
    cudaMemsetAsync(w.hist, 0, sizeof(int) * C, st);
    int nchunks = (int)((np + kSortChunk - 1) / kSortChunk);
    pair_hist_kernel<<<nchunks, GT, sizeof(int) * C, st>>>(wsel, np, C, w.hist);
    hist_scan_kernel<<<1, 1024, 0, st>>>(w.hist, C, w.start, w.cursor);
    pair_scatter_kernel<<<nchunks, GT, sc_smem, st>>>(wsel, np, C, w.cursor, w.sorted);
    tile_count_kernel<<<(C + 255) / 256, 256, 0, st>>>(w.hist, C, w.ntile);
    hist_scan_kernel<<<1, 1024, 0, st>>>(w.ntile, C, w.tile_start, w.cursor);
    tile_build_kernel<<<(C + 255) / 256, 256, 0, st>>>(w.hist, w.start, w.tile_start, C, w.tiles);
    TVK_CHECK_LAUNCH("pair sort");
    // the kernel reads the tile count from tile_start[C]
    GroupWs wc = w;
    wc.tile_start = w.tile_start + C;
    if (vec)
      TVK_TRY((launch_whiten<XT, true>(x + f0 * F, F, ptab, K, wc, sel_ll + f0 * K, sms, st)));
    else
      TVK_TRY((launch_whiten<XT, false>(x + f0 * F, F, ptab, K, wc, sel_ll + f0 * K, sms, st)));
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
  TVK_REQUIRE(C >= 1 && F >= 1 && F <= tvk::GP, "precision_table: need 1 <= F <= 64");
  size_t smem = 2 * sizeof(double) * F * F;
  cudaFuncSetAttribute(tvk::whiten_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * sizeof(double) * tvk::GP * tvk::GP));
  tvk::whiten_table_kernel<<<C, 256, smem, (cudaStream_t)stream>>>(weights, means, covariances, C, F, table, status);
  TVK_CHECK_LAUNCH("precision_table");
  return TVK_OK;
}

extern "C" int64_t tvk_precision_table_stride(int F) { return tvk::precision_stride(F); }
