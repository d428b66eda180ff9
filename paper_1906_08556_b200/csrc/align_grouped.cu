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

#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "spd_small.cuh"
#include "finalize.cuh"
#include "tc.cuh"

namespace tvk {

constexpr int GP = 64;          // padded feature width (F <= 64)
constexpr int GROWS = 128;      // pairs per tile
constexpr int GT = 256;         // threads (8 warps of 32 rows x 4 column blocks)
constexpr int GS = GP + 4;      // smem row stride of U (doubles) and of the frame rows (elements)
constexpr int kSortChunk = 4096;
constexpr int64_t kGroupWindowFrames = 131072;  // 31 MB of f32 frames: the 20 gathers of a frame hit L2

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

__global__ void pair_hist_kernel(const int32_t* sel, const uint8_t* need, int64_t n_pairs, int C, int* hist) {
  extern __shared__ int lh[];
  for (int c = threadIdx.x; c < C; c += blockDim.x) lh[c] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortChunk;
  for (int i = threadIdx.x; i < kSortChunk; i += blockDim.x)
    if (base + i < n_pairs && (!need || need[base + i])) atomicAdd(&lh[sel[base + i]], 1);
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x)
    if (lh[c]) atomicAdd(&hist[c], lh[c]);
}

__global__ void hist_scan_kernel(int* hist, int C, int* start, int* cursor) {
  // single CTA exclusive scan of C counters
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

__global__ void pair_scatter_kernel(const int32_t* sel, const uint8_t* need, int64_t n_pairs, int C, int* cursor,
                                    int32_t* sorted) {
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
    comp[k] = (p < n_pairs && (!need || need[p])) ? sel[p] : -1;
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
                                           int kkmax, double (&acc)[2][8][2]) {
#pragma unroll
  for (int kk = 0; kk < GP / 4; kk++) {
    if (kk >= kkmax) break;  // k-steps past F: zero rows of U
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
  // pair indices of a tile, loaded one tile before the tile's rows are requested (the loads are in
  // flight during a tile's math instead of stalling the copy issue): pp = the pair of row tid (for
  // S.pair), pf = the pair of row warp + 8 lane (its frame is this lane's to fetch), -1 past the tile
  struct Pairs {
    int4 d;
    int pp, pf;
  };
  auto pairs_of = [&](int ti) {
    Pairs q{make_int4(0, 0, 0, 0), -1, -1};
    if (ti < te) {
      q.d = tiles[ti];
      const int myrow = warp + (GT / 32) * lane;
      if (tid < GROWS && tid < q.d.y) q.pp = sorted[q.d.x + tid];
      if (lane < GROWS / (GT / 32) && myrow < q.d.y) q.pf = sorted[q.d.x + myrow];
    }
    return q;
  };
  auto issue = [&](const Pairs& q, int b) {
    const int4 d = q.d;
    if (tid < GROWS) S.pair[b][tid] = q.pp;
    // frame rows: row r <- x[sorted / K], F elements; warp w copies rows w, w+8, ... (lanes over
    // 16-byte pieces), lane j holds the frame index of the warp's j-th row
    const int per_row = VEC ? (F * (int)sizeof(XT)) / 16 : F;
    // frame = pair / K by a 40-bit reciprocal (exact for pair < 2^31, K <= 32)
    const int myframe = q.pf >= 0 ? (int)(((uint64_t)(uint32_t)q.pf * kinv) >> 40) : 0;
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
  Pairs nxt = pairs_of(tb);
  issue(nxt, 0);
  int4 dcur = nxt.d;  // descriptor of tile ti (also loaded a tile ahead)
  nxt = pairs_of(tb + 1);
  for (int ti = tb; ti < te; ti++) {
    const int xb = (ti - tb) & 1;
    const int4 d = dcur;
    if (d.z != comp) {  // new component: stage U once every warp is done with the previous tile
      __syncthreads();
      stage_U(d.z);
      comp = d.z;
    }
    cp_async_wait<0>();
    __syncthreads();
    // prefetch the next tile's frame rows into the other buffer (its last readers passed the barrier)
    if (ti + 1 < te) issue(nxt, xb ^ 1);
    dcur = nxt.d;
    nxt = pairs_of(ti + 2);
    // warp w owns rows 16w..16w+15 of the tile: Z rows, q = rowsum(Z o Z), ll, store -- no more barriers
    if (warp * 16 < d.y) {
      double acc[2][8][2];
#pragma unroll
      for (int i = 0; i < 2; i++)
#pragma unroll
        for (int n = 0; n < 8; n++) acc[i][n][0] = acc[i][n][1] = 0.0;
      whiten_mma(S.X[xb], S.U, S.mu, warp, g, t4, (F + 3) / 4, acc);
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
  double* approx_ll;  // sparse path: 3xTF32 log-likelihood of every pair of the window
  float* approx_err;  // and its rigorous error bound
  uint8_t* need;      // pairs that need the exact FP64 value
  int2* state;        // per frame: (kept set known, kept mask)
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
  w.approx_ll = (double*)take(sizeof(double) * n_pairs);
  w.approx_err = (float*)take(sizeof(float) * n_pairs);
  w.need = (uint8_t*)take(n_pairs);
  w.state = (int2*)take(sizeof(int2) * n_pairs);  // >= frames of the window
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
  const int64_t one = (int64_t)group_carve(nullptr, std::min<int64_t>(n_pairs, kGroupWindowFrames * 32), C).bytes;
  return n_pairs > kGroupWindowFrames ? 2 * one : one;  // two windows in flight (see grouped_full_ll)
}

// Second stream of the window pipeline, one per device (fork/join events are per call, so concurrent
// host threads cannot cross their dependencies).
static cudaStream_t window_stream() {
  static cudaStream_t s2[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!s2[dev & 63]) cudaStreamCreateWithFlags(&s2[dev & 63], cudaStreamNonBlocking);
  return s2[dev & 63];
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

// the bucketing kernels' dynamic shared memory grows with C: allow the largest supported C once
// (lowering the limit to one call's C would break a later call with a larger C)
static void set_sort_smem_limits() {
  cudaFuncSetAttribute(pair_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(int) * 2 * kGroupedMaxC));
  cudaFuncSetAttribute(pair_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(int) * kGroupedMaxC));
}

// bucket the window's pairs (optionally only those with need[p]) by component into <=128-pair tiles
static int sort_tiles(const int32_t* wsel, const uint8_t* need, int64_t np, int C, const GroupWs& w,
                      cudaStream_t st) {
  cudaMemsetAsync(w.hist, 0, sizeof(int) * C, st);
  int nchunks = (int)((np + kSortChunk - 1) / kSortChunk);
  pair_hist_kernel<<<nchunks, GT, sizeof(int) * C, st>>>(wsel, need, np, C, w.hist);
  hist_scan_kernel<<<1, 1024, 0, st>>>(w.hist, C, w.start, w.cursor);
  pair_scatter_kernel<<<nchunks, GT, sizeof(int) * 2 * C, st>>>(wsel, need, np, C, w.cursor, w.sorted);
  tile_count_kernel<<<(C + 255) / 256, 256, 0, st>>>(w.hist, C, w.ntile);
  hist_scan_kernel<<<1, 1024, 0, st>>>(w.ntile, C, w.tile_start, w.cursor);
  tile_build_kernel<<<(C + 255) / 256, 256, 0, st>>>(w.hist, w.start, w.tile_start, C, w.tiles);
  TVK_CHECK_LAUNCH("pair sort");
  return TVK_OK;
}

template <typename XT>
int grouped_full_ll(const XT* x, int64_t T, int F, const double* ptab, int C, int K, const int32_t* sel,
                    double* sel_ll, void* ws_base, int64_t ws_bytes, cudaStream_t st) {
  TVK_REQUIRE(F <= kWideMaxF, "full log-likelihood supports F <= 128");
  TVK_REQUIRE(K >= 1 && K <= kWideMaxK, "full log-likelihood supports top_k <= 8192");
  TVK_REQUIRE(C <= kGroupedMaxC, "full log-likelihood supports C <= 24576");
  const int64_t n_pairs = T * K;
  TVK_REQUIRE(n_pairs < (1ll << 31) - 1, "too many (frame, component) pairs for one call");
  // frame windows sized so the window's frames and the whitening table stay L2-resident while the
  // window's pairs (sorted by component, i.e. random in frame order) gather their frame rows; a
  // window holds at most kGroupWindowFrames * 32 pairs (frame = pair / K stays exact, see kinv)
  const int64_t win = std::min<int64_t>(T, K <= 32 ? kGroupWindowFrames : std::max<int64_t>(1, kGroupWindowFrames * 32 / K));
  const int nwin = (int)((T + win - 1) / win);
  // windows alternate between the caller's stream and a second one, each with its own workspace set,
  // so one window's pair sort and kernel ramp overlap the previous window's whitening tail
  GroupWs w[2];
  w[0] = group_carve(ws_base, win * K, C);
  TVK_REQUIRE(ws_base != nullptr && (int64_t)w[0].bytes * (nwin > 1 ? 2 : 1) <= ws_bytes,
              "grouped full log-likelihood: workspace too small");
  if (nwin > 1) w[1] = group_carve((char*)ws_base + w[0].bytes, win * K, C);
  set_sort_smem_limits();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool vec = ((F * sizeof(XT)) % 16 == 0) && ((uintptr_t)x % 16 == 0);
  cudaStream_t s2 = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  if (nwin > 1) {
    s2 = window_stream();
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    cudaEventRecord(fork, st);
    cudaStreamWaitEvent(s2, fork, 0);
  }
  int rc = TVK_OK;
  for (int i = 0; i < nwin; i++) {
    const int64_t f0 = (int64_t)i * win;
    const int64_t nf = std::min<int64_t>(win, T - f0);
    const int64_t np = nf * K;
    const int32_t* wsel = sel + f0 * K;
    cudaStream_t s = (i & 1) ? s2 : st;
    const GroupWs& wi = w[i & 1];
    rc = sort_tiles(wsel, nullptr, np, C, wi, s);
    if (rc != TVK_OK) break;
    // the kernel reads the tile count from tile_start[C]
    GroupWs wc = wi;
    wc.tile_start = wi.tile_start + C;
    if (F > GP)  // wide features: FMA whitening of the same component tiles (align_wide.cu)
      rc = wide_whiten<XT>(x + f0 * F, F, ptab, K, wi.sorted, wi.tiles, wc.tile_start, np / GROWS + C + 1,
                           sel_ll + f0 * K, s);
    else
      rc = vec ? launch_whiten<XT, true>(x + f0 * F, F, ptab, K, wc, sel_ll + f0 * K, sms, s)
               : launch_whiten<XT, false>(x + f0 * F, F, ptab, K, wc, sel_ll + f0 * K, sms, s);
    if (rc != TVK_OK) break;
  }
  if (s2) {  // always join, also after an error
    cudaEventRecord(join, s2);
    cudaStreamWaitEvent(st, join, 0);
    cudaEventDestroy(fork);  // released once the recorded work completes
    cudaEventDestroy(join);
  }
  if (rc != TVK_OK) return rc;
  TVK_CHECK_LAUNCH("grouped windows");
  return TVK_OK;
}

// ============================================================================ sparse (approximate + exact)
// align_frames only needs FP64 log-likelihoods for the entries it keeps (weights exp(ll - lse_kept))
// and for frames whose prune decision is not certain.  whiten_approx_kernel evaluates every pair's
// Z = (x - mu) U with tcgen05 3xTF32 (A = rows in TMEM, B = U in shared memory) together with a
// rigorous bound |q~ - q| <= sum_j (2|z~_j| e_j + e_j^2), e_j = kappa_z ||y||_2 ||U_:,j||_2;
// decide_kernel proves the kept set (or flags the frame); the FP64 whitening kernel then runs on the
// flagged pairs only (~4.3 of 20 per frame on the config-2 data) and finalize_sparse writes weights.
constexpr int AT = 128;                      // threads of the approximate kernel: one pair row each
constexpr float KAPPA_Z = 1.0f / 262144.0f;  // 3xTF32 relative error bound

template <typename XT>
struct ApproxSmem {
  float B[2][GP * GP];  // U^T hi / lo words (N = 64 output dims x K = 64 features, K-major core matrices)
  double mu[GP];
  float cn[GP];         // ||U[:, j]||_2, rounded up
  double cst[2];        // const (16 bytes: keeps X 16-byte aligned for cp.async)
  XT X[2][GROWS * GS];  // frame rows (columns F..63 stay zero)
  int pair[2][GROWS];
  uint64_t mbar;
  uint32_t tbase;
};

template <typename XT, bool VEC>
__global__ void __launch_bounds__(AT)
    whiten_approx_kernel(const XT* __restrict__ x, int F, const double* __restrict__ tab, int K, uint64_t kinv,
                         const int32_t* __restrict__ sorted, const int4* __restrict__ tiles,
                         const int* __restrict__ ntile_p, double* __restrict__ approx_ll,
                         float* __restrict__ approx_err) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  ApproxSmem<XT>& S = *reinterpret_cast<ApproxSmem<XT>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntiles = *ntile_p;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int tb = blockIdx.x * per, te = min(tb + per, ntiles);
  if (tb >= te) return;
  for (int i = tid; i < 2 * GROWS * GS; i += AT) (&S.X[0][0])[i] = (XT)0;
  if (tid == 0) {
    tc::mbar_init(&S.mbar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<256>(&S.tbase);  // A hi [0,64) | A lo [64,128) | Z [128,192)
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tbase, lane_addr = tmem + ((uint32_t)(warp * 32) << 16);

  auto issue = [&](int ti, int b) {  // frame rows of tile ti into buffer b (cp.async), as whiten_ll
    const int4 d = tiles[ti];
    for (int r = tid; r < GROWS; r += AT) S.pair[b][r] = r < d.y ? sorted[d.x + r] : -1;
    const int per_row = VEC ? (F * (int)sizeof(XT)) / 16 : F;
    // lane j fetches the frame of the warp's j-th row (rows warp, warp+4, ...): one round of loads
    const int myrow = warp + (AT / 32) * lane;
    const int myframe = myrow < d.y ? (int)(((uint64_t)(uint32_t)sorted[d.x + myrow] * kinv) >> 40) : 0;
    if (VEC && per_row <= 16) {  // two rows per warp step: lanes 0-15 and 16-31
      const int sub = lane >> 4, c = lane & 15;
      for (int jr = 0; jr < GROWS / (AT / 32); jr += 2) {
        const int r = warp + (AT / 32) * (jr + sub);
        const int fr = __shfl_sync(0xffffffffu, myframe, jr + sub);
        if (warp + (AT / 32) * jr >= d.y) break;
        if (r < d.y && c < per_row)
          cp_async16(reinterpret_cast<uint8_t*>(&S.X[b][r * GS]) + 16 * c,
                     reinterpret_cast<const uint8_t*>(x + (int64_t)fr * F) + 16 * c, 16);
      }
      cp_async_commit();
      return;
    }
    for (int jr = 0; jr < GROWS / (AT / 32); jr++) {
      const int r = warp + (AT / 32) * jr;
      const int fr = __shfl_sync(0xffffffffu, myframe, jr);
      if (r >= d.y) break;
      const XT* src = x + (int64_t)fr * F;
      for (int c = lane; c < per_row; c += 32) {
        if (VEC) cp_async16(reinterpret_cast<uint8_t*>(&S.X[b][r * GS]) + 16 * c,
                            reinterpret_cast<const uint8_t*>(src) + 16 * c, 16);
        else cp_async_elem<(int)sizeof(XT)>(&S.X[b][r * GS + c], src + c);
      }
    }
    cp_async_commit();
  };

  int comp = -1;
  uint32_t phase = 0;
  issue(tb, 0);
  for (int ti = tb; ti < te; ti++) {
    const int xb = (ti - tb) & 1;
    const int4 d = tiles[ti];
    if (d.z != comp) {  // stage U^T as TF32 hi/lo, column norms, mu, const
      __syncthreads();
      const double* src = tab + (int64_t)d.z * kWhitenStride;
      for (int idx = tid; idx < GP * GP; idx += AT) {
        const int i = idx / GP, j = idx % GP;  // U[i][j] -> B[j][i]
        const float u = (float)src[idx];
        const float hi = tc::tf32_round(u), lo = tc::tf32_round(u - hi);
        const uint32_t o = tc::kmajor_offset(j, i, GP) / 4;
        S.B[0][o] = hi;
        S.B[1][o] = lo;
      }
      for (int j = warp; j < GP; j += AT / 32) {
        double c2 = 0.0;
        for (int i = lane; i < GP; i += 32) c2 += src[i * GP + j] * src[i * GP + j];
        c2 = warp_sum(c2);
        if (lane == 0) S.cn[j] = __double2float_ru(sqrt(c2)) * (1.0f + 1.0f / 1048576.0f);
      }
      for (int i = tid; i < GP; i += AT) S.mu[i] = src[GP * GP + i];
      if (tid == 0) S.cst[0] = src[GP * GP + GP];
      tc::fence_proxy_async();  // the tensor core reads B through the async proxy
      comp = d.z;
    }
    cp_async_wait<0>();
    __syncthreads();
    if (ti + 1 < te) issue(ti + 1, xb ^ 1);
    // A rows: y = x - mu (FP64 difference, then f32), TF32 hi/lo words into TMEM
    const int r = tid;
    double yn2 = 0.0;
    {
      float wh[32], wl[32];
#pragma unroll 1
      for (int j = 0; j < 2; j++) {
#pragma unroll
        for (int u = 0; u < 32; u++) {
          const int i = 32 * j + u;
          const float y = i < F ? (float)((double)S.X[xb][r * GS + i] - S.mu[i]) : 0.0f;
          yn2 += (double)y * y;
          wh[u] = tc::tf32_round(y);
          wl[u] = tc::tf32_round(y - wh[u]);
        }
        tc::tmem_st32(lane_addr + 32 * j, wh);
        tc::tmem_st32(lane_addr + 64 + 32 * j, wl);
      }
    }
    tc::tmem_st_wait();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
      const uint32_t idesc = tc::idesc_tf32(GROWS, GP);
      const uint32_t b0 = tc::smem_u32(S.B[0]), b1 = tc::smem_u32(S.B[1]);
      const int ks = (F + 7) / 8;
      for (int k = 0; k < ks; k++) {
        const uint64_t bh = tc::smem_desc(b0 + 256 * k, 128, 8 * GP * 4);
        const uint64_t bl = tc::smem_desc(b1 + 256 * k, 128, 8 * GP * 4);
        tc::mma_tf32_ts(tmem + 128, tmem + 8 * k, bh, idesc, k > 0);
        tc::mma_tf32_ts(tmem + 128, tmem + 8 * k, bl, idesc, 1);
        tc::mma_tf32_ts(tmem + 128, tmem + 64 + 8 * k, bh, idesc, 1);
      }
      tc::mma_commit(&S.mbar);
    }
    tc::mbar_wait(&S.mbar, phase);
    phase ^= 1u;
    tc::fence_after_sync();
    // q~ = sum z~^2 in f32 (its own rounding, <= 64 ulp of q~, joins the bound), bound in f32
    float q = 0.0f, dq = 0.0f;
    const float ky = KAPPA_Z * (float)sqrt(yn2) * 1.0001f;
#pragma unroll 1
    for (int j = 0; j < 2; j++) {
      float z[32];
      tc::tmem_ld32(lane_addr + 128 + 32 * j, z);
      tc::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 32; u++) {
        const float ej = ky * S.cn[32 * j + u];
        q = fmaf(z[u], z[u], q);
        dq = fmaf(fmaf(2.0f, fabsf(z[u]), ej), ej, dq);
      }
    }
    if (r < d.y) {
      const int p = S.pair[xb][r];
      approx_ll[p] = S.cst[0] - 0.5 * (double)q;
      approx_err[p] = (0.5f * dq + 4.0e-6f * q) * 1.001f + 1e-12f;
    }
    tc::fence_before_sync();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

// per frame: prove the kept set from the approximate values or ask for every exact value
__global__ void decide_kernel(int64_t nf, int K, double prune, const double* __restrict__ approx_ll,
                              const float* __restrict__ approx_err, uint8_t* __restrict__ need,
                              int2* __restrict__ state) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nf) return;
  const double* ll = approx_ll + t * K;
  const float* er = approx_err + t * K;
  bool ok = true;
  double mx = -INFINITY, D = 0.0;
  for (int j = 0; j < K; j++) {
    ok = ok && isfinite(ll[j]) && isfinite(er[j]);
    mx = fmax(mx, ll[j]);
    D = fmax(D, (double)er[j]);
  }
  unsigned kept = 0u;
  if (ok) {
    double s = 0.0;
    for (int j = 0; j < K; j++) s += exp(ll[j] - mx);
    const double lse = log(s) + mx;
    const double lp = log(prune);  // -inf for prune = 0: everything is kept
    const double tie = 1e-12;
    for (int j = 0; j < K && ok; j++) {
      const double lo = ll[j] - er[j] - (lse + D), hi = ll[j] + er[j] - (lse - D);
      if (lo >= lp + tie) kept |= 1u << j;
      else if (!(hi < lp - tie)) ok = false;
    }
    if (ok && kept == 0u) {  // degenerate: the arg-max (first in selection order) must be certain
      int best = 0;
      for (int j = 1; j < K; j++)
        if (ll[j] > ll[best]) best = j;
      for (int j = 0; j < K && ok; j++)
        if (j != best && !(ll[best] - er[best] > ll[j] + er[j])) ok = false;
      kept = 1u << best;
    }
  }
  const bool exact_kept = ok && __popc(kept) > 1;
  for (int j = 0; j < K; j++) need[t * K + j] = !ok || (exact_kept && ((kept >> j) & 1u));
  state[t] = make_int2(ok ? 1 : 0, (int)kept);
}

__global__ void finalize_sparse_kernel(int64_t nf, int K, double prune, const int32_t* sel, const double* sel_ll,
                                       const int2* state, int32_t* comp_pad, float* w_pad, int64_t* counts) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nf) return;
  double ll[kMaxTopK];
  int id[kMaxTopK], oc[kMaxTopK];
  float ow[kMaxTopK];
  const int2 s = state[t];
  for (int j = 0; j < K; j++) {
    id[j] = sel[t * K + j];
    ll[j] = (s.x == 0 || ((s.y >> j) & 1)) ? sel_ll[t * K + j] : 0.0;
  }
  const int n = s.x == 0 ? finalize_frame(K, prune, ll, id, oc, ow) : finalize_known(K, (unsigned)s.y, ll, id, oc, ow);
  for (int e = 0; e < n; e++) {
    comp_pad[t * K + e] = oc[e];
    w_pad[t * K + e] = ow[e];
  }
  counts[t] = n;
}

template <typename XT, bool VEC>
static int launch_approx(const XT* x, int F, const double* tab, int K, uint64_t kinv, const GroupWs& w,
                         const int* ntile, int sms, cudaStream_t st) {
  const size_t smem = sizeof(ApproxSmem<XT>);
  cudaFuncSetAttribute(whiten_approx_kernel<XT, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  whiten_approx_kernel<XT, VEC><<<2 * sms, AT, smem, st>>>(x, F, tab, K, kinv, w.sorted, w.tiles, ntile,
                                                            w.approx_ll, w.approx_err);
  TVK_CHECK_LAUNCH("whiten_approx");
  return TVK_OK;
}

// align_frames' stages 2-3 (gmm.py:412-438) for the grouped path: frames in L2-sized windows;
// per window the approximate LLs of all pairs, the kept-set proof, FP64 LLs for the pairs that need
// them and the per-frame CSR rows (comp_pad / w_pad / counts of the window's frames).
template <typename XT>
int grouped_align_sparse(const XT* x, int64_t T, int F, const double* ptab, int C, int K, double prune,
                         const int32_t* sel, double* sel_ll, int32_t* comp_pad, float* w_pad, int64_t* counts,
                         void* ws_base, int64_t ws_bytes, cudaStream_t st) {
  TVK_REQUIRE(F <= GP, "grouped full log-likelihood supports F <= 64");
  TVK_REQUIRE(K >= 1 && K <= 32, "grouped full log-likelihood supports K <= 32");
  TVK_REQUIRE(C <= 8192, "grouped full log-likelihood supports C <= 8192");
  TVK_REQUIRE(T * K < (1ll << 31) - 1, "too many (frame, component) pairs for one call");
  const int64_t win = std::min<int64_t>(T, kGroupWindowFrames);
  GroupWs w = group_carve(ws_base, win * K, C);
  TVK_REQUIRE(ws_base != nullptr && (int64_t)w.bytes <= ws_bytes, "grouped full log-likelihood: workspace too small");
  set_sort_smem_limits();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool vec = ((F * sizeof(XT)) % 16 == 0) && ((uintptr_t)x % 16 == 0);
  const uint64_t kinv = ((1ull << 40) + K - 1) / K;
  GroupWs wc = w;
  wc.tile_start = w.tile_start + C;  // the kernels read the tile count from tile_start[C]
  for (int64_t f0 = 0; f0 < T; f0 += win) {
    const int64_t nf = std::min<int64_t>(win, T - f0);
    const int64_t np = nf * K;
    const int32_t* wsel = sel + f0 * K;
    const XT* wx = x + f0 * F;
    TVK_TRY(sort_tiles(wsel, nullptr, np, C, w, st));
    if (vec) TVK_TRY((launch_approx<XT, true>(wx, F, ptab, K, kinv, w, wc.tile_start, sms, st)));
    else TVK_TRY((launch_approx<XT, false>(wx, F, ptab, K, kinv, w, wc.tile_start, sms, st)));
    decide_kernel<<<(int)((nf + 127) / 128), 128, 0, st>>>(nf, K, prune, w.approx_ll, w.approx_err, w.need, w.state);
    TVK_CHECK_LAUNCH("decide");
    TVK_TRY(sort_tiles(wsel, w.need, np, C, w, st));
    if (vec) TVK_TRY((launch_whiten<XT, true>(wx, F, ptab, K, wc, sel_ll + f0 * K, sms, st)));
    else TVK_TRY((launch_whiten<XT, false>(wx, F, ptab, K, wc, sel_ll + f0 * K, sms, st)));
    finalize_sparse_kernel<<<(int)((nf + 127) / 128), 128, 0, st>>>(nf, K, prune, wsel, sel_ll + f0 * K, w.state,
                                                                    comp_pad + f0 * K, w_pad + f0 * K, counts + f0);
    TVK_CHECK_LAUNCH("finalize_sparse");
  }
  return TVK_OK;
}
template int grouped_align_sparse<float>(const float*, int64_t, int, const double*, int, int, double, const int32_t*,
                                         double*, int32_t*, float*, int64_t*, void*, int64_t, cudaStream_t);
template int grouped_align_sparse<double>(const double*, int64_t, int, const double*, int, int, double,
                                          const int32_t*, double*, int32_t*, float*, int64_t*, void*, int64_t,
                                          cudaStream_t);

template int grouped_full_ll<float>(const float*, int64_t, int, const double*, int, int, const int32_t*, double*,
                                    void*, int64_t, cudaStream_t);
template int grouped_full_ll<double>(const double*, int64_t, int, const double*, int, int, const int32_t*,
                                     double*, void*, int64_t, cudaStream_t);

}  // namespace tvk

extern "C" int tvk_precision_table(const double* weights, const double* means, const double* covariances, int C,
                                   int F, double* table, int32_t* status, void* stream) {
  TVK_REQUIRE(C >= 1 && F >= 1 && F <= tvk::kWideMaxF, "precision_table: need 1 <= F <= 128");
  if (F > tvk::GP) return tvk::wide_precision_table(weights, means, covariances, C, F, table, status, (cudaStream_t)stream);
  size_t smem = 2 * sizeof(double) * F * F;
  cudaFuncSetAttribute(tvk::whiten_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * sizeof(double) * tvk::GP * tvk::GP));
  tvk::whiten_table_kernel<<<C, 256, smem, (cudaStream_t)stream>>>(weights, means, covariances, C, F, table, status);
  TVK_CHECK_LAUNCH("precision_table");
  return TVK_OK;
}

extern "C" int64_t tvk_precision_table_stride(int F) { return tvk::precision_stride(F); }
