// Alignment outside the fast path's shape envelope (gmm.py:376-439 for any top_k <= 8192, F <= 128).
//
// The fast path (select_tc.cu, align_grouped.cu, align.cu) is specialised for the shapes the
// reference is run at -- top_k <= 32, F <= 64 -- and the reference accepts any top_k <= C and any F.
// These kernels keep every other shape on the device with the same semantics:
//
//   wide_select_kernel   one CTA per frame: all C diagonal-model scores in FP64 (coalesced columns of
//                        the (2F+1) x C table), a running top-K kept by bitonic sorts of
//                        [current K | next chunk] on (value desc, index asc) -- numpy's stable argsort
//                        order (gmm.py:409), NaN last;
//   wide_whiten_kernel   F in (64, 128]: the grouped path's component tiles (pairs bucketed by the
//                        selected component, align_grouped.cu) with L_c^-1 (column-packed) staged in
//                        shared memory once per tile; one warp per pair, lane i forms
//                        z_i = sum_{m<=i} (L^-1)_im (x - mu)_m, ll = const_c - ||z||^2 / 2 (gmm.py:111-118);
//   finalize_wide_kernel top_k > 32: one CTA per frame: logsumexp over the selection, prune, the
//                        degenerate rule, renormalisation, kept entries sorted by component
//                        (gmm.py:414-439), fixed-order block reductions;
//   wide_table_kernel    the F > 64 precision table: Cholesky in shared memory, column-packed L^-1,
//                        log w - (F log 2pi + log|Sigma|)/2.
#include <math.h>

#include "common.cuh"
#include "internal.h"
#include "spd_small.cuh"

namespace tvk {

constexpr int WT = 256;  // threads of the per-frame kernels

__device__ __forceinline__ bool wide_better(double v, int i, double w, int j) {  // (v, i) ranks before (w, j)
  const bool a = isnan(v), b = isnan(w);
  if (a != b) return b;
  if (a) return i < j;
  return v > w || (v == w && i < j);
}

// Bitonic sort of n (power of two) (key, index) pairs in shared memory into wide_better order.
__device__ __forceinline__ void bitonic_rank_sort(double* key, int* idx, int n) {
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int l = i ^ j;
        if (l <= i) continue;
        const double a = key[i], b = key[l];
        const int ia = idx[i], ib = idx[l];
        const bool up = (i & k) == 0;
        if (up ? wide_better(b, ib, a, ia) : wide_better(a, ia, b, ib)) {
          key[i] = b;
          key[l] = a;
          idx[i] = ib;
          idx[l] = ia;
        }
      }
      __syncthreads();
    }
}

int wide_select_span(int K) {  // sort buffer: the top K plus a chunk of >= 256 new components
  int s = 512;
  while (s < K + 256) s <<= 1;
  return s;
}

template <typename XT>
__global__ void __launch_bounds__(WT) wide_select_kernel(const XT* __restrict__ x, int64_t T, int F,
                                                         const double* __restrict__ tab, int C, int K, int S,
                                                         int32_t* __restrict__ sel, double* __restrict__ val) {
  extern __shared__ __align__(16) double sm[];
  double* key = sm;                               // [S]
  int* idx = reinterpret_cast<int*>(key + S);     // [S]
  double* xs = reinterpret_cast<double*>(idx + S);  // [F]
  const int CH = S - K;
  const double* ca = tab;                  // rows 0..F-1: coefficient of x^2
  const double* cb = tab + (int64_t)F * C;  // rows F..2F-1: coefficient of x
  const double* cc = tab + (int64_t)2 * F * C;
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    for (int f = threadIdx.x; f < F; f += WT) xs[f] = (double)x[t * F + f];
    for (int i = threadIdx.x; i < K; i += WT) {
      key[i] = NAN;
      idx[i] = 0x7fffffff;
    }
    __syncthreads();
    for (int c0 = 0; c0 < C; c0 += CH) {
      for (int e = threadIdx.x; e < CH; e += WT) {
        const int c = c0 + e;
        double s = NAN;
        int id = 0x7fffffff;
        if (c < C) {
          s = cc[c];
          for (int f = 0; f < F; f++) s = fma(xs[f], fma(ca[(int64_t)f * C + c], xs[f], cb[(int64_t)f * C + c]), s);
          id = c;
        }
        key[K + e] = s;
        idx[K + e] = id;
      }
      __syncthreads();
      bitonic_rank_sort(key, idx, S);
    }
    for (int i = threadIdx.x; i < K; i += WT) {
      sel[t * K + i] = idx[i];
      if (val) val[t * K + i] = key[i];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------- finalize (top_k > 32)

template <typename T, class Op>
__device__ __forceinline__ T block_reduce(T v, T* red, Op op) {  // fixed-order tree, result in every thread
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  T r = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); w++) r = op(r, red[w]);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(WT) finalize_wide_kernel(int64_t T, int K, int K2, double prune,
                                                           const int32_t* sel, const double* sel_ll,
                                                           int32_t* comp_pad, float* w_pad, int64_t* counts) {
  extern __shared__ __align__(16) double fsm[];
  int* kc = reinterpret_cast<int*>(fsm);       // [K2] kept components (sort keys), K2 = pow2 >= K
  float* kw = reinterpret_cast<float*>(kc + K2);  // [K2] their weights
  __shared__ double redd[WT / 32];
  __shared__ long long redl[WT / 32];
  __shared__ int base[WT];
  const int tid = threadIdx.x;
  const double ninf = -INFINITY;
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const double* ll = sel_ll + t * K;
    double mx = ninf;
    for (int j = tid; j < K; j += WT) mx = fmax(mx, ll[j]);
    mx = block_reduce(mx, redd, [](double a, double b) { return fmax(a, b); });
    if (!isfinite(mx)) mx = 0.0;  // scipy logsumexp convention
    double s = 0.0;
    for (int j = tid; j < K; j += WT) s += exp(ll[j] - mx);
    s = block_reduce(s, redd, [](double a, double b) { return a + b; });
    const double lse = log(s) + mx;
    // kept count and the first maximal posterior (packed as (post bits, -j) is not order-safe for
    // NaN: compare explicitly)
    long long nkeep = 0;
    double bp = -1.0;
    int bj = 0x7fffffff;
    for (int j = tid; j < K; j += WT) {
      const double p = exp(ll[j] - lse);
      if (p >= prune) nkeep++;
      if (p > bp || (p == bp && j < bj)) {
        bp = p;
        bj = j;
      }
    }
    nkeep = block_reduce(nkeep, redl, [](long long a, long long b) { return a + b; });
    {  // arg-max with the lowest index on ties
      long long key2 = bj;
      double v = bp;
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const long long k2 = __shfl_xor_sync(0xffffffffu, key2, o);
        if (v2 > v || (v2 == v && k2 < key2)) {
          v = v2;
          key2 = k2;
        }
      }
      if ((tid & 31) == 0) {
        redd[tid >> 5] = v;
        redl[tid >> 5] = key2;
      }
      __syncthreads();
      v = redd[0];
      key2 = redl[0];
      for (int w = 1; w < WT / 32; w++)
        if (redd[w] > v || (redd[w] == v && redl[w] < key2)) {
          v = redd[w];
          key2 = redl[w];
        }
      __syncthreads();
      bj = (int)key2;
    }
    const bool degenerate = nkeep == 0;
    double tot = 0.0;
    for (int j = tid; j < K; j += WT) {
      const double p = exp(ll[j] - lse);
      const bool keep = degenerate ? (j == bj) : (p >= prune);
      if (keep) tot += p;
    }
    tot = block_reduce(tot, redd, [](double a, double b) { return a + b; });
    // compact the kept entries (thread-contiguous ranges keep the selection order), then sort them
    // by component
    const int per = (K + WT - 1) / WT, j0 = tid * per, j1 = min(K, j0 + per);
    int mine = 0;
    for (int j = j0; j < j1; j++) {
      const double p = exp(ll[j] - lse);
      mine += degenerate ? (j == bj) : (p >= prune);
    }
    base[tid] = mine;
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int i = 0; i < WT; i++) {
        const int v = base[i];
        base[i] = run;
        run += v;
      }
    }
    __syncthreads();
    const int n = degenerate ? 1 : (int)nkeep;
    int pos = base[tid];
    for (int j = j0; j < j1; j++) {
      const double p = exp(ll[j] - lse);
      if (degenerate ? (j == bj) : (p >= prune)) {
        kc[pos] = sel[t * K + j];
        kw[pos] = (float)(p / tot);
        pos++;
      }
    }
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int i = n + tid; i < n2; i += WT) kc[i] = 0x7fffffff;
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < n2; i += WT) {
          const int l = i ^ j;
          if (l <= i) continue;
          const int a = kc[i], b = kc[l];
          if (((i & k) == 0) ? (b < a) : (a < b)) {
            kc[i] = b;
            kc[l] = a;
            const float wa = kw[i];
            kw[i] = kw[l];
            kw[l] = wa;
          }
        }
        __syncthreads();
      }
    for (int e = tid; e < n; e += WT) {
      comp_pad[t * K + e] = kc[e];
      w_pad[t * K + e] = kw[e];
    }
    if (tid == 0) counts[t] = n;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------- F > 64 precision table

__host__ __device__ inline int64_t colpack(int i, int m, int F) {  // (i >= m), column m contiguous
  return (int64_t)m * F - (int64_t)m * (m - 1) / 2 + (i - m);
}

__global__ void wide_table_kernel(const double* w, const double* mu, const double* cov, int C, int F, double* tab,
                                  int32_t* status) {
  extern __shared__ double a[];  // [F][F]
  __shared__ int bad;
  __shared__ double logdet;
  const int c = blockIdx.x;
  const int64_t P = (int64_t)F * (F + 1) / 2, stride = precision_stride(F);
  double* dst = tab + (int64_t)c * stride;
  for (int i = threadIdx.x; i < F * F; i += blockDim.x) a[i] = cov[(int64_t)c * F * F + i];
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
  // Y = L^-1, thread j forms column j by forward substitution straight into the table
  for (int j = threadIdx.x; j < F; j += blockDim.x) {
    dst[colpack(j, j, F)] = 1.0 / a[j * F + j];
    for (int i = j + 1; i < F; i++) {
      double s = 0.0;
      for (int k = j; k < i; k++) s += a[i * F + k] * dst[colpack(k, j, F)];
      dst[colpack(i, j, F)] = -s / a[i * F + i];
    }
  }
  for (int i = threadIdx.x; i < F; i += blockDim.x) dst[P + i] = mu[(int64_t)c * F + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    dst[P + F] = log(w[c]) - 0.5 * (F * kLog2Pi + logdet);
    dst[P + F + 1] = 0.0;
    status[c] = TVK_ITEM_OK;
  }
}

// ---------------------------------------------------------------------------- F > 64 whitening

template <typename XT>
__global__ void __launch_bounds__(WT) wide_whiten_kernel(const XT* __restrict__ x, int F, const double* __restrict__ tab,
                                                         int K, const int32_t* __restrict__ sorted,
                                                         const int4* __restrict__ tiles,
                                                         const int* __restrict__ ntile_p, double* __restrict__ sel_ll) {
  extern __shared__ __align__(16) double wsm[];
  const int64_t P = (int64_t)F * (F + 1) / 2, stride = precision_stride(F);
  double* Y = wsm;              // [P] column-packed L^-1
  double* mu = Y + P;           // [F]
  double* d = mu + F;           // [WT/32][F] per-warp x - mu
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ntiles = *ntile_p;
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const int4 tl = tiles[ti];
    const double* src = tab + (int64_t)tl.z * stride;
    for (int64_t i = threadIdx.x; i < P + F; i += WT) Y[i] = src[i];
    const double cst = src[P + F];
    __syncthreads();
    double* dw = d + warp * F;
    for (int r = warp; r < tl.y; r += WT / 32) {
      const int p = sorted[tl.x + r];
      const int64_t t = p / K;
      for (int f = lane; f < F; f += 32) dw[f] = (double)x[t * F + f] - mu[f];
      __syncwarp();
      double q = 0.0;
      for (int i = lane; i < F; i += 32) {
        double z = 0.0;
        for (int m = 0; m <= i; m++) z = fma(Y[colpack(i, m, F)], dw[m], z);
        q = fma(z, z, q);
      }
      q = warp_sum(q);
      if (lane == 0) sel_ll[p] = cst - 0.5 * q;
      __syncwarp();
    }
    __syncthreads();
  }
}

template <typename XT>
int wide_whiten(const XT* x, int F, const double* ptab, int K, const int32_t* sorted, const int4* tiles,
                const int* ntile_dev, int64_t max_tiles, double* sel_ll, cudaStream_t st) {
  const size_t smem = sizeof(double) * ((size_t)F * (F + 1) / 2 + F + (WT / 32) * (size_t)F);
  TVK_REQUIRE(smem <= 227 * 1024, "align_frames: F too large for the wide whitening tile");
  cudaFuncSetAttribute(wide_whiten_kernel<XT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(max_tiles, 4 * (int64_t)sms));
  wide_whiten_kernel<XT><<<grid, WT, smem, st>>>(x, F, ptab, K, sorted, tiles, ntile_dev, sel_ll);
  TVK_CHECK_LAUNCH("wide_whiten");
  return TVK_OK;
}
template int wide_whiten<float>(const float*, int, const double*, int, const int32_t*, const int4*, const int*,
                                int64_t, double*, cudaStream_t);
template int wide_whiten<double>(const double*, int, const double*, int, const int32_t*, const int4*, const int*,
                                 int64_t, double*, cudaStream_t);

// ---------------------------------------------------------------------------- host launchers

static int grid_for(int64_t items, int per_sm) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)per_sm * sms));
}

template <typename XT>
int wide_select(const XT* x, int64_t T, int F, const double* tab, int C, int K, int32_t* sel, double* val,
                cudaStream_t st) {
  TVK_REQUIRE(K >= 1 && K <= kWideMaxK && K <= C, "select: top_k must be in [1, min(C, 8192)]");
  if (T == 0) return TVK_OK;
  const int S = wide_select_span(K);
  const size_t smem = (sizeof(double) + sizeof(int)) * (size_t)S + sizeof(double) * F;
  cudaFuncSetAttribute(wide_select_kernel<XT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  wide_select_kernel<XT><<<grid_for(T, 8), WT, smem, st>>>(x, T, F, tab, C, K, S, sel, val);
  TVK_CHECK_LAUNCH("wide_select");
  return TVK_OK;
}
template int wide_select<float>(const float*, int64_t, int, const double*, int, int, int32_t*, double*, cudaStream_t);
template int wide_select<double>(const double*, int64_t, int, const double*, int, int, int32_t*, double*,
                                 cudaStream_t);

int finalize_wide(int64_t T, int K, double prune, const int32_t* sel, const double* sel_ll, int32_t* comp_pad,
                  float* w_pad, int64_t* counts, cudaStream_t st) {
  if (T == 0) return TVK_OK;
  int K2 = 1;
  while (K2 < K) K2 <<= 1;
  const size_t smem = (sizeof(int) + sizeof(float)) * (size_t)K2;
  cudaFuncSetAttribute(finalize_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  finalize_wide_kernel<<<grid_for(T, 8), WT, smem, st>>>(T, K, K2, prune, sel, sel_ll, comp_pad, w_pad, counts);
  TVK_CHECK_LAUNCH("finalize_wide");
  return TVK_OK;
}

int wide_precision_table(const double* w, const double* mu, const double* cov, int C, int F, double* tab,
                         int32_t* status, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)F * F;
  TVK_REQUIRE(smem <= 227 * 1024, "precision_table: F too large");
  cudaFuncSetAttribute(wide_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  wide_table_kernel<<<C, 128, smem, st>>>(w, mu, cov, C, F, tab, status);
  TVK_CHECK_LAUNCH("wide precision_table");
  return TVK_OK;
}

}  // namespace tvk
