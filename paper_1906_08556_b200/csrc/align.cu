// Frame posteriors (gmm.py:389-439) as three FP64 tensor-pipe stages plus a CSR build:
//   1. select_topk_kernel: diag log-likelihoods [x^2, x, 1] . Wdiag (DMMA) for 64 frames x
//      all components, streamed in 64-component blocks, merged into a per-frame stable top-K
//      (lower index wins ties, gmm.py:410);
//   2. full_ll_kernel: quadratic-feature GEMM phi(x) . Wq (K = 1+F+F(F+1)/2) for 128 frames x
//      128 components; the epilogue keeps only the K preselected components of each frame
//      (gmm.py:412-413) so the T x C log-likelihood matrix never reaches HBM;
//   3. finalize_kernel: softmax over the selection (scipy logsumexp), prune (post >= prune),
//      degenerate rule (argmax in selection order), renormalize, sort by component (gmm.py:414-438);
//   4. exclusive scan of the per-frame counts and a compaction into the CSR arrays.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "gemm_f64.cuh"
#include "internal.h"
#include "spd_small.cuh"
#include "finalize.cuh"

namespace tvk {


// ----------------------------------------------------------------------------- tables

__global__ void diag_table_kernel(const double* w, const double* mu, const double* var, int C, int F, double* tab) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double logvar = 0.0, m2 = 0.0;
  for (int f = 0; f < F; f++) {
    double p = 1.0 / var[(int64_t)c * F + f];
    double m = mu[(int64_t)c * F + f];
    tab[(int64_t)f * C + c] = -0.5 * p;
    tab[(int64_t)(F + f) * C + c] = m * p;
    logvar += log(var[(int64_t)c * F + f]);
    m2 += m * m * p;
  }
  tab[(int64_t)(2 * F) * C + c] = log(w[c]) - 0.5 * (F * kLog2Pi + logvar) - 0.5 * m2;
}

// One CTA per component: Cholesky, precision P = Sigma^-1, log|Sigma|, then the column
// [k_c, P mu, -P_ii/2 | -P_ij (i<j)] of the quadratic-feature table.
__global__ void full_table_kernel(const double* w, const double* mu, const double* cov, int C, int F, double* tab,
                                  int32_t* status) {
  extern __shared__ double sm[];
  double* a = sm;
  double* y = sm + F * F;
  double* pm = y + F * F;  // P mu
  __shared__ int bad;
  __shared__ double red[2];
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
    if (threadIdx.x == 0) red[0] = 2.0 * s;
  }
  __syncthreads();
  block_spd_inverse(a, y, F);
  const double* m = mu + (int64_t)c * F;
  for (int i = threadIdx.x; i < F; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < F; j++) s += a[i * F + j] * m[j];
    pm[i] = s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < F; i += 32) s += m[i] * pm[i];
    s = warp_sum(s);
    if (threadIdx.x == 0) red[1] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tab[c] = log(w[c]) - 0.5 * (F * kLog2Pi + red[0]) - 0.5 * red[1];
    status[c] = TVK_ITEM_OK;
  }
  for (int i = threadIdx.x; i < F; i += blockDim.x) tab[(int64_t)(1 + i) * C + c] = pm[i];
  // quadratic rows, pair order (i, j>=i) row-major
  int npair = F * (F + 1) / 2;
  for (int p = threadIdx.x; p < npair; p += blockDim.x) {
    // invert p = i*F - i*(i-1)/2 + (j - i)
    int i = 0, base = 0;
    while (base + (F - i) <= p) {
      base += F - i;
      i++;
    }
    int j = i + (p - base);
    double v = (i == j) ? -0.5 * a[i * F + i] : -a[i * F + j];
    tab[(int64_t)(1 + F + p) * C + c] = v;
  }
}

// ----------------------------------------------------------------------------- stage 1: top-K

namespace sel {
// Warp-specialized: warps 0-3 run the DMMA GEMM (64 frames x 64 components per block, K streamed
// through a 3-stage cp.async ring of 16-deep table chunks), warps 4-7 merge the finished block into
// the per-frame top-K lists.  Two LL tile buffers let the merge of block n overlap the MMA of
// block n+1 (named barriers FULL/EMPTY per buffer).
constexpr int BM = 64, BN = 64, BK = 64, NSTAGE = 2;  // long chunks: few barriers per DMMA
constexpr int NMMA = 256, NMERGE = 384, NT = NMMA + NMERGE;  // 2 MMA warps per SMSP
constexpr int BS = BN + 4;  // == 4 (mod 16): conflict-free B fragments
constexpr int LS = BN + 1;
using Cfg = GemmCfg<BM, BN, BK, 2, 2, NSTAGE>;  // 4 MMA warps of 32x32
__host__ __device__ inline int kpad(int F) { return ((2 * F + 1) + BK - 1) / BK * BK; }
__host__ __device__ inline int astride(int F) { int kp = kpad(F); return kp + ((4 - kp % 16) + 16) % 16; }
__host__ inline size_t smem_bytes(int F, int K) {
  return sizeof(double) * ((size_t)BM * astride(F) + NSTAGE * BK * BS + 2 * BM * LS + (size_t)BM * K) +
         sizeof(int) * ((size_t)BM * K + BM);
}
}  // namespace sel

__device__ __forceinline__ bool ranks_before(double v, int i, double w, int j) {  // (v,i) strictly better
  return v > w || (v == w && i < j);
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n));
}

template <typename XT>
__global__ void __launch_bounds__(sel::NT, 1) select_topk_kernel(const XT* x, int64_t T, int F, const double* tab,
                                                                 int C, int K, int32_t* sel_out, double* sel_val) {
  using namespace sel;
  extern __shared__ __align__(16) double smem[];
  const int KD = 2 * F + 1;
  const int KP = kpad(F), AS = astride(F);
  double* sA = smem;                          // [BM][AS]
  double* sB = sA + BM * AS;                  // [NSTAGE][BK][BS]
  double* sL = sB + NSTAGE * BK * BS;         // [2][BM][LS]
  double* lv = sL + 2 * BM * LS;              // [BM][K]
  int* li = reinterpret_cast<int*>(lv + BM * K);  // [BM][K]
  int* lc = li + BM * K;                      // [BM]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * BM;
  const int nblocks = (C + BN - 1) / BN, nk = KP / BK;

  for (int idx = tid; idx < BM * KP; idx += NT) {  // features [x^2, x, 1, 0-pad]
    int r = idx / KP, k = idx % KP;
    double v = 0.0;
    if (t0 + r < T) {
      if (k < F) {
        double xv = (double)x[(t0 + r) * F + k];
        v = xv * xv;
      } else if (k < 2 * F) {
        v = (double)x[(t0 + r) * F + (k - F)];
      } else if (k == KD - 1) {
        v = 1.0;
      }
    }
    sA[r * AS + k] = v;
  }
  for (int r = tid; r < BM; r += NT) lc[r] = 0;
  __syncthreads();

  if (warp < NMMA / 32) {
    // ------------------------------------------------------------ MMA warps
    const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps of 32 x 16
    const int g = lane >> 2, t = lane & 3;
    const int total = nblocks * nk;
    auto load = [&](int chunk) {
      int blk = chunk / nk, kc = chunk % nk;
      double* dst = sB + (chunk % NSTAGE) * BK * BS;
      for (int idx = tid; idx < BK * BN; idx += NMMA) {
        int k = idx / BN, c = idx % BN;
        int gk = kc * BK + k, gc = blk * BN + c;
        bool ok = gk < KD && gc < C;
        cp_async8(&dst[k * BS + c], ok ? tab + (int64_t)gk * C + gc : tab, ok);
      }
    };
    for (int s = 0; s < NSTAGE - 1; s++) {
      if (s < total) load(s);
      cp_async_commit();
    }
    int chunk = 0;
    for (int blk = 0; blk < nblocks; blk++) {
      double acc[4][2][2];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int kc = 0; kc < nk; kc++, chunk++) {
        cp_async_wait<NSTAGE - 2>();
        named_sync(1, NMMA);
        if (chunk + NSTAGE - 1 < total) load(chunk + NSTAGE - 1);
        cp_async_commit();
        const double* b_s = sB + (chunk % NSTAGE) * BK * BS;
        const double* a_s = sA + kc * BK;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
          double a[4], b[2];
#pragma unroll
          for (int i = 0; i < 4; i++) a[i] = a_s[(wm * 32 + i * 8 + g) * AS + kk + t];
#pragma unroll
          for (int j = 0; j < 2; j++) b[j] = b_s[(kk + t) * BS + wn * 16 + j * 8 + g];
#pragma unroll
          for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 2; j++) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
      }
      const int buf = blk & 1;
      if (blk >= 2) named_sync(4 + buf, NT);  // wait until the merge warps released this buffer
      double* L = sL + buf * BM * LS;
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) {
          int r = wm * 32 + i * 8 + g, c = wn * 16 + j * 8 + 2 * t;
          L[r * LS + c] = acc[i][j][0];
          L[r * LS + c + 1] = acc[i][j][1];
        }
      __threadfence_block();
      named_arrive(2 + buf, NT);  // FULL[buf]
    }
    cp_async_wait<0>();
  } else {
    // ------------------------------------------------------------ merge warps
    const int mw = warp - NMMA / 32;
    for (int blk = 0; blk < nblocks; blk++) {
      const int buf = blk & 1;
      named_sync(2 + buf, NT);  // FULL[buf]
      const double* L = sL + buf * BM * LS;
      const int n0 = blk * BN, nb = min(BN, C - n0);
      for (int r = mw; r < BM; r += NMERGE / 32) {
        if (t0 + r >= T) continue;
        int cnt = lc[r];
        double myv = (lane < cnt) ? lv[r * K + lane] : -INFINITY;
        int myi = (lane < cnt) ? li[r * K + lane] : 0x7fffffff;
        for (int base = 0; base < nb; base += 32) {
          int ci = base + lane;
          double cv = ci < nb ? L[r * LS + ci] : -INFINITY;
          int gi = n0 + ci;
          double wv = __shfl_sync(0xffffffffu, myv, K - 1);
          int wi = __shfl_sync(0xffffffffu, myi, K - 1);
          bool cand = ci < nb && (cnt < K || ranks_before(cv, gi, wv, wi));
          unsigned mask = __ballot_sync(0xffffffffu, cand);
          while (mask) {
            int src = __ffs(mask) - 1;
            mask &= mask - 1;
            double v = __shfl_sync(0xffffffffu, cv, src);
            int vi = __shfl_sync(0xffffffffu, gi, src);
            wv = __shfl_sync(0xffffffffu, myv, K - 1);
            wi = __shfl_sync(0xffffffffu, myi, K - 1);
            if (cnt == K && !ranks_before(v, vi, wv, wi)) continue;
            unsigned better = __ballot_sync(0xffffffffu, lane < cnt && ranks_before(myv, myi, v, vi));
            int pos = __popc(better);
            double upv = __shfl_up_sync(0xffffffffu, myv, 1);
            int upi = __shfl_up_sync(0xffffffffu, myi, 1);
            if (lane > pos) {
              myv = upv;
              myi = upi;
            } else if (lane == pos) {
              myv = v;
              myi = vi;
            }
            cnt = min(cnt + 1, K);
          }
        }
        if (lane < K) {
          lv[r * K + lane] = myv;
          li[r * K + lane] = myi;
        }
        if (lane == 0) lc[r] = cnt;
      }
      if (blk + 2 < nblocks) named_arrive(4 + buf, NT);  // EMPTY[buf]
    }
  }
  __syncthreads();
  for (int idx = tid; idx < BM * K; idx += NT) {
    int r = idx / K, j = idx % K;
    if (t0 + r < T) {
      sel_out[(t0 + r) * K + j] = li[r * K + j];
      if (sel_val) sel_val[(t0 + r) * K + j] = lv[r * K + j];
    }
  }
}

// ----------------------------------------------------------------------------- stage 2: full LL

namespace fll {
using Cfg = GemmCfg<128, 128, 32, 2, 4, 2>;
}

// A operand: phi_k(x) = xe[i_k] * xe[j_k] with xe = [x, 1]; pairs (F,F) -> 1, (i,F) -> x_i.
template <typename XT>
__global__ void __launch_bounds__(fll::Cfg::NT) full_ll_kernel(const XT* x, int64_t T, int F, const double* tab,
                                                               int C, int K, const int32_t* sel, double* sel_ll) {
  using Cfg = fll::Cfg;
  using L = SmemLayout<Cfg::BM, Cfg::BN, Cfg::BK, false, false>;
  extern __shared__ __align__(16) double smem[];
  const int Q = 1 + F + F * (F + 1) / 2;
  double* stages = smem;
  XT* xs = reinterpret_cast<XT*>(stages + Cfg::STAGES * L::STAGE);  // [BM][F+1]
  int* pairs = reinterpret_cast<int*>(xs + Cfg::BM * (F + 1));          // [Qpad] packed (i<<16)|j
  const int Qpad = (Q + Cfg::BK - 1) / Cfg::BK * Cfg::BK;
  unsigned char* slot = reinterpret_cast<unsigned char*>(pairs + Qpad);  // [BM][BN] selection slot or 255

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  const int64_t m0 = (int64_t)(blockIdx.x % ((T + Cfg::BM - 1) / Cfg::BM)) * Cfg::BM;
  const int n0 = (int)(blockIdx.x / ((T + Cfg::BM - 1) / Cfg::BM)) * Cfg::BN;
  const int FE = F + 1;

  for (int idx = tid; idx < Cfg::BM * FE; idx += Cfg::NT) {
    int r = idx / FE, f = idx % FE;
    XT v = XT(0);
    if (m0 + r < T) v = (f < F) ? x[(m0 + r) * F + f] : XT(1);
    xs[idx] = v;
  }
  for (int k = tid; k < Qpad; k += Cfg::NT) {
    int i, j;
    if (k == 0 || k >= Q) {
      i = F;
      j = F;
    } else if (k <= F) {
      i = k - 1;
      j = F;
    } else {
      int p = k - 1 - F, base = 0;
      i = 0;
      while (base + (F - i) <= p) {
        base += F - i;
        i++;
      }
      j = i + (p - base);
    }
    pairs[k] = (i << 16) | j;
  }
  for (int idx = tid; idx < Cfg::BM * Cfg::BN; idx += Cfg::NT) slot[idx] = 255;
  __syncthreads();
  for (int idx = tid; idx < Cfg::BM * K; idx += Cfg::NT) {
    int r = idx / K, j = idx % K;
    if (m0 + r >= T) continue;
    int c = sel[(m0 + r) * K + j] - n0;
    if (c >= 0 && c < Cfg::BN) slot[r * Cfg::BN + c] = (unsigned char)j;
  }

  const int nk = Qpad / Cfg::BK;
  auto load_stage = [&](int stage, int kt) {
    double* sA = stages + stage * L::STAGE;
    double* sB = sA + L::A_ELEMS;
    int k0 = kt * Cfg::BK;
    load_tile_async<Cfg::BK, Cfg::BN, Cfg::BN + 4, Cfg::NT, false>(sB, tab, C, k0, n0, Q, C, tid);
    for (int idx = tid; idx < Cfg::BM * Cfg::BK; idx += Cfg::NT) {
      int r = idx / Cfg::BK, kk = idx % Cfg::BK;
      int pr = pairs[k0 + kk];
      const XT* xr = xs + r * FE;
      sA[L::a_off(r, kk)] = (double)xr[pr >> 16] * (double)xr[pr & 0xffff];
    }
  };

  Acc<Cfg> acc;
  acc.zero();
#pragma unroll
  for (int s = 0; s < Cfg::STAGES - 1; s++) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<Cfg::STAGES - 2>();
    __syncthreads();
    int nxt = kt + Cfg::STAGES - 1;
    if (nxt < nk) load_stage(nxt % Cfg::STAGES, nxt);
    cp_async_commit();
    const double* sA = stages + (kt % Cfg::STAGES) * L::STAGE;
    mma_stage<Cfg, L>(acc, sA, sA + L::A_ELEMS, wm, wn, lane);
  }
  cp_async_wait<0>();
  for_each_acc<Cfg>(acc, wm, wn, lane, [&](int r, int c, double v) {
    int j = slot[r * Cfg::BN + c];
    if (j != 255) sel_ll[(m0 + r) * K + j] = v;
  });
}

// ----------------------------------------------------------------------------- stage 3: finalize

__global__ void finalize_kernel(int64_t T, int K, double prune, const int32_t* sel, const double* sel_ll,
                                int32_t* comp_pad, float* w_pad, int64_t* counts) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  double ll[kMaxTopK];
  int id[kMaxTopK], oc[kMaxTopK];
  float ow[kMaxTopK];
  for (int j = 0; j < K; j++) {
    ll[j] = sel_ll[t * K + j];
    id[j] = sel[t * K + j];
  }
  const int n = finalize_frame(K, prune, ll, id, oc, ow);
  for (int e = 0; e < n; e++) {
    comp_pad[t * K + e] = oc[e];
    w_pad[t * K + e] = ow[e];
  }
  counts[t] = n;
}

// Fixed-K variant (the default top-20): the CTA's 128 frames are staged through shared memory with
// coalesced loads and stores, and every per-frame array lives in registers (static indices: no local
// memory).  Arithmetic and summation order are finalize_frame's, so the outputs are bit-identical.
template <int KT>
__global__ void __launch_bounds__(128) finalize_fixed_kernel(int64_t T, double prune, const int32_t* __restrict__ sel,
                                                             const double* __restrict__ sel_ll,
                                                             int32_t* __restrict__ comp_pad, float* __restrict__ w_pad,
                                                             int64_t* __restrict__ counts) {
  constexpr int LD = KT + 1;  // odd row stride: conflict-free row-per-thread accesses
  __shared__ double sll[128 * LD];
  __shared__ int sid[128 * LD];
  __shared__ float sw[128 * LD];
  const int64_t t0 = (int64_t)blockIdx.x * 128;
  const int nfr = T - t0 < 128 ? (int)(T - t0) : 128;
  for (int i = threadIdx.x; i < nfr * KT; i += 128) {
    const int r = i / KT, c = i - r * KT;
    sll[r * LD + c] = sel_ll[t0 * KT + i];
    sid[r * LD + c] = sel[t0 * KT + i];
  }
  __syncthreads();
  const int f = threadIdx.x;
  if (f < nfr) {
    double ll[KT];
    int id[KT];
#pragma unroll
    for (int j = 0; j < KT; j++) {
      ll[j] = sll[f * LD + j];
      id[j] = sid[f * LD + j];
    }
    double mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < KT; j++) mx = fmax(mx, ll[j]);
    if (!isfinite(mx)) mx = 0.0;  // scipy logsumexp convention
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < KT; j++) s += exp(ll[j] - mx);
    const double lse = log(s) + mx;
    int nkeep = 0, best = 0;
    double bestv = 0.0;
#pragma unroll
    for (int j = 0; j < KT; j++) {
      ll[j] = exp(ll[j] - lse);  // posterior over the selection
      if (j == 0 || ll[j] > bestv) {
        best = j;
        bestv = ll[j];
      }
      if (ll[j] >= prune) nkeep++;
    }
    const bool degenerate = nkeep == 0;
    bool keep[KT];
    double tot = 0.0;
#pragma unroll
    for (int j = 0; j < KT; j++) {
      keep[j] = degenerate ? (j == best) : (ll[j] >= prune);
      tot += keep[j] ? ll[j] : 0.0;
    }
    int n = 0;
#pragma unroll
    for (int j = 0; j < KT; j++) {
      if (!keep[j]) continue;
      int pos = 0;  // kept entries with a smaller component id (ids of a selection are distinct)
#pragma unroll
      for (int q = 0; q < KT; q++) pos += (keep[q] && id[q] < id[j]) ? 1 : 0;
      sid[f * LD + pos] = id[j];
      sw[f * LD + pos] = (float)(ll[j] / tot);
      n++;
    }
    counts[t0 + f] = n;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nfr * KT; i += 128) {
    const int r = i / KT, c = i - r * KT;
    comp_pad[t0 * KT + i] = sid[r * LD + c];
    w_pad[t0 * KT + i] = sw[r * LD + c];
  }
}

// ----------------------------------------------------------------------------- stage 4: scan + compact

constexpr int kScanBlock = 1024;

__global__ void scan_block_sums(const int64_t* counts, int64_t T, int64_t* block_sums) {
  __shared__ int64_t red[32];
  int64_t base = (int64_t)blockIdx.x * kScanBlock;
  int64_t s = 0;
  for (int i = threadIdx.x; i < kScanBlock; i += blockDim.x)
    if (base + i < T) s += counts[base + i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) tot += red[w];
    block_sums[blockIdx.x] = tot;
  }
}

__global__ void scan_block_prefix(int64_t* block_sums, int nblocks) {
  // single CTA exclusive scan over the block sums (sequential chunks, parallel within)
  __shared__ int64_t carry;
  __shared__ int64_t buf[1024];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nblocks; base += 1024) {
    int i = base + threadIdx.x;
    int64_t v = i < nblocks ? block_sums[i] : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      int64_t add = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < nblocks) block_sums[i] = carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += buf[1023];
    __syncthreads();
  }
}

__global__ void scan_write_offsets(const int64_t* counts, int64_t T, const int64_t* block_prefix, int64_t* offsets) {
  __shared__ int64_t buf[kScanBlock];
  int64_t base = (int64_t)blockIdx.x * kScanBlock;
  int i = threadIdx.x;  // blockDim == kScanBlock
  int64_t v = base + i < T ? counts[base + i] : 0;
  buf[i] = v;
  __syncthreads();
  for (int o = 1; o < kScanBlock; o <<= 1) {
    int64_t add = i >= o ? buf[i - o] : 0;
    __syncthreads();
    buf[i] += add;
    __syncthreads();
  }
  int64_t pre = block_prefix[blockIdx.x];
  if (base + i < T) offsets[base + i] = pre + buf[i] - v;
  if (base + i == T - 1) offsets[T] = pre + buf[i];
}

// Warp per 32 consecutive frames: their CSR range [offsets[t0], offsets[t0 + 32]) is contiguous, so
// lane l writes entries l, l + 32, ... of it (coalesced); the frame of an entry is found by a binary
// search over the warp's 33 offsets (shuffled), its slot in the padded arrays follows.
__global__ void compact_kernel(int64_t T, int K, const int64_t* offsets, const int32_t* comp_pad, const float* w_pad,
                               int32_t* comps, float* wts) {
  const int lane = threadIdx.x & 31;
  const int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
  if (t0 >= T) return;
  const int nf = T - t0 < 32 ? (int)(T - t0) : 32;
  const int64_t my = offsets[t0 + min(lane, nf)];  // lane l: offset of frame t0 + l (lane nf: the end)
  const int64_t o0 = __shfl_sync(0xffffffffu, my, 0);
  const int64_t oend = __shfl_sync(0xffffffffu, offsets[t0 + nf], 0);
  const int total = (int)(oend - o0);
  for (int e = lane; e < total + 31 - (total + 31) % 32; e += 32) {
    // largest frame f with offset(f) - o0 <= e
    int lo = 0, hi = nf - 1;
#pragma unroll 1
    for (int step = 0; step < 5; step++) {
      const int mid = (lo + hi + 1) >> 1;
      const int64_t om = __shfl_sync(0xffffffffu, my, mid);
      if (om - o0 <= e) lo = mid;
      else hi = mid - 1;
    }
    const int64_t of = __shfl_sync(0xffffffffu, my, lo);
    if (e < total) {
      const int64_t src = (t0 + lo) * K + (o0 + e - of);
      comps[o0 + e] = comp_pad[src];
      wts[o0 + e] = w_pad[src];
    }
  }
}

int exclusive_scan_counts(const int64_t* counts, int64_t T, int64_t* offsets, int64_t* block_sums, cudaStream_t st) {
  int nb = (int)((T + kScanBlock - 1) / kScanBlock);
  scan_block_sums<<<nb, 256, 0, st>>>(counts, T, block_sums);
  scan_block_prefix<<<1, 1024, 0, st>>>(block_sums, nb);
  scan_write_offsets<<<nb, kScanBlock, 0, st>>>(counts, T, block_sums, offsets);
  TVK_CHECK_LAUNCH("scan");
  return TVK_OK;
}

static size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

struct AlignWs {
  int32_t* sel;
  double* sel_ll;
  int32_t* comp_pad;
  float* w_pad;
  int64_t* counts;
  int64_t* block_sums;
  void* group;  // grouped-path scratch (pair sort)
  int64_t group_bytes;
  size_t bytes;
};

static AlignWs carve(void* base, int64_t T, int K, int C) {
  AlignWs w{};
  size_t off = 0;
  char* b = (char*)base;
  auto take = [&](size_t n) {
    char* p = b ? b + off : nullptr;
    off += align_up(n);
    return p;
  };
  w.sel = (int32_t*)take(sizeof(int32_t) * T * K);
  w.sel_ll = (double*)take(sizeof(double) * T * K);
  w.comp_pad = (int32_t*)take(sizeof(int32_t) * T * K);
  w.w_pad = (float*)take(sizeof(float) * T * K);
  w.counts = (int64_t*)take(sizeof(int64_t) * (T + 1));
  w.block_sums = (int64_t*)take(sizeof(int64_t) * ((T + kScanBlock - 1) / kScanBlock + 1));
  w.group_bytes = grouped_workspace_bytes(T * K, C);
  w.group = take((size_t)w.group_bytes);
  w.bytes = off;
  return w;
}

}  // namespace tvk

using namespace tvk;

extern "C" int tvk_diag_table(const double* weights, const double* means, const double* variances, int C, int F,
                              double* table, void* stream) {
  TVK_REQUIRE(C >= 1 && F >= 1, "diag_table: empty model");
  diag_table_kernel<<<ceil_div(C, 128), 128, 0, (cudaStream_t)stream>>>(weights, means, variances, C, F, table);
  TVK_CHECK_LAUNCH("diag_table");
  return diag_table_tc(table, C, F, (cudaStream_t)stream);
}

extern "C" int64_t tvk_diag_table_bytes(int C, int F) { return (int64_t)diag_table_bytes(C, F); }

extern "C" int tvk_full_table(const double* weights, const double* means, const double* covariances, int C, int F,
                              double* table, int32_t* status, void* stream) {
  TVK_REQUIRE(C >= 1 && F >= 1 && F <= kSmallSpdMax, "full_table: need 1 <= F <= 96");
  size_t smem = sizeof(double) * (2 * F * F + F);
  cudaFuncSetAttribute(full_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double) * (2 * kSmallSpdMax * kSmallSpdMax + kSmallSpdMax)));
  full_table_kernel<<<C, 256, smem, (cudaStream_t)stream>>>(weights, means, covariances, C, F, table, status);
  TVK_CHECK_LAUNCH("full_table");
  return TVK_OK;
}

extern "C" int64_t tvk_align_workspace_bytes(int64_t T, int K, int C) { return (int64_t)carve(nullptr, T, K, C).bytes; }

namespace tvk {

static bool sparse_disabled() {  // TVK_ALIGN_SPARSE=1 opts into the approximate + exact path (align_grouped.cu)
  const char* e = getenv("TVK_ALIGN_SPARSE");
  return !(e && strcmp(e, "1") == 0);
}

static bool select_dmma_forced() {  // TVK_SELECT=dmma: the FP64 DMMA preselection (A/B comparisons)
  const char* e = getenv("TVK_SELECT");
  return e && strcmp(e, "dmma") == 0;
}

template <typename XT>
static int launch_select(const XT* x, int64_t T, int F, const double* diag_table, int C, int K, int32_t* sel,
                         double* val, cudaStream_t st) {
  if (select_tc_supported(F, K, C) && !select_dmma_forced()) return select_tc<XT>(x, T, F, diag_table, C, K, sel, val, st);
  size_t smem = sel::smem_bytes(F, K);
  // shapes outside both fast kernels (top_k > 32, wide F): the generic per-frame selection
  if (K > kMaxTopK || smem > 227 * 1024) return wide_select<XT>(x, T, F, diag_table, C, K, sel, val, st);
  cudaFuncSetAttribute(select_topk_kernel<XT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t grid = (T + sel::BM - 1) / sel::BM;
  TVK_REQUIRE(grid < (1ll << 31), "align_frames: too many frames for one call");
  select_topk_kernel<XT><<<(unsigned)grid, sel::NT, smem, st>>>(x, T, F, diag_table, C, K, sel, val);
  TVK_CHECK_LAUNCH("select_topk");
  return TVK_OK;
}

template <typename XT>
static int launch_full_ll(const XT* x, int64_t T, int F, const double* full_table, int C, int K, const int32_t* sel,
                          double* sel_ll, cudaStream_t st) {
  using Cfg = fll::Cfg;
  using L = SmemLayout<Cfg::BM, Cfg::BN, Cfg::BK, false, false>;
  int Q = 1 + F + F * (F + 1) / 2;
  int Qpad = (Q + Cfg::BK - 1) / Cfg::BK * Cfg::BK;
  size_t smem = sizeof(double) * Cfg::STAGES * L::STAGE + sizeof(XT) * Cfg::BM * (F + 1) + sizeof(int) * Qpad +
                Cfg::BM * Cfg::BN;
  TVK_REQUIRE(smem <= 227 * 1024, "align_frames: F too large for the full-covariance tile");
  cudaFuncSetAttribute(full_ll_kernel<XT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t mt = (T + Cfg::BM - 1) / Cfg::BM, nt = (C + Cfg::BN - 1) / Cfg::BN;
  TVK_REQUIRE(mt * nt < (1ll << 31), "align_frames: too many frames for one call");
  full_ll_kernel<XT><<<(unsigned)(mt * nt), Cfg::NT, smem, st>>>(x, T, F, full_table, C, K, sel, sel_ll);
  TVK_CHECK_LAUNCH("full_ll");
  return TVK_OK;
}

template <typename XT>
static int full_ll_dispatch(const XT* x, int64_t T, int F, const double* full_table, const double* prec_table,
                            int C, int K, int flags, const int32_t* sel, double* sel_ll, void* group_ws,
                            int64_t group_bytes, cudaStream_t st) {
  if (flags & TVK_ALIGN_DENSE) {
    TVK_REQUIRE(full_table != nullptr, "align_frames: dense mode needs the quadratic-feature table");
    TVK_REQUIRE(K <= kMaxTopK, "align_frames: dense mode supports top_k <= 32");
    return launch_full_ll<XT>(x, T, F, full_table, C, K, sel, sel_ll, st);
  }
  TVK_REQUIRE(prec_table != nullptr, "align_frames: grouped mode needs the precision table");
  return grouped_full_ll<XT>(x, T, F, prec_table, C, K, sel, sel_ll, group_ws, group_bytes, st);
}

template <typename XT>
__global__ void frame_features_kernel(const XT* x, int64_t T, int F, int kind, double* out) {
  // kind 0: [x^2, x, 1] (2F+1); kind 1: [1, x_i, x_i x_j (i<=j)] (1+F+F(F+1)/2)
  int Q = kind == 0 ? 2 * F + 1 : 1 + F + F * (F + 1) / 2;
  int64_t total = T * Q;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = idx / Q;
    int k = (int)(idx % Q);
    const XT* xr = x + t * F;
    double v;
    if (kind == 0) {
      v = k < F ? (double)xr[k] * (double)xr[k] : (k < 2 * F ? (double)xr[k - F] : 1.0);
    } else if (k == 0) {
      v = 1.0;
    } else if (k <= F) {
      v = (double)xr[k - 1];
    } else {
      int p = k - 1 - F, i = 0, base = 0;
      while (base + (F - i) <= p) {
        base += F - i;
        i++;
      }
      v = (double)xr[i] * (double)xr[i + (p - base)];
    }
    out[idx] = v;
  }
}

template <typename XT>
static int align_impl(const XT* x, int64_t T, int F, const double* diag_table, const double* full_table,
                      const double* prec_table, int C, int K, double prune, int flags, void* workspace,
                      int64_t workspace_bytes, int64_t* offsets, int32_t* components, float* weights,
                      int32_t* selected, double* sel_ll_out, cudaStream_t st) {
  AlignWs w = carve(workspace, T, K, C);
  TVK_REQUIRE(workspace != nullptr && (int64_t)w.bytes <= workspace_bytes, "align_frames: workspace too small");
  TVK_TRY(launch_select<XT>(x, T, F, diag_table, C, K, w.sel, nullptr, st));
  int fb = (int)((T + 127) / 128);
  if (!(flags & TVK_ALIGN_DENSE) && sel_ll_out == nullptr && !sparse_disabled() && K <= kMaxTopK && F <= 64) {
    // FP64 log-likelihoods only where the kept set or its weights need them
    TVK_REQUIRE(prec_table != nullptr, "align_frames: grouped mode needs the precision table");
    TVK_TRY(grouped_align_sparse<XT>(x, T, F, prec_table, C, K, prune, w.sel, w.sel_ll, w.comp_pad, w.w_pad,
                                     w.counts, w.group, w.group_bytes, st));
  } else {
    TVK_TRY(full_ll_dispatch<XT>(x, T, F, full_table, prec_table, C, K, flags, w.sel, w.sel_ll, w.group,
                                 w.group_bytes, st));
    if (K == 20) {
      finalize_fixed_kernel<20><<<fb, 128, 0, st>>>(T, prune, w.sel, w.sel_ll, w.comp_pad, w.w_pad, w.counts);
      TVK_CHECK_LAUNCH("finalize");
    } else if (K <= kMaxTopK) {
      finalize_kernel<<<fb, 128, 0, st>>>(T, K, prune, w.sel, w.sel_ll, w.comp_pad, w.w_pad, w.counts);
      TVK_CHECK_LAUNCH("finalize");
    } else {
      TVK_TRY(finalize_wide(T, K, prune, w.sel, w.sel_ll, w.comp_pad, w.w_pad, w.counts, st));
    }
  }
  TVK_TRY(exclusive_scan_counts(w.counts, T, offsets, w.block_sums, st));
  compact_kernel<<<(int)((T + 127) / 128), 128, 0, st>>>(T, K, offsets, w.comp_pad, w.w_pad, components, weights);
  TVK_CHECK_LAUNCH("compact");
  if (selected) cudaMemcpyAsync(selected, w.sel, sizeof(int32_t) * T * K, cudaMemcpyDeviceToDevice, st);
  if (sel_ll_out) cudaMemcpyAsync(sel_ll_out, w.sel_ll, sizeof(double) * T * K, cudaMemcpyDeviceToDevice, st);
  TVK_CHECK_LAUNCH("align_frames copies");
  return TVK_OK;
}

}  // namespace tvk

extern "C" int tvk_align_frames(const void* x, int x_f64, int64_t T, int F, const double* diag_table,
                                const double* full_table, const double* prec_table, int C, int K, double prune,
                                int flags, void* workspace, int64_t workspace_bytes, int64_t* offsets,
                                int32_t* components, float* weights, int32_t* selected, double* sel_ll_out,
                                void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TVK_REQUIRE(T >= 0 && F >= 1 && C >= 1, "align_frames: bad shape");
  TVK_REQUIRE(K >= 1 && K <= kWideMaxK && K <= C, "align_frames: top_k must be in [1, min(C, 8192)]");
  TVK_REQUIRE(F <= kWideMaxF, "align_frames: F must be <= 128");
  TVK_REQUIRE(C <= kGroupedMaxC, "align_frames: C must be <= 24576");
  if (T == 0) {
    cudaMemsetAsync(offsets, 0, sizeof(int64_t), st);
    TVK_CHECK_LAUNCH("align_frames memset");
    return TVK_OK;
  }
  if (x_f64)
    return align_impl<double>((const double*)x, T, F, diag_table, full_table, prec_table, C, K, prune, flags,
                              workspace, workspace_bytes, offsets, components, weights, selected, sel_ll_out, st);
  return align_impl<float>((const float*)x, T, F, diag_table, full_table, prec_table, C, K, prune, flags, workspace,
                           workspace_bytes, offsets, components, weights, selected, sel_ll_out, st);
}

extern "C" int tvk_select_topk(const void* x, int x_f64, int64_t T, int F, const double* diag_table, int C, int K,
                               int32_t* selected, double* values, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TVK_REQUIRE(T >= 0 && F >= 1 && C >= 1, "select_topk: bad shape");
  TVK_REQUIRE(K >= 1 && K <= kWideMaxK && K <= C, "select_topk: k must be in [1, min(C, 8192)]");
  if (T == 0) return TVK_OK;
  if (x_f64) return launch_select<double>((const double*)x, T, F, diag_table, C, K, selected, values, st);
  return launch_select<float>((const float*)x, T, F, diag_table, C, K, selected, values, st);
}

extern "C" int tvk_frame_features(const void* x, int x_f64, int64_t T, int F, int kind, double* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TVK_REQUIRE(T >= 0 && F >= 1 && (kind == 0 || kind == 1), "frame_features: bad arguments");
  if (T == 0) return TVK_OK;
  int64_t Q = kind == 0 ? 2 * F + 1 : 1 + F + (int64_t)F * (F + 1) / 2;
  int blocks = (int)std::min<int64_t>((T * Q + 255) / 256, 148 * 32);
  if (x_f64)
    frame_features_kernel<double><<<blocks, 256, 0, st>>>((const double*)x, T, F, kind, out);
  else
    frame_features_kernel<float><<<blocks, 256, 0, st>>>((const float*)x, T, F, kind, out);
  TVK_CHECK_LAUNCH("frame_features");
  return TVK_OK;
}

extern "C" int64_t tvk_full_loglik_workspace_bytes(int64_t T, int K, int C) {
  return grouped_workspace_bytes(T * K, C);
}

extern "C" int tvk_full_loglik_selected(const void* x, int x_f64, int64_t T, int F, const double* full_table,
                                        const double* prec_table, int C, int K, int flags, const int32_t* selected,
                                        double* sel_ll, void* workspace, int64_t workspace_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TVK_REQUIRE(T >= 0 && F >= 1 && C >= 1 && K >= 1 && K <= kWideMaxK && K <= C, "full_loglik_selected: bad shape");
  if (T == 0) return TVK_OK;
  if (x_f64)
    return full_ll_dispatch<double>((const double*)x, T, F, full_table, prec_table, C, K, flags, selected, sel_ll,
                                    workspace, workspace_bytes, st);
  return full_ll_dispatch<float>((const float*)x, T, F, full_table, prec_table, C, K, flags, selected, sel_ll,
                                 workspace, workspace_bytes, st);
}
