// Baum-Welch statistics (gmm.py:442-492), deterministic (no floating-point atomics).
//
// bw_first_order_kernel: one CTA per utterance.  The utterance's alignment entries are
// counting-sorted by component in shared memory (stable: frame order is kept inside a
// component, gmm.py:479 uses a stable argsort), then one warp per component sums
//   n_c = sum w,   f_c = sum w (x - m_c)
// in frame order and writes dense rows of N (U x C) and F (U x C*F) -- the operands of
// the E-step GEMMs.  Optionally the per-utterance second order S (API path).
//
// bw_second_order_kernel: one CTA per component accumulates the corpus second-order sum
//   Ssum_c += sum_u sum_t w (x - m_c)(x - m_c)^T
// over the component's runs, utterance by utterance, each accumulator element owned by one
// thread (fixed summation order).
#include "common.cuh"
#include "internal.h"

namespace tvk {

constexpr int kBwThreads = 256;
constexpr int kBwMaxC = 49152;  // first-order counting sort: C+1 ints of shared memory

struct BwWs {
  int32_t* ent_frame;   // [Ecap] frame of each entry
  int32_t* sorted_frame;  // [Ecap] entries of each utterance sorted by component
  double* sorted_w;     // [Ecap]
  int32_t* comp_start;  // [U][C+1] run starts (relative to the utterance's first entry)
  size_t bytes;
};

static size_t aup(size_t v) { return (v + 255) & ~size_t(255); }

static BwWs bw_carve(void* base, int64_t E, int U, int C) {
  BwWs w{};
  char* b = (char*)base;
  size_t off = 0;
  auto take = [&](size_t n) {
    char* p = b ? b + off : nullptr;
    off += aup(n);
    return p;
  };
  w.ent_frame = (int32_t*)take(sizeof(int32_t) * (E + 1));
  w.sorted_frame = (int32_t*)take(sizeof(int32_t) * (E + 1));
  w.sorted_w = (double*)take(sizeof(double) * (E + 1));
  w.comp_start = (int32_t*)take(sizeof(int32_t) * (int64_t)U * (C + 1));
  w.bytes = off;
  return w;
}

template <typename XT>
__global__ void __launch_bounds__(kBwThreads) bw_first_order_kernel(
    const XT* x, int F, const int64_t* utt_frames, const int64_t* ali_off, const int32_t* comps,
    const float* wts, int C, const double* center, double* n_out, double* f_out, double* S_out, BwWs ws) {
  extern __shared__ int cnt[];  // [C+1] counts -> starts -> cursors
  __shared__ int part[kBwThreads];
  const int u = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t t0 = utt_frames[u], t1 = utt_frames[u + 1];
  const int64_t ebase = ali_off[utt_frames[0]];
  const int64_t e0 = ali_off[t0], e1 = ali_off[t1];
  const int ne = (int)(e1 - e0);
  const int64_t r0 = e0 - ebase;  // this utterance's region in the sorted arrays

  for (int c = tid; c <= C; c += kBwThreads) cnt[c] = 0;
  for (int64_t t = t0 + tid; t < t1; t += kBwThreads)
    for (int64_t e = ali_off[t]; e < ali_off[t + 1]; e++) ws.ent_frame[e - ebase] = (int32_t)t;
  __syncthreads();
  for (int i = tid; i < ne; i += kBwThreads) atomicAdd(&cnt[comps[e0 + i]], 1);  // integer: exact
  __syncthreads();
  // exclusive scan of cnt[0..C) -> starts; cnt[C] = ne
  {
    int per = (C + kBwThreads - 1) / kBwThreads;
    int lo = tid * per, hi = min(lo + per, C);
    int s = 0;
    for (int c = lo; c < hi; c++) s += cnt[c];
    part[tid] = s;
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int i = 0; i < kBwThreads; i++) {
        int v = part[i];
        part[i] = run;
        run += v;
      }
    }
    __syncthreads();
    int run = part[tid];
    for (int c = lo; c < hi; c++) {
      int v = cnt[c];
      cnt[c] = run;
      run += v;
    }
    if (tid == 0) cnt[C] = ne;
    __syncthreads();
  }
  int32_t* cs = ws.comp_start + (int64_t)u * (C + 1);
  for (int c = tid; c <= C; c += kBwThreads) cs[c] = cnt[c];
  __syncthreads();
  // stable scatter (warp 0, entries in order): cnt[] becomes the running cursor
  if (warp == 0) {
    for (int base = 0; base < ne; base += 32) {
      __syncwarp();  // the previous round's cursor updates (other lanes) are visible to this round's leaders
      int i = base + lane;
      bool act = i < ne;
      unsigned am = __ballot_sync(0xffffffffu, act);
      if (!act) continue;
      int key = comps[e0 + i];
      unsigned peers = __match_any_sync(am, key);
      int leader = __ffs(peers) - 1;
      int rank = __popc(peers & ((1u << lane) - 1));
      int p0 = 0;
      if (lane == leader) {
        p0 = cnt[key];
        cnt[key] = p0 + __popc(peers);
      }
      p0 = __shfl_sync(am, p0, leader);
      int pos = p0 + rank;
      ws.sorted_frame[r0 + pos] = ws.ent_frame[e0 - ebase + i];
      ws.sorted_w[r0 + pos] = (double)wts[e0 + i];
    }
  }
  __syncthreads();
  // one warp per component: n_c, f_c (dense rows, zero for absent components)
  double* nrow = n_out + (int64_t)u * C;
  double* frow = f_out + (int64_t)u * C * F;
  for (int c = warp; c < C; c += kBwThreads / 32) {
    int s = cs[c], n = cs[c + 1] - s;
    double* fc = frow + (int64_t)c * F;
    if (n == 0) {
      for (int j = lane; j < F; j += 32) fc[j] = 0.0;
      if (lane == 0) nrow[c] = 0.0;
      continue;
    }
    const double* mc = center ? center + (int64_t)c * F : nullptr;
    // one pass over the component's entries for all features (lane j takes j, j + 32, j + 64, j + 96):
    // each f_c[j] and n_c still sums in entry order, as the reference's stable-sorted sums do
    double acc[4] = {0.0, 0.0, 0.0, 0.0}, mcj[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 4; q++)
      if (mc && lane + 32 * q < F) mcj[q] = mc[lane + 32 * q];
    double occ = 0.0;
#pragma unroll 4
    for (int r = 0; r < n; r++) {
      const int t = ws.sorted_frame[r0 + s + r];
      const double w = ws.sorted_w[r0 + s + r];
      occ += w;
      const XT* xr = x + (int64_t)t * F;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int j = lane + 32 * q;
        if (32 * q < F && j < F) {
          double xv = (double)xr[j];
          if (mc) xv -= mcj[q];
          acc[q] += w * xv;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; q++)
      if (lane + 32 * q < F) fc[lane + 32 * q] = acc[q];
    if (lane == 0) nrow[c] = occ;
  }
  if (S_out == nullptr) return;
  // per-utterance second order (reference API path): S_c = sym(sum (x w) x^T)
  double* Srow = S_out + (int64_t)u * C * F * F;
  for (int c = warp; c < C; c += kBwThreads / 32) {
    int s = cs[c], n = cs[c + 1] - s;
    double* Sc = Srow + (int64_t)c * F * F;
    const double* mc = center ? center + (int64_t)c * F : nullptr;
    for (int p = lane; p < F * F; p += 32) {
      int i = p / F, j = p % F;
      if (j > i) continue;
      double acc = 0.0;
      for (int r = 0; r < n; r++) {
        int t = ws.sorted_frame[r0 + s + r];
        double w = ws.sorted_w[r0 + s + r];
        double xi = (double)x[(int64_t)t * F + i], xj = (double)x[(int64_t)t * F + j];
        if (mc) {
          xi -= mc[i];
          xj -= mc[j];
        }
        acc += (xi * w) * xj;
      }
      Sc[i * F + j] = acc;
      Sc[j * F + i] = acc;
    }
  }
}

constexpr int kSoUttChunk = 1024;  // utterance runs gathered per pass
constexpr int kSoMaxF = 128;

// MP = lower-triangle pairs per thread: 8 covers F <= 63 (F(F+1)/2 <= 8*256), 33 covers F <= 128
template <typename XT, int kSoMaxPairs>
__global__ void __launch_bounds__(kBwThreads) bw_second_order_kernel(const XT* x, int F, int U, int C,
                                                                     const int64_t* utt_frames,
                                                                     const int64_t* ali_off, const double* center,
                                                                     double* ssum, BwWs ws) {
  __shared__ int run_s[kSoUttChunk], run_n[kSoUttChunk];
  __shared__ int64_t run_r0[kSoUttChunk];
  constexpr int kSoBatch = kSoMaxPairs > 8 ? 16 : 32;  // entries staged per round (48 KB static smem)
  __shared__ double xe[kSoBatch][kSoMaxPairs > 8 ? kSoMaxF : 64];
  __shared__ double we[kSoBatch];
  const int c = blockIdx.x, tid = threadIdx.x;
  const int npair = F * (F + 1) / 2;
  int pi[kSoMaxPairs], pj[kSoMaxPairs];
  double acc[kSoMaxPairs];
#pragma unroll
  for (int k = 0; k < kSoMaxPairs; k++) {
    int p = tid + k * kBwThreads;
    int i = 0, base = 0;
    if (p < npair) {
      while (base + (i + 1) <= p) {  // row-major lower: row i has i+1 entries
        base += i + 1;
        i++;
      }
    }
    pi[k] = i;
    pj[k] = p - base;
    acc[k] = 0.0;
  }
  const int64_t ebase = ali_off[utt_frames[0]];
  const double* mc = center ? center + (int64_t)c * F : nullptr;
  for (int u0 = 0; u0 < U; u0 += kSoUttChunk) {
    int nu = min(kSoUttChunk, U - u0);
    __syncthreads();
    for (int k = tid; k < nu; k += kBwThreads) {
      const int32_t* cs = ws.comp_start + (int64_t)(u0 + k) * (C + 1);
      run_s[k] = cs[c];
      run_n[k] = cs[c + 1] - cs[c];
      run_r0[k] = ali_off[utt_frames[u0 + k]] - ebase;
    }
    __syncthreads();
    // walk the runs in utterance order, staging kSoBatch entries at a time
    int k = 0, r = 0;
    while (true) {
      // collect the next batch positions (identical walk in every thread)
      int kk = k, rr = r, nb = 0;
      int64_t pos[kSoBatch];
      while (nb < kSoBatch && kk < nu) {
        if (rr < run_n[kk]) {
          pos[nb++] = run_r0[kk] + run_s[kk] + rr;
          rr++;
        } else {
          kk++;
          rr = 0;
        }
      }
      if (nb == 0) break;
      __syncthreads();
      for (int idx = tid; idx < nb * F; idx += kBwThreads) {
        int e = idx / F, j = idx % F;
        int t = ws.sorted_frame[pos[e]];
        double v = (double)x[(int64_t)t * F + j];
        if (mc) v -= mc[j];
        xe[e][j] = v;
      }
      for (int e = tid; e < nb; e += kBwThreads) we[e] = ws.sorted_w[pos[e]];
      __syncthreads();
      for (int e = 0; e < nb; e++) {
        double w = we[e];
#pragma unroll
        for (int q = 0; q < kSoMaxPairs; q++)
          if (tid + q * kBwThreads < npair) acc[q] += (xe[e][pi[q]] * w) * xe[e][pj[q]];
      }
      k = kk;
      r = rr;
    }
  }
  double* S = ssum + (int64_t)c * F * F;
#pragma unroll
  for (int q = 0; q < kSoMaxPairs; q++) {
    if (tid + q * kBwThreads >= npair) continue;
    int i = pi[q], j = pj[q];
    double v = S[i * F + j] + acc[q];
    S[i * F + j] = v;
    if (i != j) S[j * F + i] = v;
  }
}

// F <= 64: the same corpus sum as a tensor-pipe product.  Per component, S_c += X_c^T (w X_c) over the
// component's entries in utterance / frame order: the entry positions of a chunk of utterances are
// listed once in shared memory (block scan over the utterances' run lengths), then staged 64 entries
// at a time (x - m_c and w (x - m_c), all 16 loads of a thread in flight together; rows zero-padded
// to a multiple of 4, columns to 64) and each warp accumulates its share of the 8x8 blocks of the lower
// triangle with DMMA.8x8x4 (K = entries).  Diagonal blocks store their lower half and mirror it, so
// S_c stays exactly symmetric.
constexpr int kSoDmmaChunk = 256;   // utterances per position list
constexpr int kSoPosCap = 4096;     // positions per list (a longer chunk is split)
constexpr int kSoEB = 64;           // entries staged per round
constexpr int kSoLD = 68;           // = 4 mod 16 doubles: conflict-free DMMA fragment loads
constexpr size_t so_dmma_smem() {
  return sizeof(double) * 2 * kSoEB * kSoLD + sizeof(int) * (kSoPosCap + 2 * kSoDmmaChunk + 8);
}
template <typename XT>
__global__ void __launch_bounds__(kBwThreads, 2) bw_second_order_dmma_kernel(const XT* x, int F, int U, int C,
                                                                             const int64_t* utt_frames,
                                                                             const int64_t* ali_off,
                                                                             const double* center, double* ssum,
                                                                             BwWs ws) {
  extern __shared__ __align__(16) double sod[];
  double (*xe)[kSoLD] = reinterpret_cast<double (*)[kSoLD]>(sod);
  double (*wxe)[kSoLD] = reinterpret_cast<double (*)[kSoLD]>(sod + kSoEB * kSoLD);
  int* pos = reinterpret_cast<int*>(sod + 2 * kSoEB * kSoLD);  // [kSoPosCap] entry positions
  int* roff = pos + kSoPosCap;                                 // [kSoDmmaChunk + 1] run offsets
  int* scan = roff + kSoDmmaChunk + 1;                         // [kSoDmmaChunk] block scan scratch
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nbF = (F + 7) / 8, nblk = nbF * (nbF + 1) / 2;
  constexpr int MAXQ = 5;  // 36 lower 8x8 blocks at F = 64 over 8 warps
  int bi[MAXQ], bj[MAXQ];
  double acc[MAXQ][2];
#pragma unroll
  for (int q = 0; q < MAXQ; q++) {
    int b = warp + 8 * q, i = 0;
    while ((i + 1) * (i + 2) / 2 <= b) i++;  // block b -> (i, j), j <= i, row-major lower
    bi[q] = i;
    bj[q] = b - i * (i + 1) / 2;
    acc[q][0] = acc[q][1] = 0.0;
  }
  const int nq = (nblk - warp + 7) / 8;  // blocks of this warp
  const int64_t ebase = ali_off[utt_frames[0]];
  const double* mc = center ? center + (int64_t)c * F : nullptr;
  for (int u0 = 0; u0 < U;) {
    int nu = min(kSoDmmaChunk, U - u0);
    __syncthreads();  // the previous list is consumed
    // run lengths of this component in utterances u0.., exclusive scan -> roff
    int len = 0, r0 = 0, s0 = 0;
    if (tid < nu) {
      const int32_t* cs = ws.comp_start + (int64_t)(u0 + tid) * (C + 1);
      s0 = cs[c];
      len = cs[c + 1] - s0;
      r0 = (int)(ali_off[utt_frames[u0 + tid]] - ebase);
    }
    scan[tid] = len;
    __syncthreads();
    for (int o = 1; o < kSoDmmaChunk; o <<= 1) {  // Hillis-Steele inclusive scan
      const int v = tid >= o ? scan[tid - o] : 0;
      __syncthreads();
      scan[tid] += v;
      __syncthreads();
    }
    // the chunk's entries in windows of kSoPosCap positions (a long run spans windows)
    const int total_all = scan[nu - 1];
    const int off = scan[tid < nu ? tid : 0] - len;
    for (int w0 = 0; w0 < total_all; w0 += kSoPosCap) {
      const int total = min(kSoPosCap, total_all - w0);
      __syncthreads();  // the previous window is consumed
      if (tid < nu)
        for (int rr = max(0, w0 - off); rr < len && off + rr < w0 + kSoPosCap; rr++) pos[off + rr - w0] = r0 + s0 + rr;
      __syncthreads();
      // rounds of kSoEB entries; the gathers of round r + 1 (position -> frame -> features, two
      // dependent global loads) are issued before round r's DMMAs, so their latency overlaps the math
      constexpr int NV = kSoEB * 64 / kBwThreads;
      double v[NV], wv[NV];
      auto gather = [&](int e0, int nb) {
#pragma unroll
        for (int i = 0; i < NV; i++) {
          const int idx = tid + kBwThreads * i, e = idx >> 6, j = idx & 63;
          v[i] = wv[i] = 0.0;
          if (e < nb && j < F) {
            const int p = pos[e0 + e];
            const int tt = ws.sorted_frame[p];
            double xv = (double)x[(int64_t)tt * F + j];
            if (mc) xv -= mc[j];
            v[i] = xv;
            wv[i] = ws.sorted_w[p] * xv;
          }
        }
      };
      if (total > 0) gather(0, min(kSoEB, total));
      for (int e0 = 0; e0 < total; e0 += kSoEB) {
        const int nb = min(kSoEB, total - e0);
        __syncthreads();  // the previous round's DMMAs are done with xe / wxe
#pragma unroll
        for (int i = 0; i < NV; i++) {
          const int idx = tid + kBwThreads * i, e = idx >> 6, j = idx & 63;
          xe[e][j] = v[i];
          wxe[e][j] = wv[i];
        }
        __syncthreads();
        if (e0 + kSoEB < total) gather(e0 + kSoEB, min(kSoEB, total - e0 - kSoEB));
        const int nks = (nb + 3) >> 2;
        for (int ks = 0; ks < nks; ks++) {
          const int e = 4 * ks + t4;
#pragma unroll
          for (int q = 0; q < MAXQ; q++)
            if (q < nq) dmma884(acc[q][0], acc[q][1], xe[e][8 * bi[q] + g], wxe[e][8 * bj[q] + g]);
        }
      }
    }
    u0 += nu;
  }
  double* S = ssum + (int64_t)c * F * F;
#pragma unroll
  for (int q = 0; q < MAXQ; q++) {
    if (q >= nq) continue;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int row = 8 * bi[q] + g, col = 8 * bj[q] + 2 * t4 + h;  // D[g][2t + h]
      if (row >= F || col >= F || col > row) continue;
      const double val = S[row * F + col] + acc[q][h];
      S[row * F + col] = val;
      if (row != col) S[col * F + row] = val;
    }
  }
}

}  // namespace tvk

using namespace tvk;

extern "C" int64_t tvk_bw_workspace_bytes(int64_t E, int U, int C) { return (int64_t)bw_carve(nullptr, E, U, C).bytes; }

extern "C" int tvk_bw_stats(const void* x, int x_f64, int F, const int64_t* utt_frames, int U, const int64_t* ali_offsets,
                            const int32_t* components, const float* weights, int C, const double* center,
                            double* n_out, double* f_out, double* S_out, double* ssum_acc, int64_t entry_capacity,
                            void* workspace, int64_t workspace_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TVK_REQUIRE(F >= 1 && C >= 1 && U >= 0, "bw_stats: bad shape");
  TVK_REQUIRE(C <= kBwMaxC, "bw_stats: C > 49152 not supported");
  if (U == 0) return TVK_OK;
  TVK_REQUIRE(workspace != nullptr, "bw_stats: workspace required");
  TVK_REQUIRE((int64_t)bw_carve(nullptr, entry_capacity, U, C).bytes <= workspace_bytes,
              "bw_stats: workspace too small for the entry capacity");
  BwWs ws = bw_carve(workspace, entry_capacity, U, C);
  size_t smem = sizeof(int) * (C + 1);
  if (x_f64) {
    cudaFuncSetAttribute(bw_first_order_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bw_first_order_kernel<double><<<U, kBwThreads, smem, st>>>((const double*)x, F, utt_frames, ali_offsets,
                                                               components, weights, C, center, n_out, f_out, S_out,
                                                               ws);
  } else {
    cudaFuncSetAttribute(bw_first_order_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bw_first_order_kernel<float><<<U, kBwThreads, smem, st>>>((const float*)x, F, utt_frames, ali_offsets,
                                                              components, weights, C, center, n_out, f_out, S_out,
                                                              ws);
  }
  TVK_CHECK_LAUNCH("bw_first_order");
  if (ssum_acc) {
    TVK_REQUIRE(F <= kSoMaxF, "bw_stats: corpus second order supports F <= 128");
    if (F <= 64) {  // DMMA tensor-pipe product
      const size_t sm = so_dmma_smem();
      if (x_f64) {
        cudaFuncSetAttribute(bw_second_order_dmma_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        bw_second_order_dmma_kernel<double><<<C, kBwThreads, sm, st>>>((const double*)x, F, U, C, utt_frames,
                                                                        ali_offsets, center, ssum_acc, ws);
      } else {
        cudaFuncSetAttribute(bw_second_order_dmma_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        bw_second_order_dmma_kernel<float><<<C, kBwThreads, sm, st>>>((const float*)x, F, U, C, utt_frames,
                                                                       ali_offsets, center, ssum_acc, ws);
      }
    } else {
      if (x_f64)
        bw_second_order_kernel<double, 33><<<C, kBwThreads, 0, st>>>((const double*)x, F, U, C, utt_frames,
                                                                     ali_offsets, center, ssum_acc, ws);
      else
        bw_second_order_kernel<float, 33><<<C, kBwThreads, 0, st>>>((const float*)x, F, U, C, utt_frames,
                                                                    ali_offsets, center, ssum_acc, ws);
    }
    TVK_CHECK_LAUNCH("bw_second_order");
  }
  return TVK_OK;
}
