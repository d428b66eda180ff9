// FP64 tensor-pipe GEMM core (DMMA.8x8x4) used by every dense contraction of the
// i-vector path: L = I + N U (E-step precision), b = F W, A += N^T M, B += F^T phi,
// workspace U_c = T_c^T Sigma_c^-1 T_c, T <- T R, plus the fused alignment kernels
// (quadratic-feature log-likelihoods) which supply their own A-operand producer.
//
// Tiles are staged global->shared with cp.async (LDGSTS), multi-stage; the shared
// layouts are padded so that the 8x4 / 4x8 fragment reads are bank-conflict free.
#pragma once
#include "common.cuh"

namespace tvk {

// Shared-memory operand layouts.
//  A: MK = [BM][BK+4] (k contiguous), KM = [BK][BM+4] (m contiguous)
//  B: KN = [BK][BN+4] (n contiguous), NK = [BN][BK+4] (k contiguous)
template <int BM, int BN, int BK, bool A_KM, bool B_NK>
struct SmemLayout {
  static constexpr int A_ELEMS = A_KM ? BK * (BM + 4) : BM * (BK + 4);
  static constexpr int B_ELEMS = B_NK ? BN * (BK + 4) : BK * (BN + 4);
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  __device__ static __forceinline__ int a_off(int m, int k) { return A_KM ? k * (BM + 4) + m : m * (BK + 4) + k; }
  __device__ static __forceinline__ int b_off(int k, int n) { return B_NK ? n * (BK + 4) + k : k * (BN + 4) + n; }
};

// Loads a BROWS x BCOLS tile of a row-major global matrix (leading dim ld) whose
// contiguous axis is the column axis, into smem rows of stride SROW doubles.
// Rows >= nrows or cols >= ncols are zero-filled.  VEC uses 16-byte copies and
// requires ld even and a 16-byte aligned base.
template <int BROWS, int BCOLS, int SROW, int NT, bool VEC>
__device__ __forceinline__ void load_tile_async(double* s, const double* g, int64_t ld, int row0, int col0,
                                                int nrows, int ncols, int tid) {
  if constexpr (VEC) {
    constexpr int CPR = BCOLS / 2;  // 16-byte chunks per row
    constexpr int TOTAL = BROWS * CPR;
#pragma unroll
    for (int i = tid; i < TOTAL; i += NT) {
      int r = i / CPR, c = (i % CPR) * 2;
      int gr = row0 + r, gc = col0 + c;
      int valid = 0;
      const double* src = g;
      if (gr < nrows && gc < ncols) {
        valid = (gc + 1 < ncols) ? 16 : 8;
        src = g + (int64_t)gr * ld + gc;
      }
      cp_async16(s + r * SROW + c, src, valid);
    }
  } else {
    constexpr int TOTAL = BROWS * BCOLS;
#pragma unroll 4
    for (int i = tid; i < TOTAL; i += NT) {
      int r = i / BCOLS, c = i % BCOLS;
      int gr = row0 + r, gc = col0 + c;
      bool ok = gr < nrows && gc < ncols;
      cp_async8(s + r * SROW + c, ok ? g + (int64_t)gr * ld + gc : g, ok);
    }
  }
}

template <int BM_, int BN_, int BK_, int WARPS_M_, int WARPS_N_, int STAGES_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int STAGES = STAGES_;
  static constexpr int NT = 32 * WARPS_M * WARPS_N;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static_assert(BK % 4 == 0, "BK multiple of 4");
};

// Accumulator fragment set of one warp.
template <class Cfg>
struct Acc {
  double v[Cfg::FM][Cfg::FN][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < Cfg::FM; i++)
#pragma unroll
      for (int j = 0; j < Cfg::FN; j++) v[i][j][0] = v[i][j][1] = 0.0;
  }
};

// One BK-deep step of tensor-core MMAs over a staged tile.
template <class Cfg, class L>
__device__ __forceinline__ void mma_stage(Acc<Cfg>& acc, const double* sA, const double* sB, int wm, int wn, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int kk = 0; kk < Cfg::BK; kk += 4) {
    double a[Cfg::FM], b[Cfg::FN];
#pragma unroll
    for (int i = 0; i < Cfg::FM; i++) a[i] = sA[L::a_off(wm * Cfg::WTM + i * 8 + g, kk + t)];
#pragma unroll
    for (int j = 0; j < Cfg::FN; j++) b[j] = sB[L::b_off(kk + t, wn * Cfg::WTN + j * 8 + g)];
#pragma unroll
    for (int i = 0; i < Cfg::FM; i++)
#pragma unroll
      for (int j = 0; j < Cfg::FN; j++) dmma884(acc.v[i][j][0], acc.v[i][j][1], a[i], b[j]);
  }
}

// Visit every accumulator element: f(row_in_tile, col_in_tile, value)
template <class Cfg, class F>
__device__ __forceinline__ void for_each_acc(const Acc<Cfg>& acc, int wm, int wn, int lane, F&& f) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < Cfg::FM; i++)
#pragma unroll
    for (int j = 0; j < Cfg::FN; j++) {
      int r = wm * Cfg::WTM + i * 8 + g;
      int c = wn * Cfg::WTN + j * 8 + 2 * t;
      f(r, c, acc.v[i][j][0]);
      f(r, c + 1, acc.v[i][j][1]);
    }
}

}  // namespace tvk
