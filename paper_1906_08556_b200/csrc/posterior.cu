// Batched SPD factor / inverse / solve for the i-vector posterior (tvm.py:183-215) and the
// T update (tvm.py:317-334), on packed-lower D x D matrices (D = 400 at the configs).
//
// One CTA (8 warps) per SM, persistent over the batch, one matrix at a time, factored IN PLACE so
// that the 148 resident matrices (148 x 642 KB) stay L2-resident.  Every O(D^3) part is a
// 32x32x32 tile product on the FP64 tensor pipe (DMMA.8x8x4), fragments loaded from L2:
//   potrf : 32x32 diagonal block by one warp in shared memory, panel TRSM row-parallel,
//           trailing SYRK tile-parallel;
//   trtri : Y = R^-1 row block by row block, T_IJ = sum_K R_IK Y_KJ staged in shared memory;
//   phi   : phi = Y^T (Y b) (two triangular mat-vecs: L^-1 b without a sequential solve);
//   lauum : M = Y^T Y (+ phi phi^T) row block by row block, in place (diagonal tile staged),
//           i.e. the packed moment the A-accumulation GEMM consumes (tvm.py:298-301).
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"
#include "spd_small.cuh"
#include "tc.cuh"

namespace tvk {

constexpr int PT = 256;  // threads per CTA (8 warps), one CTA per SM
constexpr int NW = PT / 32;
constexpr int NB = 32;   // panel / tile width
constexpr int kPosteriorMaxD = 768;

struct Opnd {
  const double* p;
  int64_t ld;  // dense leading dimension (packed_n == 0)
  int n;       // packed order (> 0) or dense rows
  int ncols;   // dense cols
  int r0, c0;
  bool packed, trans;
  bool sym;  // packed symmetric: (r, c) with c > r reads (c, r)
};

__device__ __forceinline__ Opnd packed_op(const double* p, int n, int r0, int c0, bool trans) {
  Opnd o;
  o.p = p;
  o.ld = 0;
  o.n = n;
  o.ncols = n;
  o.r0 = r0;
  o.c0 = c0;
  o.packed = true;
  o.trans = trans;
  o.sym = false;
  return o;
}
__device__ __forceinline__ Opnd dense_op(const double* p, int64_t ld, int nr, int nc, int r0, int c0, bool trans) {
  Opnd o;
  o.p = p;
  o.ld = ld;
  o.n = nr;
  o.ncols = nc;
  o.r0 = r0;
  o.c0 = c0;
  o.packed = false;
  o.trans = trans;
  o.sym = false;
  return o;
}

__device__ __forceinline__ double ld_elem(const Opnd& o, int r, int c) {
  if (o.packed) {
    if (o.sym && c > r) {
      int t = r;
      r = c;
      c = t;
    }
    return (r < o.n && c <= r && c >= 0) ? o.p[packed_index(r, c)] : 0.0;
  }
  return (r < o.n && c < o.ncols && r >= 0 && c >= 0) ? o.p[(int64_t)r * o.ld + c] : 0.0;
}

// acc(32x32) += A(32 x klen) * B(klen x 32); A logical (i,k), B logical (k,j).
__device__ __forceinline__ void tile_mma(double (&acc)[4][4][2], const Opnd& A, const Opnd& B, int klen, int lane) {
  const int g = lane >> 2, t = lane & 3;
  // four k-steps of fragments in flight (32 loads) per 64 MMAs
#pragma unroll 1
  for (int ks0 = 0; ks0 < 8; ks0 += 4) {
    double a[4][4], b[4][4];
#pragma unroll
    for (int h = 0; h < 4; h++) {
      int k = (ks0 + h) * 4 + t;
      bool kin = k < klen;
#pragma unroll
      for (int f = 0; f < 4; f++) {
        int i = f * 8 + g;
        double av = 0.0, bv = 0.0;
        if (kin) {
          av = A.trans ? ld_elem(A, A.r0 + k, A.c0 + i) : ld_elem(A, A.r0 + i, A.c0 + k);
          bv = B.trans ? ld_elem(B, B.r0 + i, B.c0 + k) : ld_elem(B, B.r0 + k, B.c0 + i);
        }
        a[h][f] = av;
        b[h][f] = bv;
      }
    }
#pragma unroll
    for (int h = 0; h < 4; h++)
#pragma unroll
      for (int fi = 0; fi < 4; fi++)
#pragma unroll
        for (int fj = 0; fj < 4; fj++) dmma884(acc[fi][fj][0], acc[fi][fj][1], a[h][fi], b[h][fj]);
  }
}

__device__ __forceinline__ void zero_acc(double (&acc)[4][4][2]) {
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
}

template <class Fn>
__device__ __forceinline__ void acc_foreach(const double (&acc)[4][4][2], int lane, Fn&& fn) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int fi = 0; fi < 4; fi++)
#pragma unroll
    for (int fj = 0; fj < 4; fj++) {
      fn(fi * 8 + g, fj * 8 + 2 * t, acc[fi][fj][0]);
      fn(fi * 8 + g, fj * 8 + 2 * t + 1, acc[fi][fj][1]);
    }
}

// ------------------------------------------------------------------ blocked Cholesky (in place, packed)

// n x n (n <= 32) lower Cholesky of the shared-memory block a (row stride n) by warp 0 alone.
__device__ void warp_cholesky(double* a, int n, int* bad, int lane) {
  for (int k = 0; k < n; k++) {
    if (lane == 0) {
      double d = a[k * n + k];
      if (!(d > 0.0)) *bad = 1;
      else a[k * n + k] = sqrt(d);
    }
    __syncwarp();
    if (*bad) return;
    const double piv = a[k * n + k];
    if (lane > k && lane < n) a[lane * n + k] /= piv;
    __syncwarp();
    if (lane > k && lane < n) {
      const double lik = a[lane * n + k];
      for (int j = k + 1; j <= lane; j++) a[lane * n + j] -= lik * a[j * n + k];
    }
    __syncwarp();
  }
}

// Returns false (uniformly across the CTA) if the matrix is not positive definite.
__device__ bool packed_cholesky(double* P, int n, double* sdiag /* NB*NB */, int* bad) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = (n + NB - 1) / NB;
  for (int kb = 0; kb < nblk; kb++) {
    const int k0 = kb * NB, kw = min(NB, n - k0);
    for (int idx = tid; idx < kw * kw; idx += PT) {
      int r = idx / kw, c = idx % kw;
      sdiag[idx] = c <= r ? P[packed_index(k0 + r, k0 + c)] : 0.0;
    }
    if (tid == 0) *bad = 0;
    __syncthreads();
    if (warp == 0) warp_cholesky(sdiag, kw, bad, lane);
    __syncthreads();
    if (*bad) return false;
    for (int idx = tid; idx < kw * kw; idx += PT) {
      int r = idx / kw, c = idx % kw;
      if (c <= r) P[packed_index(k0 + r, k0 + c)] = sdiag[idx];
    }
    // panel: rows below, X = W R_kk^-T (row-parallel forward substitution)
    for (int i = k0 + kw + tid; i < n; i += PT) {
      double* row = P + packed_index(i, k0);
      double x[NB];
#pragma unroll
      for (int j = 0; j < NB; j++) x[j] = j < kw ? row[j] : 0.0;
#pragma unroll
      for (int j = 0; j < NB; j++) {
        if (j < kw) {
          double s = x[j];
#pragma unroll
          for (int l = 0; l < j; l++) s -= x[l] * sdiag[j * kw + l];
          x[j] = s / sdiag[j * kw + j];
        }
      }
#pragma unroll
      for (int j = 0; j < NB; j++)
        if (j < kw) row[j] = x[j];
    }
    __syncthreads();
    // trailing update of the lower triangle: C_IJ -= P_I P_J^T, tiles I >= J > kb
    const int nt = nblk - kb - 1;
    const int ntiles = nt * (nt + 1) / 2;
    for (int tix = warp; tix < ntiles; tix += NW) {
      int I = 0, base = 0;
      while (base + I + 1 <= tix) {
        base += I + 1;
        I++;
      }
      int J = tix - base;
      const int i0 = k0 + kw + I * NB, j0 = k0 + kw + J * NB;
      double acc[4][4][2];
      zero_acc(acc);
      tile_mma(acc, packed_op(P, n, i0, k0, false), packed_op(P, n, j0, k0, true), kw, lane);
      acc_foreach(acc, lane, [&](int r, int c, double v) {
        int gi = i0 + r, gj = j0 + c;
        if (gi < n && gj <= gi) P[packed_index(gi, gj)] -= v;
      });
    }
    __syncthreads();
  }
  return true;
}

// ------------------------------------------------------------------ SPD inverse (trtri + lauum)

__host__ __device__ inline int tmp_ld(int D) { return ((D + 11) / 16) * 16 + 4; }  // == 4 (mod 16)

// After packed_cholesky (L holds R): overwrite L with Y = R^-1 (row block by row block:
// Y_IJ = -Y_II sum_{K=J}^{I-1} R_IK Y_KJ with T_IJ staged in the shared `tmp` [NB][ldt]).
__device__ void packed_trtri(double* L, int D, double* tmp, int ldt, double* sdiag, double* sinv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = (D + NB - 1) / NB;
  for (int I = 0; I < nblk; I++) {
    const int i0 = I * NB, iw = min(NB, D - i0);
    for (int idx = tid; idx < NB * NB; idx += PT) {
      int r = idx / NB, c = idx % NB;
      sdiag[idx] = (r < iw && c <= r) ? L[packed_index(i0 + r, i0 + c)] : (r == c ? 1.0 : 0.0);
    }
    __syncthreads();
    if (warp == NW - 1) {  // Y_II = R_II^-1, lane = column (forward substitution)
      const int j = lane;
      for (int r = 0; r < j; r++) sinv[r * NB + j] = 0.0;
      sinv[j * NB + j] = 1.0 / sdiag[j * NB + j];
      for (int r = j + 1; r < NB; r++) {
        double acc = 0.0;
        for (int k = j; k < r; k++) acc += sdiag[r * NB + k] * sinv[k * NB + j];
        sinv[r * NB + j] = -acc / sdiag[r * NB + r];
      }
    }
    for (int J = warp; J < I; J += NW - 1) {  // T_IJ = sum_{K=J}^{I-1} R_IK Y_KJ  (warps 0..NW-2)
      if (warp == NW - 1) break;
      double acc[4][4][2];
      zero_acc(acc);
      for (int K = J; K < I; K++)
        tile_mma(acc, packed_op(L, D, i0, K * NB, false), packed_op(L, D, K * NB, J * NB, false), NB, lane);
      acc_foreach(acc, lane, [&](int r, int c, double val) { tmp[r * ldt + J * NB + c] = val; });
    }
    __syncthreads();
    for (int J = warp; J < I; J += NW) {  // Y_IJ = -Y_II T_IJ (overwrites R_IJ)
      double acc[4][4][2];
      zero_acc(acc);
      tile_mma(acc, dense_op(sinv, NB, NB, NB, 0, 0, false), dense_op(tmp, ldt, NB, ldt, 0, J * NB, false), NB, lane);
      acc_foreach(acc, lane, [&](int r, int c, double val) {
        if (r < iw) L[packed_index(i0 + r, J * NB + c)] = -val;
      });
    }
    for (int idx = tid; idx < iw * iw; idx += PT) {
      int r = idx / iw, c = idx % iw;
      if (c <= r) L[packed_index(i0 + r, i0 + c)] = sinv[r * NB + c];
    }
    __syncthreads();
  }
}

// M = Y^T Y (+ v v^T) written over Y (M may alias L): row block I ascending; the off-diagonal tiles
// of row I only read rows K >= I and their own slot, the diagonal tile (which every tile of the
// row reads through the K = I term) is staged in `dtmp` and stored after the row completes.
__device__ void packed_lauum(double* L, int D, double* M, const double* v, double* dtmp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = (D + NB - 1) / NB;
  for (int I = 0; I < nblk; I++) {
    for (int J = warp; J <= I; J += NW) {
      double acc[4][4][2];
      zero_acc(acc);
      for (int K = I; K < nblk; K++)
        tile_mma(acc, packed_op(L, D, K * NB, I * NB, true), packed_op(L, D, K * NB, J * NB, false),
                 min(NB, D - K * NB), lane);
      acc_foreach(acc, lane, [&](int r, int c, double val) {
        int gi = I * NB + r, gj = J * NB + c;
        if (gi >= D || gj > gi) return;
        double out = v ? val + v[gi] * v[gj] : val;
        if (J == I) dtmp[r * NB + c] = out;
        else M[packed_index(gi, gj)] = out;
      });
    }
    __syncthreads();
    for (int idx = tid; idx < NB * NB; idx += PT) {
      int r = idx / NB, c = idx % NB, gi = I * NB + r, gj = I * NB + c;
      if (gi < D && c <= r) M[packed_index(gi, gj)] = dtmp[idx];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ posterior kernel

__global__ void __launch_bounds__(PT, 1) posterior_kernel(double* lpk, const double* bvec, int U, int D, int flags,
                                                          double* phi_out, double* mpk, double* logdet_out,
                                                          double* bphi_out, int32_t* status) {
  extern __shared__ __align__(16) double sm[];
  const int ldt = tmp_ld(D);
  double* tmp = sm;                 // [NB][ldt]
  double* sdiag = tmp + NB * ldt;   // [NB*NB]
  double* sinv = sdiag + NB * NB;   // [NB*NB]
  double* dtmp = sinv + NB * NB;    // [NB*NB]
  double* vb = dtmp + NB * NB;      // [D] b, then phi
  double* vz = vb + D;              // [D] Y b
  double* vp = vz + D;              // [D] phi
  __shared__ int bad;
  __shared__ double red;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t P = packed_size(D);

  for (int u = blockIdx.x; u < U; u += gridDim.x) {
    double* L = lpk + (int64_t)u * P;
    if (flags & TVK_POST_ADD_IDENTITY)
      for (int i = tid; i < D; i += PT) L[packed_index(i, i)] += 1.0;
    __syncthreads();
    if (!packed_cholesky(L, D, sdiag, &bad)) {
      if (tid == 0 && status) status[u] = TVK_ITEM_NOT_SPD;
      continue;
    }
    if (tid == 0 && status) status[u] = TVK_ITEM_OK;
    if (warp == 0) {
      double s = 0.0;
      for (int i = lane; i < D; i += 32) s += log(L[packed_index(i, i)]);
      s = warp_sum(s);
      if (lane == 0) red = 2.0 * s;
    }
    for (int i = tid; i < D; i += PT) vb[i] = bvec ? bvec[(int64_t)u * D + i] : 0.0;
    packed_trtri(L, D, tmp, ldt, sdiag, sinv);  // L <- Y = R^-1 (syncs inside)
    // phi = Y^T (Y b): z_i = sum_{j<=i} Y_ij b_j (rows), phi_j = sum_{i>=j} Y_ij z_i (columns)
    for (int i = warp; i < D; i += NW) {
      const double* row = L + packed_index(i, 0);
      double s = 0.0;
      for (int j = lane; j <= i; j += 32) s += row[j] * vb[j];
      s = warp_sum(s);
      if (lane == 0) vz[i] = s;
    }
    __syncthreads();
    for (int j = tid; j < D; j += PT) {
      double s = 0.0;
      for (int i = j; i < D; i++) s += L[packed_index(i, j)] * vz[i];
      if (phi_out) phi_out[(int64_t)u * D + j] = s;
      vp[j] = s;
    }
    __syncthreads();
    if (warp == 0 && (bphi_out || logdet_out)) {
      double s = 0.0;
      for (int i = lane; i < D; i += 32) s += vb[i] * vp[i];
      s = warp_sum(s);
      if (lane == 0) {
        if (bphi_out) bphi_out[u] = s;
        if (logdet_out) logdet_out[u] = red;
      }
    }
    if (mpk == nullptr) continue;
    const bool moment = (flags & TVK_POST_MOMENT) && bvec;
    packed_lauum(L, D, mpk + (int64_t)u * P, moment ? vp : nullptr, dtmp);
  }
}

// ------------------------------------------------------------------ row solve (update_T)

// X_c = B_c A_c^-1 via the explicit SPD inverse (Cholesky, trtri, lauum in place on a scratch copy)
// and a tile GEMM against the symmetric packed inverse: all O(D^3) work on the tensor pipe.
__global__ void __launch_bounds__(PT, 1) spd_solve_rows_kernel(const double* apk, const double* bmat, int batch,
                                                               int D, int R, const int32_t* skip, double* x,
                                                               int32_t* status, double* scratch) {
  extern __shared__ __align__(16) double sm[];
  const int ldt = tmp_ld(D);
  double* tmp = sm;
  double* sdiag = tmp + NB * ldt;
  double* sinv = sdiag + NB * NB;
  double* dtmp = sinv + NB * NB;
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t P = packed_size(D);
  double* W = scratch + (int64_t)blockIdx.x * P;
  const int nblk = (D + NB - 1) / NB, rblk = (R + NB - 1) / NB;
  for (int c = blockIdx.x; c < batch; c += gridDim.x) {
    if (skip && skip[c]) {
      if (tid == 0 && status) status[c] = TVK_ITEM_SKIPPED;
      continue;
    }
    const double* A = apk + (int64_t)c * P;
    for (int64_t i = tid; i < P; i += PT) W[i] = A[i];
    __syncthreads();
    if (!packed_cholesky(W, D, sdiag, &bad)) {
      if (tid == 0 && status) status[c] = TVK_ITEM_NOT_SPD;
      continue;
    }
    if (tid == 0 && status) status[c] = TVK_ITEM_OK;
    packed_trtri(W, D, tmp, ldt, sdiag, sinv);
    packed_lauum(W, D, W, nullptr, dtmp);  // W <- A^-1 (packed)
    const double* B = bmat + (int64_t)c * R * D;
    double* X = x + (int64_t)c * R * D;
    for (int tix = warp; tix < rblk * nblk; tix += NW) {
      const int I = tix / nblk, J = tix % nblk;
      double acc[4][4][2];
      zero_acc(acc);
      for (int K = 0; K < nblk; K++) {
        Opnd Bo = dense_op(B, D, R, D, I * NB, K * NB, false);
        Opnd Ao = packed_op(W, D, K * NB, J * NB, false);
        Ao.sym = true;
        tile_mma(acc, Bo, Ao, min(NB, D - K * NB), lane);
      }
      acc_foreach(acc, lane, [&](int r, int cc, double val) {
        int gi = I * NB + r, gj = J * NB + cc;
        if (gi < R && gj < D) X[(int64_t)gi * D + gj] = val;
      });
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ block sweep (EM posterior moments)
//
// The E-step needs, per utterance, M = L^-1 + phi phi^T with phi = L^-1 b and log|L| (tvm.py:195-200).
// sweep_posterior_kernel obtains all three from ONE pass of the symmetric block sweep operator over the
// bordered matrix [[L, b], [b^T, 0]]: sweeping the 32-wide pivot blocks k = 0..nb-1 in turn
//   P = A_kk,  A_kk <- -P^-1,  B_i = A_ik P^-1,  A_ij <- A_ij - B_i A_jk^T (i, j != k),  A_ik <- B_i
// leaves [[-L^-1, L^-1 b], [b^T L^-1, -b^T L^-1 b]] (the sweep-operator identity), and
// log|L| = sum of the log pivots (the Schur complements are SPD exactly when L is, so a non-positive
// pivot is the not-SPD signal, like a failed Cholesky).  Compared with potrf + trtri + lauum (the
// posterior_kernel below, still used when only phi and log|L| are needed) every step has the same
// shape -- 78 independent 32x32x32 tile updates at D = 400 -- so 16 warps stay busy with no
// triangular dependency chains, and every operand of a step comes from shared memory:
//   pa = the old column panel A_:k (D x 32, pivot block inverted in place to -P^-1),
//   pb = the new column panel B_:k;
// only the updated tile itself travels to and from L2 (read-modify-write in the output buffer, which
// may alias the input).  The last step writes M = -A + phi phi^T (or Phi) directly.
// sw::CL = 2 would let two CTAs (a cluster, two SMs) share one matrix: both load the panels and compute
// B, the bordered row and the look-ahead pivot redundantly, split the tile updates, and order the
// global tiles with one cluster barrier per step.  74 matrices in flight (47 MB at D = 400) then stay
// L2-resident (DRAM 0.66 GB read + 0.76 GB written per 1024 matrices, vs 0.86 + 7.3 GB with 148
// single-SM matrices), but the duplicated per-step work made it 1.4x slower (8.3 vs 5.9 ms), so one
// CTA per matrix is the default.
#ifdef TVK_SWEEP_PROF
__device__ unsigned long long g_sweep_prof[8];
#define SWP(i)                                                              \
  do {                                                                      \
    if (threadIdx.x == 0) {                                                 \
      const long long t_ = clock64();                                       \
      atomicAdd(&g_sweep_prof[i], (unsigned long long)(t_ - swp_prev));     \
      swp_prev = t_;                                                        \
    }                                                                       \
  } while (0)
#else
#define SWP(i) \
  do {         \
  } while (0)
#endif
namespace sw {
// internal flag (not in the C ABI): no Phi / M output -- phi and log|L| only.  The sweep then runs as
// block elimination: only the trailing Schur complement (i, j > k) is updated (~1/3 of the tile
// updates at D = 400), column k below the pivot keeps B_i, the bordered column yields
// z_k = P_k^-1 y_k, and phi = A^-1 b follows by block back substitution (phi_k = z_k - sum_{i>k} B_i' phi_i).
constexpr int PHI_ONLY = 1 << 8;
constexpr int NT = 512;  // 16 warps, one CTA per SM
constexpr int CL = 1;    // CTAs (SMs) per matrix (2 = cluster pair: no L2 thrash but slower, see below)
constexpr int NWARP = NT / 32;
constexpr int MAXB = 13;  // D <= 416: two 416 x 32 FP64 panels fill 208 KB of shared memory
constexpr int TILE = 1024;
// bank swizzle: conflict-free for DMMA fragments (rows 8f+g, cols 4ks+t), for one column across 16
// consecutive rows (transposed panel loads / write-back / bordered row) and for one row across lanes
__device__ __forceinline__ int sidx(int r, int c) { return r * 32 + (c ^ (((r & 3) << 2) | ((r >> 2) & 3))); }
constexpr size_t smem_bytes() { return sizeof(double) * (2 * MAXB * TILE + TILE + MAXB * 32 + 8 + 32); }
}  // namespace sw

// Old column k of the symmetric matrix held in row-major packed storage -> pa (swizzled 32x32 tiles).
// With `pivot` (the look-ahead result, already -P^-1) the pivot block is copied from it instead.
__device__ __forceinline__ void sweep_load_panel(const double* S, int D, int nb, int k, double* pa, bool add_identity,
                                                 const double* pivot, bool below_only = false) {
  const int tid = threadIdx.x;
  const int k0 = k * 32, kw = min(32, D - k0);
  // rows above the pivot block: element (R, c) = S(k0 + c, R), R fastest (contiguous in row k0 + c);
  // the elimination (phi-only) mode never reads them
  for (int e = tid; e < (below_only ? 0 : k0 * kw); e += sw::NT) {
    const int c = e / k0, R = e - c * k0;
    cp_async8(&pa[(R >> 5) * sw::TILE + sw::sidx(R & 31, c)], S + packed_index(k0 + c, R), true);
  }
  for (int e = tid; e < (below_only ? 0 : k0 * (32 - kw)); e += sw::NT) {  // columns past D (last block only)
    const int c = kw + e / k0, R = e % k0;
    pa[(R >> 5) * sw::TILE + sw::sidx(R & 31, c)] = 0.0;
  }
  // pivot block and rows below: element (R, c) = S(R, k0 + c) for R >= k0 + c, c fastest
  const int rows = nb * 32 - k0;
  for (int e = tid; e < rows * 32; e += sw::NT) {
    const int r = e >> 5, c = e & 31, R = k0 + r, Cc = k0 + c;
    double* dst = &pa[(R >> 5) * sw::TILE + sw::sidx(R & 31, c)];
    if (pivot && r < 32) *dst = pivot[sw::sidx(r, c)];
    else if (R >= D || Cc >= D) *dst = (R == Cc) ? 1.0 : 0.0;  // padding: identity pivot, zero rows
    else if (R >= Cc) cp_async8(dst, S + packed_index(R, Cc), true);
    else cp_async8(dst, S + packed_index(Cc, R), true);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (add_identity && tid < kw) pa[k * sw::TILE + sw::sidx(tid, tid)] += 1.0;
  __syncthreads();
}

// In-place scalar sweep of the 32x32 pivot block by ONE warp (lane c holds column c in registers;
// row p is broadcast through shared memory): pk <- -P^-1.  Returns the sum of log pivots through
// *ldet and sets *bad when a pivot is not positive (the block is then garbage, the caller stops).
__device__ __forceinline__ void sweep_pivot_warp(double* pk, double* rowbuf, double* ldet, int* bad, int lane) {
  double a[32];
#pragma unroll
  for (int r = 0; r < 32; r++) a[r] = pk[sw::sidx(r, lane)];
  double piv = 1.0;
#pragma unroll
  for (int p = 0; p < 32; p++) {
    rowbuf[lane] = a[p];  // row p == column p (symmetric)
    __syncwarp();
    const double d = rowbuf[p];
    const double inv = 1.0 / d;
    const double apc = a[p] * inv;
#pragma unroll
    for (int r = 0; r < 32; r++) {
      if (r == p) continue;
      const double arp = rowbuf[r];
      a[r] = (lane == p) ? arp * inv : fma(-arp, apc, a[r]);
    }
    a[p] = (lane == p) ? -inv : apc;
    if (lane == p) piv = d;
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < 32; r++) pk[sw::sidx(r, lane)] = a[r];
  const double l = warp_sum(log(piv));
  const unsigned nonpos = __ballot_sync(0xffffffffu, !(piv > 0.0));
  if (lane == 0) {
    *ldet += l;
    if (nonpos) *bad = 1;
  }
}

// acc(32x32) += sign * X_i * Y_j^T with X_i, Y_j swizzled 32x32 smem tiles; nfi/nfj/nks limit the
// 8-row fragments and 4-wide k-steps to the live part of a partial last block.
__device__ __forceinline__ void sweep_tile_mma(double (&acc)[4][4][2], const double* X, const double* Y, int nfi,
                                               int nfj, int nks, double sign, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 8; ks++) {
    if (ks >= nks) break;
    double a[4], b[4];
#pragma unroll
    for (int f = 0; f < 4; f++) {
      a[f] = sign * X[sw::sidx(8 * f + g, 4 * ks + t)];
      b[f] = Y[sw::sidx(8 * f + g, 4 * ks + t)];
    }
#pragma unroll
    for (int fi = 0; fi < 4; fi++) {
      if (fi >= nfi) break;
#pragma unroll
      for (int fj = 0; fj < 4; fj++)
        if (fj < nfj) dmma884(acc[fi][fj][0], acc[fi][fj][1], a[fi], b[fj]);
    }
  }
}

__global__ void __launch_bounds__(sw::NT, 1) sweep_posterior_kernel(const double* lpk, double* mpk,
                                                                    const double* bvec, int U, int D, int flags,
                                                                    double* phi_out, double* logdet_out,
                                                                    double* bphi_out, int32_t* status) {
  extern __shared__ __align__(16) double sm[];
  double* pa = sm;                        // [MAXB][1024] old column panel (pivot block -> -P^-1)
  double* pb = pa + sw::MAXB * sw::TILE;  // [MAXB][1024] new column panel B
  double* vr = pb + sw::MAXB * sw::TILE;  // [nb*32 + 1] bordered row (b -> phi), corner at nb*32
  double* bd = vr + sw::MAXB * 32 + 8;    // [32] bordered row of B
  double* pnext = bd + 32;                // [1024] look-ahead pivot: block k+1 after step k, then -P^-1
  __shared__ double rowbuf[32];
  __shared__ int tile_ctr;
  __shared__ int bad;
  __shared__ double ldet;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nb = (D + 31) / 32, ntile = nb * (nb + 1) / 2;
  const int nupd = 2 * ((nb - 1) * nb / 2);  // update half-tiles per step
  const int64_t P = packed_size(D);
  const bool moment = (flags & TVK_POST_MOMENT) && bvec;
  const bool elim = (flags & sw::PHI_ONLY) != 0;
#ifdef TVK_SWEEP_PROF
  long long swp_prev = clock64();
#endif
  const int rank = sw::CL > 1 ? (int)tc::cluster_ctarank() : 0, ncl = gridDim.x / sw::CL;
  for (int u = blockIdx.x / sw::CL; u < U; u += ncl) {
    const double* Lu = lpk + (int64_t)u * P;
    double* Mu = mpk + (int64_t)u * P;
    for (int i = tid; i <= nb * 32; i += sw::NT) vr[i] = (bvec && i < D) ? bvec[(int64_t)u * D + i] : 0.0;
    if (tid == 0) {
      bad = 0;
      ldet = 0.0;
    }
    __syncthreads();
    for (int k = 0; k < nb; k++) {
      const double* S = k == 0 ? Lu : Mu;
      const bool addI = k == 0 && (flags & TVK_POST_ADD_IDENTITY);
      const bool last = k == nb - 1;
      const int k0 = k * 32;
      const int nks = min(8, (D - k0 + 3) / 4);
      SWP(5);
      if (bad) break;  // uniform (a failed look-ahead pivot of step k-1)
      sweep_load_panel(S, D, nb, k, pa, addI, k > 0 ? pnext : nullptr, elim);
      SWP(0);
      double* pk = pa + k * sw::TILE;
      if (k == 0) {  // later pivots are swept ahead, during the previous step's tile updates
        if (warp == 0) sweep_pivot_warp(pk, rowbuf, &ldet, &bad, lane);
        __syncthreads();
      }
      SWP(1);
      if (bad) break;  // uniform
      // B_i = A_old_i P^-1 = -(pa_i pk) for the other blocks; the bordered row by the last warp
      for (int i = warp; i < nb; i += sw::NWARP) {
        if (i == k || (elim && i < k)) continue;
        double acc[4][4][2];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
        const int nfi = min(4, (D - i * 32 + 7) / 8);
        if (nfi == 4 && nks == 8)
          sweep_tile_mma(acc, pa + i * sw::TILE, pk, 4, 4, 8, -1.0, lane);
        else
          sweep_tile_mma(acc, pa + i * sw::TILE, pk, nfi, 4, nks, -1.0, lane);
        double* dst = pb + i * sw::TILE;
#pragma unroll
        for (int fi = 0; fi < 4; fi++)
#pragma unroll
          for (int fj = 0; fj < 4; fj++) {
            dst[sw::sidx(8 * fi + g, 8 * fj + 2 * t)] = acc[fi][fj][0];
            dst[sw::sidx(8 * fi + g, 8 * fj + 2 * t + 1)] = acc[fi][fj][1];
          }
      }
      if (tid == 0) tile_ctr = 0;  // read after the barrier below
      if (bvec && warp == sw::NWARP - 1) {
        // bd = b_k P^-1 = -(b_k . pk); corner -= bd . b_k (before b_k is replaced by bd)
        double s = 0.0;
        for (int c = 0; c < 32; c++) s -= vr[k0 + c] * pk[sw::sidx(c, lane)];
        bd[lane] = s;
        const double cs = warp_sum(s * vr[k0 + lane]);
        if (lane == 0) vr[nb * 32] -= cs;
      }
      __syncthreads();
      SWP(2);
      if (bvec) {  // vr_j -= bd . A_old(j, k-block) outside the pivot block; vr_k <- bd
        // thread per row, column order rotated by the row so the 16 rows of a half-warp hit 16 banks
        for (int j = tid; j < nb * 32; j += sw::NT) {
          const int jb = j >> 5;
          if (jb == k) {
            vr[j] = bd[j - k0];
            continue;
          }
          if (elim && jb < k) continue;  // z_j of an eliminated block stays (back substitution)
          const double* row = pa + jb * sw::TILE;
          double s = 0.0;
#pragma unroll 8
          for (int c = 0; c < 32; c++) s = fma(bd[c], row[sw::sidx(j & 31, c)], s);
          vr[j] -= s;
        }
      }
      if (last) __syncthreads();  // phi final before the M epilogue reads it
      SWP(3);
      // Tile updates A_ij -= B_i A_old_j^T (i, j != k), whole 32x32 tiles handed out by a shared-memory
      // counter (dynamic balance).  Look-ahead: warp 0 first updates the next pivot block (k+1, k+1),
      // keeps it in pnext and sweeps it (-P_{k+1}^-1 is ready when the next step starts), then joins.
      const bool ahead = !last;
      // reduced index of tile (k+1, k+1): full sweep over all (i, j) != k; elimination over i >= j > k only
      const int skip = ahead ? (elim ? 0 : k * (k + 1) / 2 + k) : -1;
      const int ntask = (elim ? (nb - k - 1) * (nb - k) / 2 : (nb - 1) * nb / 2) - (ahead ? 1 : 0);
      if (ahead && warp == 0) {
        const int I0 = k0 + 32;
        const int nf = min(4, (D - I0 + 7) / 8);
        double acc[4][4][2];
#pragma unroll
        for (int fi = 0; fi < 4; fi++)
#pragma unroll
          for (int fj = 0; fj < 4; fj++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int r = 8 * fi + g, c = 8 * fj + 2 * t + h, R = I0 + r, Cc = I0 + c;
              double x = 0.0;
              if (R < D && Cc <= R) x = S[packed_index(R, Cc)] + ((addI && R == Cc) ? 1.0 : 0.0);
              acc[fi][fj][h] = x;
            }
        sweep_tile_mma(acc, pb + (k + 1) * sw::TILE, pa + (k + 1) * sw::TILE, nf, nf, nks, -1.0, lane);
#pragma unroll
        for (int fi = 0; fi < 4; fi++)
#pragma unroll
          for (int fj = 0; fj < 4; fj++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int r = 8 * fi + g, c = 8 * fj + 2 * t + h, R = I0 + r, Cc = I0 + c;
              if (c > r) continue;
              const double v = acc[fi][fj][h];
              if (R < D) {
                if (rank == 0) Mu[packed_index(R, Cc)] = v;
                pnext[sw::sidx(r, c)] = v;
                pnext[sw::sidx(c, r)] = v;
              } else {  // padding of a partial last block: identity pivot
                pnext[sw::sidx(r, c)] = (r == c) ? 1.0 : 0.0;
                pnext[sw::sidx(c, r)] = (r == c) ? 1.0 : 0.0;
              }
            }
        __syncwarp();
        sweep_pivot_warp(pnext, rowbuf, &ldet, &bad, lane);
      }
      // column-k write-back: (i,k) <- B_i, (k,j) <- B_j^T, (k,k) <- -P^-1
      for (int i = ahead ? warp - 1 : warp; i < nb && (!ahead || warp > 0); i += ahead ? sw::NWARP - 1 : sw::NWARP) {
        if (i % sw::CL != rank) continue;
        if (elim && i <= k) continue;  // only B_i below the pivot is kept (back substitution)
        const int I0 = i * 32;
        for (int e = lane; e < 1024; e += 32) {
          const int r = e >> 5, c = e & 31;
          int R, Cc;
          double v;
          if (i > k) {
            R = I0 + r, Cc = k0 + c;
            v = pb[i * sw::TILE + sw::sidx(r, c)];
          } else if (i < k) {
            R = k0 + r, Cc = I0 + c;
            v = pb[i * sw::TILE + sw::sidx(c, r)];
          } else {
            if (c > r) continue;
            R = k0 + r, Cc = k0 + c;
            v = pk[sw::sidx(r, c)];
          }
          if (R >= D || Cc >= D) continue;
          if (last && !elim) v = -v + (moment ? vr[R] * vr[Cc] : 0.0);
          Mu[packed_index(R, Cc)] = v;
        }
      }
      for (;;) {
        int m = 0;
        if (lane == 0) m = atomicAdd(&tile_ctr, 1);
        m = __shfl_sync(0xffffffffu, m, 0) * sw::CL + rank;
        if (m >= ntask) break;
        if (m >= skip && skip >= 0) m++;
        int i = (int)((sqrt(8.0 * m + 1.0) - 1.0) * 0.5);
        while ((i + 1) * (i + 2) / 2 <= m) i++;
        while (i * (i + 1) / 2 > m) i--;
        int j = m - i * (i + 1) / 2;
        if (elim) {  // trailing block (i, j) of the Schur complement, i >= j > k
          i += k + 1;
          j += k + 1;
        } else {
          i += i >= k;
          j += j >= k;
        }
        const int I0 = i * 32, J0 = j * 32;
        const bool dg = i == j;
        // element (R, J0 + 8fj + 2t + h) of row R = I0 + 8fi + g sits at rowoff[fi] + 8fj + h
        int64_t rowoff[4];
#pragma unroll
        for (int fi = 0; fi < 4; fi++) rowoff[fi] = packed_index(I0 + 8 * fi + g, J0 + 2 * t);
        double acc[4][4][2];
#pragma unroll
        for (int fi = 0; fi < 4; fi++) {
          const double* rp = S + rowoff[fi];
#pragma unroll
          for (int fj = 0; fj < 4; fj++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int R = I0 + 8 * fi + g, Cc = J0 + 8 * fj + 2 * t + h;
              double x = 0.0;
              if (R < D && Cc < D && (!dg || Cc <= R)) x = rp[8 * fj + h];
              acc[fi][fj][h] = x;
            }
        }
        if (addI && dg) {  // L = Lpk + I (first step only)
#pragma unroll
          for (int fi = 0; fi < 4; fi++)
#pragma unroll
            for (int fj = 0; fj < 4; fj++)
#pragma unroll
              for (int h = 0; h < 2; h++)
                if (8 * fi + g == 8 * fj + 2 * t + h) acc[fi][fj][h] += 1.0;
        }
        const int nfi = min(4, (D - I0 + 7) / 8), nfj = min(4, (D - J0 + 7) / 8);
        if (nfi == 4 && nfj == 4 && nks == 8)
          sweep_tile_mma(acc, pb + i * sw::TILE, pa + j * sw::TILE, 4, 4, 8, -1.0, lane);
        else
          sweep_tile_mma(acc, pb + i * sw::TILE, pa + j * sw::TILE, nfi, nfj, nks, -1.0, lane);
#pragma unroll
        for (int fi = 0; fi < 4; fi++) {
          double* wp = Mu + rowoff[fi];
#pragma unroll
          for (int fj = 0; fj < 4; fj++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int R = I0 + 8 * fi + g, Cc = J0 + 8 * fj + 2 * t + h;
              if (R >= D || Cc >= D || (dg && Cc > R)) continue;
              double v = acc[fi][fj][h];
              if (last && !elim) v = -v + (moment ? vr[R] * vr[Cc] : 0.0);
              wp[8 * fj + h] = v;
            }
        }
      }
      (void)ntile;
      if (sw::CL > 1) tc::cluster_sync();  // both CTAs' tiles are in global memory before the next panel load
      else __syncthreads();
      SWP(4);
    }
    if (elim && !bad) {
      // block back substitution phi_k = z_k - sum_{R beyond block k} B(R, k0 + lane) phi(R): warps take
      // rows R (coalesced 256-byte reads of the packed rows), partial sums folded in fixed warp order
      double* part = pa;  // [NWARP][32] scratch (the panels are free after the last step)
      for (int k = nb - 1; k >= 0; k--) {
        const int k0 = k * 32;
        double sacc = 0.0;
        if (k0 + lane < D)
          for (int R = k0 + 32 + warp; R < D; R += sw::NWARP)
            sacc = fma(Mu[packed_index(R, k0 + lane)], vr[R], sacc);
        part[warp * 32 + lane] = sacc;
        __syncthreads();
        if (warp == 0 && k0 + lane < D) {
          double t = 0.0;
          for (int w2 = 0; w2 < sw::NWARP; w2++) t += part[w2 * 32 + lane];
          vr[k0 + lane] -= t;
        }
        __syncthreads();
      }
    }
    if (rank == 0) {
      if (tid == 0 && status) status[u] = bad ? TVK_ITEM_NOT_SPD : TVK_ITEM_OK;
      if (!bad) {
        for (int i = tid; i < D; i += sw::NT)
          if (phi_out) phi_out[(int64_t)u * D + i] = vr[i];
        if (tid == 0) {
          if (logdet_out) logdet_out[u] = ldet;
          if (bphi_out) bphi_out[u] = -vr[nb * 32];
        }
      }
    }
    if (sw::CL > 1) tc::cluster_sync();  // a failed matrix left its step loop early: resynchronize
    else __syncthreads();
  }
}

static int resident_ctas(int items) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return items < sms ? items : sms;
}

static size_t kernel_smem(int D) { return sizeof(double) * ((size_t)NB * tmp_ld(D) + 3 * NB * NB + 3 * (size_t)D); }

}  // namespace tvk

using namespace tvk;

extern "C" int64_t tvk_posterior_workspace_bytes(int D, int batch) {
  // tvk_spd_solve_rows: one packed matrix per resident CTA; tvk_posterior needs none
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t n = std::min<int64_t>(std::max(batch, 1), sms);
  return n * packed_size(D) * (int64_t)sizeof(double);
}

extern "C" int tvk_posterior(const double* lpk, const double* b, int U, int D, int flags, double* phi,
                             double* mpk, double* logdet, double* bphi, int32_t* status, void* workspace,
                             int64_t workspace_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TVK_REQUIRE(D >= 0 && D <= kPosteriorMaxD && U >= 0, "posterior: D must be in [0, 768]");
  if (U == 0) return TVK_OK;
  if (D == 0) {  // no latent space: prior == posterior, log|I_0| = 0
    if (logdet) cudaMemsetAsync(logdet, 0, sizeof(double) * U, st);
    if (bphi) cudaMemsetAsync(bphi, 0, sizeof(double) * U, st);
    if (status) cudaMemsetAsync(status, 0, sizeof(int32_t) * U, st);
    TVK_CHECK_LAUNCH("posterior D=0");
    return TVK_OK;
  }
  if (D <= 32 * sw::MAXB && !getenv("TVK_POSTERIOR_CHOL")) {
    // one block-sweep pass gives Phi, phi and log|L| together; without mpk it works in place in lpk and
    // only eliminates (phi, log|L|: a third of the tile updates at D = 400)
    const size_t ssm = sw::smem_bytes();
    cudaFuncSetAttribute(sweep_posterior_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(sw::CL * ((resident_ctas(sw::CL * U) + sw::CL - 1) / sw::CL)));
    cfg.blockDim = dim3(sw::NT);
    cfg.dynamicSmemBytes = ssm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = sw::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // without an M / Phi output the sweep runs as block elimination + back substitution (PHI_ONLY)
    const int f2 = flags | (mpk ? 0 : sw::PHI_ONLY);
    const cudaError_t le = cudaLaunchKernelEx(&cfg, sweep_posterior_kernel, lpk, mpk ? mpk : const_cast<double*>(lpk),
                                              b, U, D, f2, phi, logdet, bphi, status);
    TVK_REQUIRE(le == cudaSuccess, "sweep_posterior: cluster launch failed");
    TVK_CHECK_LAUNCH("sweep_posterior");
    return TVK_OK;
  }
  size_t smem = kernel_smem(D);
  TVK_REQUIRE(smem <= 227 * 1024, "posterior: D too large for the shared-memory panel");
  cudaFuncSetAttribute(posterior_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  posterior_kernel<<<resident_ctas(U), PT, smem, st>>>(const_cast<double*>(lpk), b, U, D, flags, phi, mpk, logdet,
                                                        bphi, status);
  TVK_CHECK_LAUNCH("posterior");
  return TVK_OK;
}

extern "C" int tvk_spd_solve_rows(const double* apk, const double* b, int batch, int D, int R, const int32_t* skip,
                                  double* x, int32_t* status, void* workspace, int64_t workspace_bytes,
                                  void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TVK_REQUIRE(D >= 0 && D <= kPosteriorMaxD && R >= 0 && batch >= 0, "spd_solve_rows: bad shape");
  if (batch == 0) return TVK_OK;
  if (D == 0) {
    if (status) cudaMemsetAsync(status, 0, sizeof(int32_t) * batch, st);
    TVK_CHECK_LAUNCH("spd_solve_rows D=0");
    return TVK_OK;
  }
  size_t smem = kernel_smem(D);
  TVK_REQUIRE(smem <= 227 * 1024, "spd_solve_rows: D too large for the shared-memory panel");
  cudaFuncSetAttribute(spd_solve_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = resident_ctas(batch);
  int64_t cap = workspace ? workspace_bytes / (packed_size(D) * (int64_t)sizeof(double)) : 0;
  TVK_REQUIRE(cap >= 1, "spd_solve_rows: workspace too small (tvk_posterior_workspace_bytes)");
  if (grid > cap) grid = (int)cap;
  spd_solve_rows_kernel<<<grid, PT, smem, st>>>(apk, b, batch, D, R, skip, x, status, (double*)workspace);
  TVK_CHECK_LAUNCH("spd_solve_rows");
  return TVK_OK;
}
