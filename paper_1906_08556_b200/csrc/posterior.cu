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

#include "common.cuh"
#include "internal.h"
#include "spd_small.cuh"

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
