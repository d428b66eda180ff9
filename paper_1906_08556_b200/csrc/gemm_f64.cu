// Batched FP64 GEMM on the DMMA tensor pipe: C = alpha*op(A)*op(B) + beta*C.
// Output either dense or packed-lower (row-major i(i+1)/2 + j, square outputs only;
// tiles strictly above the diagonal are skipped).  Deterministic split-K for tall-K
// shapes (b = F W): partials go to a workspace and are summed in fixed order.
#include "gemm_f64.cuh"
#include "internal.h"

namespace tvk {

template <class Cfg, bool TA, bool TB, bool VEC>
__global__ void __launch_bounds__(Cfg::NT) gemm_kernel(GemmArgs p, int mtiles, int ntiles) {
  using L = SmemLayout<Cfg::BM, Cfg::BN, Cfg::BK, TA, TB>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  const int tile = blockIdx.x;
  const int mt = tile % mtiles, nt = tile / mtiles;
  const int m0 = mt * Cfg::BM, n0 = nt * Cfg::BN;
  const int64_t bz = blockIdx.y;
  const int split = blockIdx.z;

  if (p.out_mode == TVK_OUT_PACKED_LOWER && m0 + Cfg::BM - 1 < n0) return;  // strictly upper tile

  const double* A = p.A + bz * p.strideA;
  const double* B = p.B + bz * p.strideB;

  int kbeg = 0, kend = p.K;
  if (p.splits > 1) {
    int64_t per = ((int64_t)p.K + p.splits - 1) / p.splits;
    per = (per + Cfg::BK - 1) / Cfg::BK * Cfg::BK;
    kbeg = (int)((int64_t)split * per < p.K ? (int64_t)split * per : p.K);
    kend = (int)((int64_t)(split + 1) * per < p.K ? (int64_t)(split + 1) * per : p.K);
  }
  const int nk = (kend - kbeg + Cfg::BK - 1) / Cfg::BK;

  auto load_stage = [&](int stage, int kt) {
    double* sA = smem + stage * L::STAGE;
    double* sB = sA + L::A_ELEMS;
    int k0 = kbeg + kt * Cfg::BK;
    // clamp the K extent to this split's range so other splits' columns stay zero
    if constexpr (TA)
      load_tile_async<Cfg::BK, Cfg::BM, Cfg::BM + 4, Cfg::NT, VEC>(sA, A, p.lda, k0, m0, kend, p.M, tid);
    else
      load_tile_async<Cfg::BM, Cfg::BK, Cfg::BK + 4, Cfg::NT, VEC>(sA, A, p.lda, m0, k0, p.M, kend, tid);
    if constexpr (TB)
      load_tile_async<Cfg::BN, Cfg::BK, Cfg::BK + 4, Cfg::NT, VEC>(sB, B, p.ldb, n0, k0, p.N, kend, tid);
    else
      load_tile_async<Cfg::BK, Cfg::BN, Cfg::BN + 4, Cfg::NT, VEC>(sB, B, p.ldb, k0, n0, kend, p.N, tid);
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
    const double* sA = smem + (kt % Cfg::STAGES) * L::STAGE;
    mma_stage<Cfg, L>(acc, sA, sA + L::A_ELEMS, wm, wn, lane);
  }
  cp_async_wait<0>();

  if (p.splits > 1) {
    double* W = p.work + (int64_t)split * p.M * p.N;
    for_each_acc<Cfg>(acc, wm, wn, lane, [&](int r, int c, double v) {
      int gr = m0 + r, gc = n0 + c;
      if (gr < p.M && gc < p.N) W[(int64_t)gr * p.N + gc] = p.alpha * v;
    });
    return;
  }
  double* C = p.C + bz * p.strideC;
  const bool packed = p.out_mode == TVK_OUT_PACKED_LOWER;
  for_each_acc<Cfg>(acc, wm, wn, lane, [&](int r, int c, double v) {
    int gr = m0 + r, gc = n0 + c;
    if (gr >= p.M || gc >= p.N) return;
    if (packed && gc > gr) return;
    int64_t idx = packed ? packed_index(gr, gc) : (int64_t)gr * p.ldc + gc;
    double out = p.alpha * v;
    if (p.beta != 0.0) out += p.beta * C[idx];
    C[idx] = out;
  });
}

__global__ void splitk_reduce(GemmArgs p) {
  int64_t total = (int64_t)p.M * p.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < p.splits; k++) s += p.work[(int64_t)k * total + i];  // fixed order
    int64_t r = i / p.N, c = i % p.N;
    if (p.out_mode == TVK_OUT_PACKED_LOWER) {
      if (c > r) continue;
      int64_t idx = packed_index(r, c);
      p.C[idx] = s + (p.beta != 0.0 ? p.beta * p.C[idx] : 0.0);
    } else {
      int64_t idx = r * p.ldc + c;
      p.C[idx] = s + (p.beta != 0.0 ? p.beta * p.C[idx] : 0.0);
    }
  }
}

using BigCfg = GemmCfg<64, 64, 16, 2, 2, 3>;  // 4 CTAs (16 warps) per SM
using SmallCfg = GemmCfg<64, 64, 16, 2, 2, 3>;

template <class Cfg, bool TA, bool TB, bool VEC>
static int launch_cfg(const GemmArgs& p, cudaStream_t st) {
  using L = SmemLayout<Cfg::BM, Cfg::BN, Cfg::BK, TA, TB>;
  size_t smem = sizeof(double) * L::STAGE * Cfg::STAGES;
  auto kern = gemm_kernel<Cfg, TA, TB, VEC>;
  static bool attr_set = false;  // benign race: idempotent attribute
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  int mt = ceil_div(p.M, Cfg::BM), nt = ceil_div(p.N, Cfg::BN);
  dim3 grid(mt * nt, p.batch, p.splits);
  kern<<<grid, Cfg::NT, smem, st>>>(p, mt, nt);
  TVK_CHECK_LAUNCH("dgemm");
  if (p.splits > 1) {
    int64_t total = (int64_t)p.M * p.N;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    splitk_reduce<<<blocks, 256, 0, st>>>(p);
    TVK_CHECK_LAUNCH("dgemm splitk reduce");
  }
  return TVK_OK;
}

template <bool TA, bool TB, bool VEC>
static int launch_t(const GemmArgs& p, cudaStream_t st) {
  int64_t big_tiles = (int64_t)ceil_div(p.M, 64) * ceil_div(p.N, 64) * p.batch * p.splits;
  bool big = p.M >= 48 && p.N >= 48 && big_tiles >= 148;
  return big ? launch_cfg<BigCfg, TA, TB, VEC>(p, st) : launch_cfg<SmallCfg, TA, TB, VEC>(p, st);
}

static bool aligned16(const void* ptr) { return ((uintptr_t)ptr & 15) == 0; }

int gemm(const GemmArgs& p_in, cudaStream_t st) {
  GemmArgs p = p_in;
  if (p.splits < 1) p.splits = 1;
  TVK_REQUIRE(p.M >= 0 && p.N >= 0 && p.K >= 0 && p.batch >= 1, "dgemm: negative size");
  TVK_REQUIRE(p.batch <= 65535, "dgemm: batch > 65535");
  TVK_REQUIRE(p.splits == 1 || (p.batch == 1 && p.work != nullptr), "dgemm: split-K needs batch 1 and a workspace");
  TVK_REQUIRE(p.out_mode != TVK_OUT_PACKED_LOWER || p.M == p.N, "dgemm: packed output needs M == N");
  if (p.M == 0 || p.N == 0) return TVK_OK;
  bool vec = (p.lda % 2 == 0) && (p.ldb % 2 == 0) && (p.strideA % 2 == 0) && (p.strideB % 2 == 0) &&
             aligned16(p.A) && aligned16(p.B);
  bool ta = p.trans_a != 0, tb = p.trans_b != 0;
#define TVK_DISPATCH(TA_, TB_)                                               \
  if (ta == TA_ && tb == TB_) {                                              \
    return vec ? launch_t<TA_, TB_, true>(p, st) : launch_t<TA_, TB_, false>(p, st); \
  }
  TVK_DISPATCH(false, false)
  TVK_DISPATCH(false, true)
  TVK_DISPATCH(true, false)
  TVK_DISPATCH(true, true)
#undef TVK_DISPATCH
  return TVK_ERR_INVALID;
}

}  // namespace tvk

extern "C" int tvk_dgemm(int trans_a, int trans_b, int m, int n, int k, double alpha, const double* a, int64_t lda,
                         int64_t stride_a, const double* b, int64_t ldb, int64_t stride_b, double beta, double* c,
                         int64_t ldc, int64_t stride_c, int batch, int out_mode, int splits, double* work,
                         void* stream) {
  tvk::GemmArgs p{};
  p.trans_a = trans_a;
  p.trans_b = trans_b;
  p.M = m;
  p.N = n;
  p.K = k;
  p.alpha = alpha;
  p.A = a;
  p.lda = lda;
  p.strideA = stride_a;
  p.B = b;
  p.ldb = ldb;
  p.strideB = stride_b;
  p.beta = beta;
  p.C = c;
  p.ldc = ldc;
  p.strideC = stride_c;
  p.batch = batch;
  p.out_mode = out_mode;
  p.splits = splits;
  p.work = work;
  return tvk::gemm(p, (cudaStream_t)stream);
}
