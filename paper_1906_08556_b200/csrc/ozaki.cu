// FP64 GEMM emulated on the int8 tensor cores (tcgen05.mma kind::i8), Ozaki scheme with exact
// int32 accumulation -- the E-step contractions of the i-vector EM (tvm.py:183-200, 283-302:
// L = N U, A += N' M, b = F W, B += F' phi).
//
// Splitting.  Every row r of the left operand (M x K) and every column n of the right operand
// (K x N) is scaled by a power of two 2^e (e = max frexp exponent of the row / column, so the
// scaled values lie in (-1, 1)) and cut into S signed 7-bit digits:
//     x = 2^e * sum_{s=1..S} d_s 2^(-7 s) + rho,   d_s in [-127, 127] (int8),  |rho| < 2^(e - 7 S),
// d_s = trunc(128 r_{s-1}), r_s = 128 r_{s-1} - d_s (each step exact in FP64).
// Product.  C_mn = 2^(e_m + e_n) sum_{s + t <= S + 1} 2^(-7 (s + t)) sum_k a_{s,mk} b_{t,kn} + error;
// every inner sum is an int8 x int8 product accumulated EXACTLY in int32 (|level sum| <= S K 127^2
// < 2^31: K is split into pieces of <= 16,600 (S = 8) / 19,000 (S = 7), summed in fixed order), so the
// only errors are the digit truncation rho and the dropped products s + t > S + 1, each < 2^(-7 S)
// relative to |row max| * |column max| per term:
//     |C~ - C| <= (2 + S) 2^(-7 S) K max_k|a_mk| max_k|b_kn|        (S = 7: 2^-45.8 K max|a| max|b|)
// plus the final combination: the S level sums are folded EXACTLY into two int64 words, converted
// and fused once (<= 2 roundings, 2^-53 relative each).
//
// Level accumulators in TMEM.  Products with the same level L = s + t share one int32 accumulator
// block of 64 columns (levels 2..S+1 -> S blocks, 64 S <= 512 TMEM columns).  The right operand's S
// digit tiles are stored consecutively along N (rows 64 (t-1) .. 64 t - 1 of one K-major tile), so
// ONE MMA of left digit s against right digits t = 1 .. S+1-s (N = 64 (S+1-s), split at 256) writes
// every product of that digit straight into its level blocks: D column offset 64 (s-1).
// Per 32-byte k-step: S MMAs of M = 128, N = 448 .. 64 (28 products at S = 7) -- 97% of the int8
// issue rate at N >= 128 (tools/i8_probe.cu: 4.4 POPS at N = 128).
//
// Kernel roles (one CTA per SM, persistent over 128 x 64 output tiles, m fastest so concurrent CTAs
// share the right operand's tiles in L2): warp 0 lane 0 streams the pre-tiled digit blobs with
// bulk copies (one A and one B copy per k-step), warp 1 lane 0 issues the MMAs, warps 2-17 (four per
// TMEM lane quarter, 16 columns each) drain the level accumulators one 32x32b.x16 load per level,
// fold them into int64, release the accumulator to the next tile's MMAs, then scale and write C.
//
// Determinism: integer products are exact and the FP64 combination has a fixed order, so results
// are bit-reproducible run to run.  Non-finite inputs make the affected rows / columns NaN.
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "tc.cuh"

namespace tvk {
namespace oz {

constexpr int BM = 128;   // left rows per tile (MMA M, TMEM lanes)
constexpr int BN = 64;    // right rows (output columns) per tile and per level block
constexpr int KB = 32;    // bytes (= int8 elements) of K per k-step (one MMA)
// ring stages: as many 42 / 48 KB stages (S = 7 / 8 digits) as fit next to the 1 KB of barriers
template <int S>
constexpr int nst() { return (227 * 1024 - 2048) / (S * (128 + 64) * 32); }
constexpr int NT = 576;   // producer, MMA, 16 epilogue warps
constexpr int EXP_BAD = 1 << 20;  // row exponent of a row holding a non-finite value

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {  // D s32, A/B signed int8, both K-major
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// ---------------------------------------------------------------- operand splitting
// Logical operand X (R rows x K) with element (r, k) at x[r * rs + k * ks]; digit blob layout
// [row tile rb][k-step][digit s][RT rows x 32 bytes, K-major core matrices (8 rows x 16 bytes):
// (rr / 8) * 256 + (k / 16) * 128 + (rr % 8) * 16 + k % 16].

// e[r] = max_k frexp exponent of x_rk (|x_rk| < 2^e[r]), EXP_BAD if the row holds a non-finite value;
// e starts at EXP_NONE (memset 0xC0) and an all-zero row keeps it.  Blocks take 32-row x K-chunk
// tiles and fold them with atomicMax (the maximum does not depend on the order).  The scan keeps the
// largest |x| bit pattern (for non-negative doubles integer order is magnitude order, and every
// non-finite pattern lies above +inf's): one integer max per element, one ilogb per row chunk.
constexpr int EXP_NONE = (int)0xC0C0C0C0;
__device__ __forceinline__ int exp_of_absmax(unsigned long long m) {
  if (m >= 0x7FF0000000000000ull) return EXP_BAD;
  if (m == 0ull) return EXP_NONE;
  return ilogb(__longlong_as_double((long long)m)) + 1;
}
__device__ __forceinline__ unsigned long long absbits(double v) {
  return (unsigned long long)__double_as_longlong(v) & 0x7FFFFFFFFFFFFFFFull;
}
__global__ void row_exp_kernel(const double* __restrict__ x, int R, int K, int64_t rs, int64_t ks, int kchunk, int* e) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int r0 = blockIdx.x * 32;
  const int kb = blockIdx.y * kchunk, ke = min(K, kb + kchunk);
  if (rs == 1) {  // rows adjacent: one row per thread, a block reads 2 KB contiguous per k
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long m = 0ull;
    if (r < R)
#pragma unroll 8
      for (int k = kb; k < ke; k++) m = max(m, absbits(__ldg(x + r + (int64_t)k * ks)));
    const int mx = exp_of_absmax(m);
    if (r < R && mx != EXP_NONE) atomicMax(&e[r], mx);
  } else if (ks != 1) {  // general strides: lanes over rows, warps over k
    const int r = r0 + lane;
    unsigned long long m = 0ull;
    if (r < R)
#pragma unroll 8
      for (int k = kb + warp; k < ke; k += nwarp) m = max(m, absbits(__ldg(x + (int64_t)r * rs + (int64_t)k * ks)));
    const int mx = exp_of_absmax(m);
    if (r < R && mx != EXP_NONE) atomicMax(&e[r], mx);
  } else {  // k contiguous: lanes over k, warps over the tile's rows
    for (int i = warp; i < 32; i += nwarp) {
      const int r = r0 + i;
      if (r >= R) break;
      unsigned long long m = 0ull;
#pragma unroll 8
      for (int k = kb + lane; k < ke; k += 32) m = max(m, absbits(__ldg(x + (int64_t)r * rs + k)));
      const int mx = __reduce_max_sync(0xffffffffu, exp_of_absmax(m));
      if (lane == 0 && mx != EXP_NONE) atomicMax(&e[r], mx);
    }
  }
}

// The S digits of one element x of a row with exponent er, 7 bits each (sign-magnitude, then two's
// complement per byte), as 8 bytes: lo = digits S, S-1, S-2, S-3 (bytes 0..3), hi = digits S-4 ..
// S-7.  f = floor(|x| 2^(7S - er)) < 2^(7S) is formed from the mantissa with one shift, and digit s
// is bits [7(S - s), 7(S - s) + 7) of f -- exactly the FP64 recurrence d_s = trunc(128 r_{s-1}),
// r_s = 128 r_{s-1} - d_s on x 2^-er, every step of which is exact.  Integer work only (the FP64
// recurrence spent 2S conversions per element on the 16/clk conversion pipe).
template <int S>
__device__ __forceinline__ void cut_digits(double x, int er, bool ok, uint32_t& lo, uint32_t& hi) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  const unsigned long long a = b & 0x7FFFFFFFFFFFFFFFull;
  const int be = (int)(a >> 52);
  const unsigned long long mant = (a & 0xFFFFFFFFFFFFFull) | ((unsigned long long)(be != 0) << 52);
  const int sh = max(be, 1) - 1075 + 7 * S - er;  // |x| = mant 2^(max(be,1) - 1075)
  unsigned long long f = sh >= 0 ? mant << min(sh, 63) : mant >> min(-sh, 63);
  if (!ok) f = 0ull;
  uint32_t l = (uint32_t)f & 0x0FFFFFFFu, h = (uint32_t)(f >> 28) & 0x0FFFFFFFu;  // 7-bit groups 0-3, 4-7
  l = (l & 0x3FFFu) | ((l << 2) & 0x3FFF0000u);
  h = (h & 0x3FFFu) | ((h << 2) & 0x3FFF0000u);
  l = (l & 0x007F007Fu) | ((l << 1) & 0x7F007F00u);
  h = (h & 0x007F007Fu) | ((h << 1) & 0x7F007F00u);
  if (b >> 63) {  // per-byte -d for d in [0, 127]: (0x80 - d) ^ 0x80, no borrow between bytes
    l = (0x80808080u - l) ^ 0x80808080u;
    h = (0x80808080u - h) ^ 0x80808080u;
  }
  lo = l;
  hi = h;
}

// One CTA per (RT-row tile, 128/RT k-steps): the RT x 32 (x 128/RT) block is staged in shared memory
// with coalesced loads along whichever of rows / k is contiguous, every thread cuts one (row, 16-k)
// chunk into S digits, and each digit tile is written as one contiguous, fully coalesced block.
template <int S, int RT>
__global__ void __launch_bounds__(256) split_tile_kernel(const double* __restrict__ x, int R, int K, int64_t rs,
                                                         int64_t ks, const int* __restrict__ e, int KSTEPS,
                                                         int8_t* __restrict__ blob) {
  __shared__ double tile[128][KB + 1];
  const int tid = threadIdx.x;
  const int per = 128 / RT;  // k-steps per CTA
  const int rb = blockIdx.x, ks0 = blockIdx.y * per;
  const int r0 = rb * RT;
  // stage: local row lr = q * RT + rr holds row r0 + rr, k-step ks0 + q
  // all 16 loads of a thread are issued before any shared-memory store (independent, in flight together)
  constexpr int NIT = 128 * KB / 256;
  double vals[NIT];
  auto stage = [&](auto rows_fast) {
#pragma unroll
    for (int it = 0; it < NIT; it++) {
      const int i = tid + 256 * it;
      const int lr = rows_fast ? i % 128 : i / KB, kk = rows_fast ? i / 128 : i % KB;
      const int q = lr / RT, rr = lr % RT;
      const int r = r0 + rr, k = (ks0 + q) * KB + kk;
      vals[it] = (r < R && k < K && ks0 + q < KSTEPS) ? __ldg(x + (int64_t)r * rs + (int64_t)k * ks) : 0.0;
    }
#pragma unroll
    for (int it = 0; it < NIT; it++) {
      const int i = tid + 256 * it;
      const int lr = rows_fast ? i % 128 : i / KB, kk = rows_fast ? i / 128 : i % KB;
      tile[lr][kk] = vals[it];
    }
  };
  // interior blocks (every row and k of the block in range) with one unit stride: one base pointer
  // per thread advanced by a constant, no per-element bounds, all 16 loads in flight before a store
  const bool full = r0 + RT <= R && (int64_t)(ks0 + per) * KB <= K;
  auto stage_fast = [&](auto rows_fast) {
    const double* p;
    int64_t step;
    if (rows_fast) {  // i = tid + 256 it: lr = tid % 128 (q = lr / RT, rr = lr % RT), kk = 2 it + tid / 128
      const int lr = tid & 127;
      p = x + (r0 + lr % RT) + ((int64_t)(ks0 + lr / RT) * KB + (tid >> 7)) * ks;
      step = 2 * ks;
    } else {  // lr = tid / 32 + 8 it (q = lr / RT, rr = lr % RT), kk = tid % 32
      p = x + (int64_t)(r0 + (tid >> 5)) * rs + (int64_t)ks0 * KB + (tid & 31);
      step = 8 * rs;
    }
#pragma unroll
    for (int it = 0; it < NIT; it++) {
      if (!rows_fast && RT == 64 && it == 8)  // rows wrap to the next k-step of the same row tile
        p += KB - (int64_t)64 * rs;
      vals[it] = __ldg(p);
      p += step;
    }
#pragma unroll
    for (int it = 0; it < NIT; it++) {
      const int i = tid + 256 * it;
      const int lr = rows_fast ? i % 128 : i / KB, kk = rows_fast ? i / 128 : i % KB;
      tile[lr][kk] = vals[it];
    }
  };
  if (full && rs == 1) stage_fast(std::true_type{});
  else if (full && ks == 1) stage_fast(std::false_type{});
  else if (rs == 1) stage(std::true_type{});
  else stage(std::false_type{});
  __syncthreads();
  // thread -> (local row, k half) so that consecutive threads write consecutive 16-byte chunks:
  // chunk offset (rr / 8) * 256 + half * 128 + (rr % 8) * 16 inside a digit tile
  const int lr = (tid >> 4) * 8 + (tid & 7), half = (tid >> 3) & 1;
  const int q = lr / RT, rr = lr % RT;
  if (ks0 + q >= KSTEPS) return;
  const int r = r0 + rr;
  const int er = r < R ? e[r] : EXP_NONE;
  const bool ok = er != EXP_BAD && er != EXP_NONE;
  uint32_t w[S][4];
#pragma unroll
  for (int j = 0; j < 4; j++) {  // four elements -> their digit bytes, transposed to one word per digit
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int i = 0; i < 4; i++) cut_digits<S>(tile[lr][half * 16 + 4 * j + i], er, ok, lo[i], hi[i]);
    uint32_t g[8];
    {
      const uint32_t p0 = __byte_perm(lo[0], lo[1], 0x5140), p1 = __byte_perm(lo[0], lo[1], 0x7362);
      const uint32_t p2 = __byte_perm(lo[2], lo[3], 0x5140), p3 = __byte_perm(lo[2], lo[3], 0x7362);
      g[0] = __byte_perm(p0, p2, 0x5410);
      g[1] = __byte_perm(p0, p2, 0x7632);
      g[2] = __byte_perm(p1, p3, 0x5410);
      g[3] = __byte_perm(p1, p3, 0x7632);
    }
    {
      const uint32_t p0 = __byte_perm(hi[0], hi[1], 0x5140), p1 = __byte_perm(hi[0], hi[1], 0x7362);
      const uint32_t p2 = __byte_perm(hi[2], hi[3], 0x5140), p3 = __byte_perm(hi[2], hi[3], 0x7362);
      g[4] = __byte_perm(p0, p2, 0x5410);
      g[5] = __byte_perm(p0, p2, 0x7632);
      g[6] = __byte_perm(p1, p3, 0x5410);
      g[7] = __byte_perm(p1, p3, 0x7632);
    }
#pragma unroll
    for (int t = 0; t < S; t++) w[t][j] = g[S - 1 - t];  // digit t + 1 = 7-bit group S - 1 - t
  }
  int8_t* dst = blob + (((int64_t)rb * KSTEPS + ks0 + q) * S) * (RT * KB) + (rr >> 3) * 256 + half * 128 + (rr & 7) * 16;
#pragma unroll
  for (int t = 0; t < S; t++)
    *reinterpret_cast<uint4*>(dst + (int64_t)t * RT * KB) = make_uint4(w[t][0], w[t][1], w[t][2], w[t][3]);
}

// ---------------------------------------------------------------- GEMM
struct Args {
  const int8_t* A;  // left digits, BM-row tiles
  const int* ea;
  const int8_t* B;  // right digits, BN-row tiles
  const int* eb;
  int M, N, KSTEPS, mt, nt, nsplit, per;
  double alpha, beta;
  double* C;
  int64_t ldc;
  double* work;  // nsplit > 1: partials [split][M][N]
  int dbg;       // diagnostics build only: 1 = epilogue drains TMEM without arithmetic / stores
};

template <int S>
__global__ void __launch_bounds__(NT, 1) gemm_i8_kernel(Args p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int ABYTES = S * BM * KB, BBYTES = S * BN * KB, STAGE = ABYTES + BBYTES;
  constexpr int NST = nst<S>();
  __shared__ uint64_t full[NST], empty[NST], tfull, tempty;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int units = p.mt * p.nt * p.nsplit;
  if (tid == 0) {
    for (int i = 0; i < NST; i++) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(&tfull, 1);
    tc::mbar_init(&tempty, 16);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;
  auto unit_of = [&](int u, int& mtile, int& ntile, int& k0, int& k1) {
    mtile = u % p.mt;
    ntile = (u / p.mt) % p.nt;
    const int sp = u / (p.mt * p.nt);
    k0 = sp * p.per;
    k1 = min(p.KSTEPS, k0 + p.per);
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------------- producer
      uint32_t q = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int mtile, ntile, k0, k1;
        unit_of(u, mtile, ntile, k0, k1);
        for (int ks = k0; ks < k1; ks++, q++) {
          const int slot = q % NST;
          tc::mbar_wait_backoff(&empty[slot], ((q / NST) & 1) ^ 1, 32);
          tc::mbar_arrive_expect_tx(&full[slot], STAGE);
          uint8_t* st = smem + slot * STAGE;
          tc::bulk_g2s(st, p.A + ((int64_t)mtile * p.KSTEPS + ks) * ABYTES, ABYTES, &full[slot]);
          tc::bulk_g2s(st + ABYTES, p.B + ((int64_t)ntile * p.KSTEPS + ks) * BBYTES, BBYTES, &full[slot]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------------- MMA issuer
      uint32_t q = 0, li = 0;
      const uint32_t sb = tc::smem_u32(smem);
      for (int u = blockIdx.x; u < units; u += gridDim.x, li++) {
        int mtile, ntile, k0, k1;
        unit_of(u, mtile, ntile, k0, k1);
        tc::mbar_wait_backoff(&tempty, (li & 1) ^ 1, 32);  // the epilogue drained the previous unit
        tc::fence_after_sync();
        for (int ks = k0; ks < k1; ks++, q++) {
          const int slot = q % NST;
          tc::mbar_wait_backoff(&full[slot], (q / NST) & 1, 0);
          tc::fence_after_sync();
          const uint32_t a0 = sb + slot * STAGE, b0 = a0 + ABYTES;
#pragma unroll
          for (int s = 0; s < S; s++) {  // left digit s + 1 against right digits 1 .. S - s
            const int Ns = BN * (S - s);
            const uint64_t ad = tc::smem_desc(a0 + s * BM * KB, 128, 256);
#pragma unroll
            for (int n0 = 0; n0 < Ns; n0 += 256) {
              const int nn = Ns - n0 < 256 ? Ns - n0 : 256;
              const uint64_t bd = tc::smem_desc(b0 + n0 * KB, 128, 256);
              mma_i8_ss(tmem + BN * s + n0, ad, bd, idesc_i8(BM, nn), (ks > k0 || s > 0) ? 1u : 0u);
            }
          }
          tc::mma_commit(&empty[slot]);
        }
        tc::mma_commit(&tfull);
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2-17)
    // four warps per TMEM lane quarter, each owns 16 of the tile's 64 columns.  The S level blocks are
    // read one at a time (tcgen05.ld 32x32b.x16) and folded exactly into two int64 words per column,
    // then the accumulator is released -- the next tile's MMAs run while the FP64 combination, the
    // scaling and the stores of this one finish.
    const int quarter = warp & 3, part = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16) + 16 * part;
    constexpr int NH = S < 4 ? S : 4;  // levels folded into the high int64 word
    uint32_t li = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, li++) {
      int mtile, ntile, k0, k1;
      unit_of(u, mtile, ntile, k0, k1);
      const int sp = u / (p.mt * p.nt);
      const int m = mtile * BM + row;
      const bool mok = m < p.M;
      const bool rmw = mok && p.nsplit == 1 && p.beta != 0.0;
      const int nb = ntile * BN + 16 * part;
      const int em = mok ? p.ea[m] : EXP_NONE;
      // column exponents of this warp's 16 columns: lane j holds column nb + j (shuffled below)
      const int en_l = (lane < 16 && nb + lane < p.N) ? p.eb[nb + lane] : EXP_NONE;
      tc::mbar_wait(&tfull, li & 1);
      tc::fence_after_sync();
      long long hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; j++) hi[j] = lo[j] = 0;
#pragma unroll
      for (int L = 0; L < S; L++) {
        uint32_t v[16];
        tmem_ld16(lane_addr + BN * L, v);
        tc::tmem_ld_wait();
        // level L (0-based) carries the products with s + t = L + 2, weight 2^(-7 (L + 2)); |level| < 2^31
        // so hi (levels 0..NH-1) < 2^53 and lo (the rest) < 2^52: exact
#pragma unroll
        for (int j = 0; j < 16; j++) {
          if (L < NH) hi[j] += (long long)(int)v[j] << (7 * (NH - 1 - L));
          else lo[j] += (long long)(int)v[j] << (7 * (S - 1 - L));
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty);
      if (p.dbg == 1) continue;  // (warp-uniform) -- rows past M stay convergent for the shuffles below
      double* crow = p.C + (int64_t)(mok ? m : 0) * p.ldc;
      double* dst = p.nsplit > 1 ? p.work + ((int64_t)sp * p.M + (mok ? m : 0)) * p.N : crow;
#pragma unroll
      for (int h = 0; h < 16; h += 8) {  // two groups of 8 columns (register budget of 576 threads)
        double cur[8];
#pragma unroll
        for (int j = 0; j < 8; j++) cur[j] = (rmw && nb + h + j < p.N) ? crow[nb + h + j] : 0.0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int en = __shfl_sync(0xffffffffu, en_l, h + j);
          double c = (double)hi[h + j] * (1.0 / (double)(1ll << (7 * (NH + 1))));
          if (S > NH) c = fma((double)lo[h + j], ldexp(1.0, -7 * (S + 1)), c);
          const int e2 = em + en;
          double r;
          if (em == EXP_BAD || en == EXP_BAD) {
            r = __longlong_as_double(0x7ff8000000000000ll);
          } else if (em == EXP_NONE || en == EXP_NONE) {
            r = 0.0;  // an all-zero row or column: all-zero digits
          } else if (e2 > -1000 && e2 < 1000) {
            r = p.alpha * (c * __longlong_as_double((long long)(e2 + 1023) << 52));
          } else {
            r = p.alpha * ldexp(c, e2);
          }
          if (rmw) r += p.beta * cur[j];
          if (mok && nb + h + j < p.N) dst[nb + h + j] = r;
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

__global__ void splitk_sum_kernel(const double* __restrict__ work, int nsplit, int M, int N, double beta, double* C,
                                  int64_t ldc) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nsplit; k++) s += work[(int64_t)k * total + i];  // fixed order
    const int64_t r = i / N, c = i % N;
    double* cp = C + r * ldc + c;
    *cp = s + (beta != 0.0 ? beta * *cp : 0.0);
  }
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// digits of a logical R x K operand into blob (RT-row tiles), exponents into e
template <int S>
static void split_operand(const double* x, int R, int K, int64_t rs, int64_t ks, int RT, int KSTEPS, int* e,
                          int8_t* blob, cudaStream_t st) {
  cudaMemsetAsync(e, 0xC0, sizeof(int) * R, st);
  // (rs == 1: 256 rows per block, else 32); k chunks so that about 8 blocks per SM exist
  const int rb = rs == 1 ? (R + 255) / 256 : (R + 31) / 32;
  int kch = std::max(1, (int)std::min<int64_t>(K, (int64_t)K * rb / (num_sms() * 8) + 1));
  kch = std::max(kch, rs == 1 ? 64 : 256);
  row_exp_kernel<<<dim3(rb, (K + kch - 1) / kch), 256, 0, st>>>(x, R, K, rs, ks, kch, e);
  const int per = 128 / RT;
  auto kern = RT == 64 ? split_tile_kernel<S, 64> : split_tile_kernel<S, 128>;
  kern<<<dim3((R + RT - 1) / RT, (KSTEPS + per - 1) / per), 256, 0, st>>>(x, R, K, rs, ks, e,
                                                                                         KSTEPS, blob);
}

// bytes of a split operand: digit blob (rows padded to the row tile, K to 32) then int32 row exponents
static size_t operand_bytes(int R, int K, int RT, int S) {
  const size_t Rp = (size_t)(R + RT - 1) / RT * RT, KSTEPS = (size_t)(K + KB - 1) / KB;
  return ((Rp * KSTEPS * KB * S + 255) & ~size_t(255)) + sizeof(int) * Rp;
}

template <int S>
static int run(const GemmArgs& g, const void* a_split, const void* b_split, cudaStream_t st) {
  const int M = g.M, N = g.N, K = g.K;
  const int mt = ceil_div(M, BM), nt = ceil_div(N, BN), KSTEPS = ceil_div(K, KB);
  const int Mp = mt * BM, Np = nt * BN;
  // split K when the tile grid leaves SMs idle (and to keep every int32 level sum below 2^31)
  int nsplit = 1;
  const int tiles = mt * nt;
  while (nsplit < 32 && (int64_t)tiles * nsplit < 2 * num_sms() && KSTEPS / (nsplit * 2) >= 16) nsplit *= 2;
  while ((int64_t)S * ceil_div(KSTEPS, nsplit) * KB * 127 * 127 >= (1ll << 31)) nsplit *= 2;
  const int per = ceil_div(KSTEPS, nsplit);
  nsplit = ceil_div(KSTEPS, per);  // every split non-empty
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  const size_t ba = a_split ? 0 : operand_bytes(M, K, BM, S), bb = b_split ? 0 : operand_bytes(N, K, BN, S);
  const size_t bw = nsplit > 1 ? sizeof(double) * (size_t)nsplit * M * N : 0;
  static bool pool_ready = false;
  if (!pool_ready) {  // keep freed scratch mapped in the stream-ordered pool between calls
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_ready = true;
  }
  uint8_t* scratch = nullptr;
  if (ba + bb + bw > 0 && cudaMallocAsync((void**)&scratch, al(ba) + al(bb) + bw, st) != cudaSuccess) {
    cudaGetLastError();
    set_error("ozaki gemm: cannot allocate %zu bytes of scratch", al(ba) + al(bb) + bw);
    return TVK_ERR_CUDA;
  }
  const uint8_t* opA = a_split ? (const uint8_t*)a_split : scratch;
  const uint8_t* opB = b_split ? (const uint8_t*)b_split : scratch + al(ba);
  const int8_t* blobA = (const int8_t*)opA;
  const int8_t* blobB = (const int8_t*)opB;
  const int* ea = (const int*)(opA + ((size_t)Mp * KSTEPS * KB * S + 255 & ~size_t(255)));
  const int* eb = (const int*)(opB + ((size_t)Np * KSTEPS * KB * S + 255 & ~size_t(255)));
  double* work = nsplit > 1 ? (double*)(scratch + al(ba) + al(bb)) : nullptr;
  // op(A): (m, k) = A[m lda + k] or A[k lda + m];  op(B) as rows n: (n, k) = B[k ldb + n] or B[n ldb + k]
  if (!a_split) {
    if (g.trans_a) split_operand<S>(g.A, M, K, 1, g.lda, BM, KSTEPS, (int*)ea, (int8_t*)blobA, st);
    else split_operand<S>(g.A, M, K, g.lda, 1, BM, KSTEPS, (int*)ea, (int8_t*)blobA, st);
  }
  if (!b_split) {
    if (g.trans_b) split_operand<S>(g.B, N, K, g.ldb, 1, BN, KSTEPS, (int*)eb, (int8_t*)blobB, st);
    else split_operand<S>(g.B, N, K, 1, g.ldb, BN, KSTEPS, (int*)eb, (int8_t*)blobB, st);
  }
  TVK_CHECK_LAUNCH("ozaki split");
  Args a{};
  a.A = blobA;
  a.ea = ea;
  a.B = blobB;
  a.eb = eb;
  a.M = M;
  a.N = N;
  a.KSTEPS = KSTEPS;
  a.mt = mt;
  a.nt = nt;
  a.nsplit = nsplit;
  a.per = per;
  a.alpha = g.alpha;
  a.beta = g.beta;
  a.C = g.C;
  a.ldc = g.ldc;
  a.work = work;
#ifdef TVK_SELECT_DIAG
  if (const char* d = getenv("TVK_OZ_DEBUG")) a.dbg = atoi(d);
#endif
  const size_t smem = (size_t)nst<S>() * S * (BM + BN) * KB;
  auto kern = gemm_i8_kernel<S>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int units = mt * nt * nsplit;
  const int grid = std::min(units, num_sms());
  kern<<<grid, NT, smem, st>>>(a);
  TVK_CHECK_LAUNCH("ozaki gemm");
  if (nsplit > 1) {
    const int64_t total = (int64_t)M * N;
    splitk_sum_kernel<<<(int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16), 256, 0, st>>>(
        work, nsplit, M, N, g.beta, g.C, g.ldc);
    TVK_CHECK_LAUNCH("ozaki split-K sum");
  }
  if (scratch) cudaFreeAsync(scratch, st);
  return TVK_OK;
}

}  // namespace oz

int ozaki_gemm(const GemmArgs& p, int digits, const void* a_split, const void* b_split, cudaStream_t st) {
  TVK_REQUIRE(p.M >= 0 && p.N >= 0 && p.K >= 0, "dgemm_i8: negative size");
  TVK_REQUIRE(digits >= 6 && digits <= 8, "dgemm_i8: digits must be 6, 7 or 8");
  TVK_REQUIRE(p.K <= (1 << 27), "dgemm_i8: K too large");
  if (p.M == 0 || p.N == 0) return TVK_OK;
  if (p.K == 0) {  // C = beta C
    GemmArgs q = p;
    q.batch = 1;
    q.out_mode = TVK_OUT_DENSE;
    q.splits = 1;
    return gemm(q, st);
  }
  switch (digits) {
    case 6: return oz::run<6>(p, a_split, b_split, st);
    case 8: return oz::run<8>(p, a_split, b_split, st);
    default: return oz::run<7>(p, a_split, b_split, st);
  }
}

}  // namespace tvk

extern "C" int64_t tvk_i8_operand_bytes(int rows, int k, int row_tile, int digits) {
  if (rows < 0 || k < 0 || (row_tile != 64 && row_tile != 128) || digits < 6 || digits > 8) return -1;
  return (int64_t)tvk::oz::operand_bytes(rows, k, row_tile, digits);
}

extern "C" int tvk_i8_split(const double* x, int rows, int k, int64_t rs, int64_t ks, int row_tile, int digits,
                            void* out, void* stream) {
  TVK_REQUIRE(rows >= 0 && k >= 0 && (row_tile == 64 || row_tile == 128), "i8_split: bad shape / row tile");
  TVK_REQUIRE(digits >= 6 && digits <= 8, "i8_split: digits must be 6, 7 or 8");
  if (rows == 0 || k == 0) return TVK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int KSTEPS = (k + tvk::oz::KB - 1) / tvk::oz::KB;
  const int Rp = (rows + row_tile - 1) / row_tile * row_tile;
  int8_t* blob = (int8_t*)out;
  int* e = (int*)((uint8_t*)out + (((size_t)Rp * KSTEPS * tvk::oz::KB * digits + 255) & ~size_t(255)));
  switch (digits) {
    case 6: tvk::oz::split_operand<6>(x, rows, k, rs, ks, row_tile, KSTEPS, e, blob, st); break;
    case 8: tvk::oz::split_operand<8>(x, rows, k, rs, ks, row_tile, KSTEPS, e, blob, st); break;
    default: tvk::oz::split_operand<7>(x, rows, k, rs, ks, row_tile, KSTEPS, e, blob, st); break;
  }
  TVK_CHECK_LAUNCH("i8_split");
  return TVK_OK;
}

extern "C" int tvk_dgemm_i8(int trans_a, int trans_b, int m, int n, int k, double alpha, const double* a, int64_t lda,
                            const void* a_split, const double* b, int64_t ldb, const void* b_split, double beta,
                            double* c, int64_t ldc, int digits, void* stream) {
  tvk::GemmArgs p{};
  p.trans_a = trans_a;
  p.trans_b = trans_b;
  p.M = m;
  p.N = n;
  p.K = k;
  p.alpha = alpha;
  p.A = a;
  p.lda = lda;
  p.B = b;
  p.ldb = ldb;
  p.beta = beta;
  p.C = c;
  p.ldc = ldc;
  p.batch = 1;
  p.out_mode = TVK_OUT_DENSE;
  p.splits = 1;
  return tvk::ozaki_gemm(p, digits, a_split, b_split, (cudaStream_t)stream);
}
