// Fixed-order (bit-reproducible) reductions used by the E-step accumulators:
//   tvk_colsum: out[j] = beta*out[j] + alpha * sum_r a[r, j]   (N_c, phi_sum, moment sums over a batch)
//   tvk_ddot:   out    = beta*out    + alpha * sum_i x_i y_i   (aux terms <Sigma^-1, Ssum>, N . const)
// No floating-point atomics: every partial sum has a fixed owner and a fixed combination order that
// does not depend on the device, so results match across runs and GPUs.
#include "common.cuh"

namespace tvk {

constexpr int kDotBlocks = 1024;  // fixed partition (device-independent)
constexpr int kDotThreads = 256;

// 32 columns x 8 row phases per CTA: thread (tx, ty) sums rows ty, ty + 8, ... of column j (coalesced
// 256-byte row segments, 8x the loads in flight of a thread per column), the 8 phase sums are then
// combined in fixed order -- deterministic for every launch.
__global__ void __launch_bounds__(256) colsum_kernel(const double* a, int64_t rows, int64_t cols, int64_t lda,
                                                     double alpha, double beta, double* out) {
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = blockIdx.x * (int64_t)32 + tx;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (j < cols) {
    int64_t r = ty;
    for (; r + 24 < rows; r += 32) {
      s0 += a[r * lda + j];
      s1 += a[(r + 8) * lda + j];
      s2 += a[(r + 16) * lda + j];
      s3 += a[(r + 24) * lda + j];
    }
    for (; r < rows; r += 8) s0 += a[r * lda + j];
  }
  red[ty][tx] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (ty == 0 && j < cols) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; q++) s += red[q][tx];
    out[j] = (beta != 0.0 ? beta * out[j] : 0.0) + alpha * s;
  }
}

// The same sums, two adjacent columns per thread (16-byte loads, 64 columns per CTA: half the CTAs and
// twice the bytes in flight per load); per column the row partition and combination order are
// colsum_kernel's, so the results are bit-identical.  Needs lda and cols even and a 16-byte aligned a.
__global__ void __launch_bounds__(256) colsum2_kernel(const double* a, int64_t rows, int64_t cols, int64_t lda,
                                                      double alpha, double beta, double* out) {
  __shared__ double2 red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = blockIdx.x * (int64_t)64 + 2 * tx;
  double2 s0 = make_double2(0.0, 0.0), s1 = s0, s2 = s0, s3 = s0;
  if (j < cols) {
    const double2* c = reinterpret_cast<const double2*>(a + j);
    const int64_t ld2 = lda / 2;
    int64_t r = ty;
    for (; r + 24 < rows; r += 32) {
      const double2 v0 = c[r * ld2], v1 = c[(r + 8) * ld2], v2 = c[(r + 16) * ld2], v3 = c[(r + 24) * ld2];
      s0.x += v0.x; s0.y += v0.y;
      s1.x += v1.x; s1.y += v1.y;
      s2.x += v2.x; s2.y += v2.y;
      s3.x += v3.x; s3.y += v3.y;
    }
    for (; r < rows; r += 8) {
      const double2 v0 = c[r * ld2];
      s0.x += v0.x; s0.y += v0.y;
    }
  }
  red[ty][tx] = make_double2((s0.x + s1.x) + (s2.x + s3.x), (s0.y + s1.y) + (s2.y + s3.y));
  __syncthreads();
  if (ty == 0 && j < cols) {
    double sx = 0.0, sy = 0.0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      sx += red[q][tx].x;
      sy += red[q][tx].y;
    }
    out[j] = (beta != 0.0 ? beta * out[j] : 0.0) + alpha * sx;
    out[j + 1] = (beta != 0.0 ? beta * out[j + 1] : 0.0) + alpha * sy;
  }
}

__global__ void dot_partial_kernel(const double* x, const double* y, int64_t n, double* partial) {
  __shared__ double red[kDotThreads];
  int64_t per = (n + kDotBlocks - 1) / kDotBlocks;
  int64_t lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kDotThreads) s += x[i] * (y ? y[i] : 1.0);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kDotThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void dot_final_kernel(const double* partial, double alpha, double beta, double* out) {
  __shared__ double red[kDotThreads];
  double s = 0.0;
  for (int i = threadIdx.x; i < kDotBlocks; i += kDotThreads) s += partial[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = kDotThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = (beta != 0.0 ? beta * out[0] : 0.0) + alpha * red[0];
}

// One warp per row: norm[r] = log sum_j exp(a[r, j]) (max-shifted), a[r, j] <- exp(a[r, j] - norm[r]).
// The GMM E-step responsibilities (gmm.py:284-287, 345-348).  Fixed order per row.
__global__ void row_softmax_kernel(double* a, int64_t rows, int cols, double* norm) {
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  double* row = a + r * cols;
  double mx = -INFINITY;
  for (int j = lane; j < cols; j += 32) mx = fmax(mx, row[j]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const double sh = isfinite(mx) ? mx : 0.0;  // scipy logsumexp convention
  double s = 0.0;
  for (int j = lane; j < cols; j += 32) s += exp(row[j] - sh);
  s = warp_sum(s);
  const double lse = log(s) + sh;
  for (int j = lane; j < cols; j += 32) row[j] = exp(row[j] - lse);
  if (lane == 0) norm[r] = lse;
}

}  // namespace tvk

extern "C" int tvk_colsum(const double* a, int64_t rows, int64_t cols, int64_t lda, double alpha, double beta,
                          double* out, void* stream) {
  TVK_REQUIRE(rows >= 0 && cols >= 0 && lda >= cols, "colsum: bad shape");
  if (cols == 0) return TVK_OK;
  if (cols % 2 == 0 && lda % 2 == 0 && ((uintptr_t)a & 15) == 0) {
    tvk::colsum2_kernel<<<(unsigned)((cols + 63) / 64), 256, 0, (cudaStream_t)stream>>>(a, rows, cols, lda, alpha,
                                                                                         beta, out);
  } else {
    tvk::colsum_kernel<<<(unsigned)((cols + 31) / 32), 256, 0, (cudaStream_t)stream>>>(a, rows, cols, lda, alpha,
                                                                                        beta, out);
  }
  TVK_CHECK_LAUNCH("colsum");
  return TVK_OK;
}

extern "C" int64_t tvk_ddot_workspace_bytes(void) { return tvk::kDotBlocks * (int64_t)sizeof(double); }

extern "C" int tvk_ddot(const double* x, const double* y, int64_t n, double alpha, double beta, double* out,
                        double* workspace, void* stream) {
  TVK_REQUIRE(n >= 0 && workspace != nullptr, "ddot: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  tvk::dot_partial_kernel<<<tvk::kDotBlocks, tvk::kDotThreads, 0, st>>>(x, y, n, workspace);
  tvk::dot_final_kernel<<<1, tvk::kDotThreads, 0, st>>>(workspace, alpha, beta, out);
  TVK_CHECK_LAUNCH("ddot");
  return TVK_OK;
}

extern "C" int tvk_row_softmax(double* a, int64_t rows, int cols, double* norm, void* stream) {
  TVK_REQUIRE(rows >= 0 && cols >= 1, "row_softmax: bad shape");
  if (rows == 0) return TVK_OK;
  const int64_t blocks = (rows * 32 + 255) / 256;
  tvk::row_softmax_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a, rows, cols, norm);
  TVK_CHECK_LAUNCH("row_softmax");
  return TVK_OK;
}
