// Shared helpers for libtvk (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/tvk.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libtvk is written for sm_100a (B200) only"
#endif

namespace tvk {

// thread-local last error message, read back through tvk_last_error()
void set_error(const char* fmt, ...);

#define TVK_CHECK_LAUNCH(what)                                                   \
  do {                                                                           \
    cudaError_t e_ = cudaGetLastError();                                         \
    if (e_ != cudaSuccess) {                                                     \
      ::tvk::set_error("%s: %s", what, cudaGetErrorString(e_));                 \
      return TVK_ERR_CUDA;                                                       \
    }                                                                            \
  } while (0)

#define TVK_REQUIRE(cond, msg)                                                   \
  do {                                                                           \
    if (!(cond)) {                                                               \
      ::tvk::set_error("%s", msg);                                               \
      return TVK_ERR_INVALID;                                                    \
    }                                                                            \
  } while (0)

#define TVK_TRY(call)                                                            \
  do {                                                                           \
    int s_ = (call);                                                             \
    if (s_ != TVK_OK) return s_;                                                 \
  } while (0)

constexpr double kLog2Pi = 1.8378770664093454835606594728112;

__host__ __device__ inline int64_t packed_index(int64_t i, int64_t j) {  // i >= j, row-major lower
  return i * (i + 1) / 2 + j;
}
__host__ __device__ inline int64_t packed_size(int64_t d) { return d * (d + 1) / 2; }

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int valid_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(valid_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// D(8x8) += A(8x4, row) * B(4x8, col) in FP64 on the tensor pipe (SASS: DMMA.8x8x4).
// lane = 4*g + t: A holds A[g][t], B holds B[t][g], D holds D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace tvk
