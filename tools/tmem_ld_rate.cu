// TMEM read throughput probe: W warps (W/4 per TMEM lane quarter) each issue tcgen05.ld 32x32b.x32
// (4 KB per warp-load) R times; reports bytes per SM cycle.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include "../paper_1906_08556_b200/csrc/tc.cuh"
using namespace tvk;
template <int W>
__global__ void __launch_bounds__(W * 32, 1) probe(int R, long long* out, float* sink) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&base);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t lane_addr = base + ((uint32_t)((warp & 3) * 32) << 16);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < R; i++) {
    float v[32];
    tc::tmem_ld32(lane_addr + ((i * 32 + (warp >> 2) * 64) & 511), v);
    tc::tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; j++) acc += v[j];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 1234.5f) sink[0] = acc;
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(base);
}
template <int W>
void run(int R) {
  long long* d; float* s;
  cudaMalloc(&d, 8 * 148); cudaMalloc(&s, 4);
  probe<W><<<148, W * 32>>>(R, d, s);
  probe<W><<<148, W * 32>>>(R, d, s);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double bytes = (double)W * R * 4096;
  printf("warps %2d: %lld cycles for %.0f KB -> %.1f B/cycle/SM (err %s)\n", W, h[0], bytes / 1024, bytes / h[0],
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<4>(2000); run<8>(2000); run<16>(2000);
}
