// Measures the FP64 issue ceilings of this B200: DFMA (FMA pipe) vs DMMA.8x8x4 (tensor pipe).
// Build+run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a[16];
  for (int i = 0; i < 16; i++) a[i] = threadIdx.x * 1e-3 + i;
  double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 16; i++) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    int iters = 20000;
    dim3 grid(sms * 2), block(32 * warps);
    dfma_loop<<<grid, block>>>(d, 100);
    cudaEventRecord(e0);
    dfma_loop<<<grid, block>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)grid.x * block.x;
    printf("DFMA  warps/CTA=%2d  %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    dmma_loop<<<grid, block>>>(d, 100);
    cudaEventRecord(e0);
    dmma_loop<<<grid, block>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 256 * 8 * iters * (double)grid.x * (block.x / 32);
    printf("DMMA  warps/CTA=%2d  %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
