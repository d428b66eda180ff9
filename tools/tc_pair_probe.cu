// Probe: cta_group::2 (CTA pair) kind::f16 MMA, M=256 (128 rows per CTA, A in each CTA's TMEM),
// N=128 split across the pair (each CTA's smem holds 64 B rows), D in each CTA's TMEM.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include "../paper_1906_08556_b200/csrc/tc.cuh"
using namespace tvk;

__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

__global__ void __cluster_dims__(2, 1, 1) pair_probe(const __half* A, const __half* B, int K, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sB = smem;  // this CTA's 64 rows of B (K-major core matrices)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  const uint32_t rank = tc::cluster_ctarank();
  const int N = 128;
  for (int i = tid; i < 64 * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sB + tc::kmajor_offset16(r, k, K)) = B[(rank * 64 + r) * K + k];
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tbase)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after_sync();
  const uint32_t tmem = tbase;
  // A rows of this CTA into TMEM columns 256+ (two f16 per column)
  const int row = (warp % 4) * 32 + (tid % 32);
  const int grow = rank * 128 + row;
  for (int c0 = 0; c0 < K / 2; c0 += 32) {
    float v[32];
    for (int j = 0; j < 32; j++) {
      __half2 h2 = (2 * (c0 + j) < K) ? __halves2half2(A[grow * K + 2 * (c0 + j)], A[grow * K + 2 * (c0 + j) + 1])
                                      : __floats2half2_rn(0.f, 0.f);
      v[j] = *reinterpret_cast<float*>(&h2);
    }
    tc::tmem_st32(tmem + ((uint32_t)((warp % 4) * 32) << 16) + 256 + c0, v);
  }
  tc::tmem_st_wait();
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after_sync();
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = tc::idesc_f16(256, N);
    for (int s = 0; s < K / 16; s++) {
      uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + 256 * s, 128, 8 * K * 2);
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
          "r"(tmem + 256 + 8 * s), "l"(bd), "r"(idesc), "r"((uint32_t)(s > 0)));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(tc::smem_u32(&bar)), "h"((uint16_t)3) : "memory");
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tmem + ((uint32_t)((warp % 4) * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; j++) D[grow * N + c0 + j] = v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

int main() {
  const int M = 256, N = 128;
  for (int K : {16, 128}) {
    std::vector<__half> A(M * K), B(N * K);
    std::vector<float> Af(M * K), Bf(N * K), D(M * N);
    srand(3);
    for (int i = 0; i < M * K; i++) { A[i] = __float2half((rand() / (float)RAND_MAX - 0.5f) * 4); Af[i] = __half2float(A[i]); }
    for (int i = 0; i < N * K; i++) { B[i] = __float2half((rand() / (float)RAND_MAX - 0.5f) * 4); Bf[i] = __half2float(B[i]); }
    __half *dA, *dB; float* dD;
    cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    size_t sm = 64 * K * 2;
    cudaFuncSetAttribute(pair_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    pair_probe<<<2, 128, sm>>>(dA, dB, K, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("K=%d: CUDA error %s\n", K, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < M; i++)
      for (int j = 0; j < N; j++) {
        double s = 0;
        for (int k = 0; k < K; k++) s += (double)Af[i * K + k] * Bf[j * K + k];
        maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
        maxref = fmax(maxref, fabs(s));
      }
    printf("pair f16 M=256 N=128 K=%d: max|err| %.3e max|ref| %.3e %s\n", K, maxerr, maxref, maxerr < 1e-4 * maxref ? "OK" : "FAIL");
  }
  return 0;
}
