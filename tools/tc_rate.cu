// Tensor-pipe issue-rate microbenchmark for tcgen05.mma (one CTA per SM, operands resident in smem/TMEM):
// kind::tf32 with A from smem (SS) or TMEM (TS), N = 64/128/256, and kind::f16 for comparison.
#include <cstdio>
#include "../paper_1906_08556_b200/csrc/tc.cuh"
using namespace tvk;

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// commit after every group of G MMAs to one of 8 barriers; WAIT: wait for the commit 8 groups back
template <int G, bool WAIT>
__global__ void rate_commit(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < (128 + 256) * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 7);
  if (tid == 0) { for (int i = 0; i < 8; i++) tc::mbar_init(&bars[i], 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  uint32_t tmem = tbase;
  if (tid == 0) {
    uint32_t b = tc::smem_u32(smem) + 128 * 32 * 4;
    uint32_t idesc = tc::idesc_tf32(128, 128);
    unsigned long long t0 = clock64();
    int q = 0;
    for (int i = 0; i < iters; i++) {
      for (int s = 0; s < 4; s += G, q++) {
        if (WAIT && q >= 8) tc::mbar_wait(&bars[q % 8], ((q / 8) - 1) & 1);
        for (int gg = 0; gg < G; gg++) {
          uint64_t bd = tc::smem_desc(b + 256 * (s + gg), 128, 8 * 32 * 4);
          tc::mma_tf32_ts(tmem, tmem + 256 + 8 * (s + gg), bd, idesc, 1);
        }
        tc::mma_commit(&bars[q % 8]);
      }
    }
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int G, bool WAIT>
void run_commit(const char* name) {
  int iters = 4000;
  unsigned long long* dc;
  cudaMalloc(&dc, 8);
  size_t sm = (128 + 256) * 32 * 4;
  cudaFuncSetAttribute(rate_commit<G, WAIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  rate_commit<G, WAIT><<<148, 128, sm>>>(10, dc);
  cudaDeviceSynchronize();
  rate_commit<G, WAIT><<<148, 128, sm>>>(iters, dc);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("%-22s: %s %.1f cycles/MMA (issue side)\n", name, err ? cudaGetErrorString(err) : "", cyc / (4.0 * iters));
}

// latency: issue n MMAs, commit, wait; repeated; cycles per round
__global__ void lat(int n, int rounds, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 80 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 7);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  uint32_t tmem = tbase;
  if (tid == 0) {
    uint32_t b = tc::smem_u32(smem) + 128 * 32 * 4;
    uint32_t idesc = tc::idesc_tf32(128, 128);
    unsigned long long t0 = clock64();
    for (int r = 0; r < rounds; r++) {
      for (int i = 0; i < n; i++) {
        uint64_t bd = tc::smem_desc(b + 256 * (i & 3), 128, 8 * 32 * 4);
        tc::mma_tf32_ts(tmem, tmem + 256 + 8 * (i & 3), bd, idesc, 1);
      }
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, r & 1);
    }
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (t1 - t0) / rounds;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int MODE, int N>  // MODE 0: tf32 SS, 1: tf32 TS, 2: f16 SS, 3: f16 TS, 4: f16 TS 2 acc, 5: f16 SS 2 acc
__global__ void rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 80 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 7);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  uint32_t tmem = tbase;
  if (tid == 0) {
    uint32_t a = tc::smem_u32(smem), b = a + 128 * 32 * 4;
    uint32_t idesc = MODE >= 2 ? ((1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24))
                               : tc::idesc_tf32(128, N);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
      for (int s = 0; s < 4; s++) {
        uint64_t ad = tc::smem_desc(a + 256 * s, 128, 8 * 32 * 4);
        uint64_t bd = tc::smem_desc(b + 256 * s, 128, 8 * 32 * 4);
        if (MODE == 0) tc::mma_tf32(tmem, ad, bd, idesc, 1);
        else if (MODE == 1) tc::mma_tf32_ts(tmem, tmem + 256 + 8 * s, bd, idesc, 1);
        else if (MODE == 2) mma_f16(tmem, ad, bd, idesc, 1);
        else if (MODE == 3) tc::mma_f16_ts(tmem, tmem + 256 + 8 * s, bd, idesc, 1);
        else if (MODE == 4) tc::mma_f16_ts(tmem + (s & 1) * 128, tmem + 256 + 8 * s, bd, idesc, 1);
        else if (MODE == 6) {  // f16 TS, fresh 4 KB K-major B tile (LBO 128, SBO 256) every MMA over 64 KB
          const uint64_t bf = tc::smem_desc(a + 4096 * ((i * 4 + s) & 15), 128, 256);
          tc::mma_f16_ts(tmem, tmem + 256 + 8 * s, bf, idesc, 1);
        } else if (MODE == 7) {  // same tile every MMA, same layout
          const uint64_t bf = tc::smem_desc(a, 128, 256);
          tc::mma_f16_ts(tmem, tmem + 256 + 8 * s, bf, idesc, 1);
        }
        else if (MODE == 5) mma_f16(tmem + (s & 1) * 128, ad, bd, idesc, 1);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int MODE, int N>
void run(const char* name) {
  int iters = 4000;
  unsigned long long* dc;
  cudaMalloc(&dc, 8);
  size_t sm = 80 * 1024;
  cudaFuncSetAttribute(rate<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  rate<MODE, N><<<148, 128, sm>>>(10, dc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<MODE, N><<<148, 128, sm>>>(iters, dc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  double nmma = 4.0 * iters;
  double kk = MODE >= 2 ? 16 : 8;
  double flops = nmma * 148 * 2.0 * 128 * N * kk;
  printf("%-14s N=%3d: %s %.1f cycles/MMA, %.0f TFLOP/s\n", name, N, err ? cudaGetErrorString(err) : "", cyc / nmma,
         flops / ms / 1e9);
}

int main() {
  run<0, 128>("tf32 SS");
  run<0, 256>("tf32 SS");
  run<1, 128>("tf32 TS");
  run<1, 256>("tf32 TS");
  run<2, 128>("f16 SS");
  run<2, 256>("f16 SS");
  run<3, 128>("f16 TS");
  run<3, 64>("f16 TS");
  run<4, 128>("f16 TS 2acc");
  run<5, 128>("f16 SS 2acc");
  run<2, 64>("f16 SS");
  run<6, 128>("f16 TS fresh B");
  run<7, 128>("f16 TS same B");
  if (getenv("RATE_ONLY")) return 0;
  {
    unsigned long long* dc;
    cudaMalloc(&dc, 8);
    size_t sm = (128 + 256) * 32 * 4;
    cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int n : {0, 1, 2, 4, 8, 16, 32, 64}) {
      for (int g : {1, 148}) {
        lat<<<g, 128, sm>>>(n, 200, dc);
        cudaDeviceSynchronize();
        unsigned long long c;
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("issue %2d MMAs + commit + wait (%3d CTAs): %llu cycles\n", n, g, c);
      }
    }
  }
  run_commit<1, false>("commit/1 MMA");
  run_commit<1, true>("commit/1 + wait 8 back");
  run_commit<2, true>("commit/2 + wait 8 back");
  run_commit<4, true>("commit/4 + wait 8 back");
  return 0;
}
