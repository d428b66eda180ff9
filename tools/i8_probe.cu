// tcgen05.mma kind::i8 probe: correctness of one M=128 x N x K=64 product (A int8 in TMEM, B int8 in
// smem, K-major no-swizzle, D s32 in TMEM) against the host, then the issue rate for N = 32/64/128.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "../paper_1906_08556_b200/csrc/tc.cuh"
using namespace tvk;

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {  // D s32, A/B signed 8-bit, K-major
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_i8_ss(uint32_t d, uint64_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__host__ __device__ inline uint32_t koff8(int r, int k, int KB) {  // byte offset, K-major, KB bytes per row
  return (uint32_t)((r >> 3) * (8 * KB) + (k >> 4) * 128 + (r & 7) * 16 + (k & 15));
}

constexpr int KB = 64;
template <int N>
__global__ void check(const int8_t* A, const int8_t* B, int* D) {  // A 128 x 64, B N x 64 (row-major)
  __shared__ __align__(1024) int8_t bs[N * KB];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < N * KB; i += blockDim.x) bs[koff8(i / KB, i % KB, KB)] = B[i];
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tbase, lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  {  // A row (= lane) into TMEM columns 256.. : 4 int8 per column, little endian
    float w[32];
    const int r = warp * 32 + (tid & 31);
    for (int c = 0; c < KB / 4; c++) {
      uint32_t u = 0;
      for (int b = 0; b < 4; b++) u |= (uint32_t)(uint8_t)A[r * KB + 4 * c + b] << (8 * b);
      w[c] = __uint_as_float(u);
    }
    for (int c = KB / 4; c < 32; c++) w[c] = 0.f;
    tc::tmem_st32(lane_addr + 256, w);
    tc::tmem_st_wait();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (tid == 0) {
    tc::fence_after_sync();
    for (int s = 0; s < KB / 32; s++) {
      uint64_t bd = tc::smem_desc(tc::smem_u32(bs) + 256 * s, 128, 8 * KB);
      mma_i8_ts(tmem, tmem + 256 + 8 * s, bd, idesc_i8(128, N), s > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(lane_addr + c0, v);
    tc::tmem_ld_wait();
    const int r = warp * 32 + (tid & 31);
    for (int j = 0; j < 32; j++) D[r * N + c0 + j] = __float_as_int(v[j]);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int N>
void run_check() {
  int8_t hA[128 * KB], hB[N * KB];
  for (int i = 0; i < 128 * KB; i++) hA[i] = (int8_t)((rand() % 255) - 127);
  for (int i = 0; i < N * KB; i++) hB[i] = (int8_t)((rand() % 255) - 127);
  int8_t *dA, *dB; int* dD;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  check<N><<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  static int hD[128 * 256];
  cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; m++)
    for (int n = 0; n < N; n++) {
      int s = 0;
      for (int k = 0; k < KB; k++) s += hA[m * KB + k] * hB[n * KB + k];
      if (s != hD[m * N + n]) { if (bad < 3) printf("  m %d n %d: got %d want %d\n", m, n, hD[m * N + n], s); bad++; }
    }
  printf("check N=%d: %s, %d mismatches\n", N, cudaGetErrorString(e), bad);
}

template <int N, bool TS>
__global__ void rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<int*>(smem)[i] = i * 77;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  uint32_t tmem = tbase;
  if (tid == 0) {
    uint32_t a = tc::smem_u32(smem), b = a + 32768;
    const uint32_t idesc = idesc_i8(128, N);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
      for (int s = 0; s < 4; s++) {
        uint64_t bd = tc::smem_desc(b + 4096 * ((i * 4 + s) & 3), 128, 256);
        if (TS) mma_i8_ts(tmem + (s & 1) * 128, tmem + 256 + 8 * s, bd, idesc, 1);
        else {
          uint64_t ad = tc::smem_desc(a + 4096 * s, 128, 256);
          mma_i8_ss(tmem + (s & 1) * 128, ad, bd, idesc, 1);
        }
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
template <int N, bool TS>
void run_rate() {
  int iters = 4000;
  unsigned long long* dc;
  cudaMalloc(&dc, 8);
  size_t sm = 64 * 1024;
  cudaFuncSetAttribute(rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  rate<N, TS><<<148, 128, sm>>>(10, dc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<N, TS><<<148, 128, sm>>>(iters, dc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  double nmma = 4.0 * iters, ops = nmma * 148 * 2.0 * 128 * N * 32;
  printf("i8 %s N=%3d: %s %.1f cycles/MMA, %.0f TOP/s\n", TS ? "TS" : "SS", N, err ? cudaGetErrorString(err) : "",
         cyc / nmma, ops / ms / 1e9);
}
int main() {
  run_check<32>(); run_check<64>(); run_check<128>();
  run_rate<32, true>(); run_rate<64, true>(); run_rate<128, true>(); run_rate<256, true>();
  run_rate<32, false>(); run_rate<64, false>(); run_rate<128, false>();
}
