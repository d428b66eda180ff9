// Probe: one CTA, D(128xN) = A(128xK) * B(NxK)^T with tcgen05.mma kind::tf32, operands in
// no-swizzle K-major smem, accumulator in TMEM, read back with tcgen05.ld 32x32b.  Validates the
// descriptor encodings in csrc/tc.cuh.   nvcc -gencode arch=compute_100a,code=sm_100a -o tc_probe tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_1906_08556_b200/csrc/tc.cuh"
using namespace tvk;

constexpr int M = 128;

template <int N>
__global__ void probe(const float* A, const float* B, int K, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + M * K * 4;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < M * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sA + tc::kmajor_offset(r, k, K)) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sB + tc::kmajor_offset(r, k, K)) = B[i];
  }
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<(N < 32 ? 32 : N)>(&tbase);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  uint32_t tmem = tbase;
  if (tid == 0) {
    uint32_t id = tc::idesc_tf32(M, N);
    for (int s = 0; s < K / 8; s++) {
      uint64_t ad = tc::smem_desc(tc::smem_u32(sA) + 256 * s, 128, 8 * K * 4);
      uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + 256 * s, 128, 8 * K * 4);
      tc::mma_tf32(tmem, ad, bd, id, s > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  int row = (warp % 4) * 32 + (tid % 32);
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tmem + ((uint32_t)((warp % 4) * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; j++) D[row * N + c0 + j] = v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<(N < 32 ? 32 : N)>(tmem);
}

// A (128 x K) in TMEM columns [N, N+K) of lane = row, written with tcgen05.st; B in smem.
template <int N>
__global__ void probe_ts(const float* A, const float* B, int K, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sB = smem;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sB + tc::kmajor_offset(r, k, K)) = B[i];
  }
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  uint32_t tmem = tbase;
  int row = (warp % 4) * 32 + (tid % 32);
  for (int c0 = 0; c0 < K; c0 += 32) {
    float v[32];
    for (int j = 0; j < 32; j++) v[j] = (c0 + j < K) ? A[row * K + c0 + j] : 0.f;
    tc::tmem_st32(tmem + ((uint32_t)((warp % 4) * 32) << 16) + N + c0, v);
  }
  tc::tmem_st_wait();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    uint32_t id = tc::idesc_tf32(M, N);
    for (int s = 0; s < K / 8; s++) {
      uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + 256 * s, 128, 8 * K * 4);
      tc::mma_tf32_ts(tmem, tmem + N + 8 * s, bd, id, s > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tmem + ((uint32_t)((warp % 4) * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; j++) D[row * N + c0 + j] = v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// f16: A (128 x K) packed two per 32-bit TMEM column (k even in the low half), B (N x K) f16 in smem.
#include <cuda_fp16.h>
template <int N>
__global__ void probe_f16_ts(const __half* A, const __half* B, int K, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sB = smem;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sB + tc::kmajor_offset16(r, k, K)) = B[i];
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  uint32_t tmem = tbase;
  int row = (warp % 4) * 32 + (tid % 32);
  for (int c0 = 0; c0 < K / 2; c0 += 32) {
    float v[32];
    for (int j = 0; j < 32; j++) {
      __half2 h2 = __halves2half2(A[row * K + 2 * (c0 + j)], A[row * K + 2 * (c0 + j) + 1]);
      v[j] = *reinterpret_cast<float*>(&h2);
    }
    tc::tmem_st32(tmem + ((uint32_t)((warp % 4) * 32) << 16) + 256 + c0, v);
  }
  tc::tmem_st_wait();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    uint32_t id = tc::idesc_f16(M, N);
    for (int s = 0; s < K / 16; s++) {
      uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + 256 * s, 128, 8 * K * 2);
      tc::mma_f16_ts(tmem, tmem + 256 + 8 * s, bd, id, s > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tmem + ((uint32_t)((warp % 4) * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; j++) D[row * N + c0 + j] = v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int N>
int run_f16(int K) {
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K), D(M * N);
  srand(2);
  for (int i = 0; i < M * K; i++) { A[i] = __float2half((rand() / (float)RAND_MAX - 0.5f) * 4); Af[i] = __half2float(A[i]); }
  for (int i = 0; i < N * K; i++) { B[i] = __float2half((rand() / (float)RAND_MAX - 0.5f) * 4); Bf[i] = __half2float(B[i]); }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  size_t sm = (size_t)N * K * 2;
  cudaFuncSetAttribute(probe_f16_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  probe_f16_ts<N><<<1, 128, sm>>>(dA, dB, K, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("f16 N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M; i++)
    for (int j = 0; j < N; j++) {
      double s = 0;
      for (int k = 0; k < K; k++) s += (double)Af[i * K + k] * Bf[j * K + k];
      maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
      maxref = fmax(maxref, fabs(s));
    }
  printf("f16 TS N=%d K=%d: max|err| %.3e  max|ref| %.3e  %s\n", N, K, maxerr, maxref, maxerr < 1e-4 * maxref ? "OK" : "FAIL");
  return maxerr < 1e-4 * maxref ? 0 : 1;
}

static float tf32h(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xffffe000u;
  memcpy(&x, &u, 4);
  return x;
}

template <int N>
int run(int K, bool ts = false) {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& a : A) a = tf32h((rand() / (float)RAND_MAX - 0.5f) * 4);
  for (auto& b : B) b = tf32h((rand() / (float)RAND_MAX - 0.5f) * 4);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  size_t sm = (size_t)(M + N) * K * 4;
  if (ts) {
    cudaFuncSetAttribute(probe_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    probe_ts<N><<<1, 128, sm>>>(dA, dB, K, dD);
  } else {
    cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    probe<N><<<1, 128, sm>>>(dA, dB, K, dD);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M; i++)
    for (int j = 0; j < N; j++) {
      double s = 0;
      for (int k = 0; k < K; k++) s += (double)A[i * K + k] * B[j * K + k];
      maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
      maxref = fmax(maxref, fabs(s));
    }
  printf("%s N=%d K=%d: max|err| %.3e  max|ref| %.3e  %s\n", ts ? "TS" : "SS", N, K, maxerr, maxref, maxerr < 1e-4 * maxref ? "OK" : "FAIL");
  return maxerr < 1e-4 * maxref ? 0 : 1;
}

int main() {
  int bad = 0;
  bad |= run<128>(8);
  bad |= run<128>(32);
  bad |= run<256>(120);
  bad |= run<64>(16);
  bad |= run<128>(128, true);
  bad |= run<256>(64, true);
  bad |= run_f16<128>(128);
  bad |= run_f16<128>(16);
  return bad;
}
