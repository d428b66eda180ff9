// Phase profile of sweep_posterior_kernel (clock64 per phase, thread 0 of each CTA):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTVK_SWEEP_PROF -o tools/sweep_prof \
//        tools/sweep_prof.cu paper_1906_08556_b200/csrc/capi.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1906_08556_b200/csrc/posterior.cu"

int main(int argc, char** argv) {
  const int U = argc > 1 ? atoi(argv[1]) : 1024, D = argc > 2 ? atoi(argv[2]) : 400;
  const int grid = argc > 3 ? atoi(argv[3]) : 0;  // 0: tvk_posterior's own launch
  const int64_t P = (int64_t)D * (D + 1) / 2;
  std::vector<double> h((size_t)U * P), hb((size_t)U * D);
  srand(1);
  for (int u = 0; u < U; u++)
    for (int i = 0; i < D; i++) {
      hb[(size_t)u * D + i] = rand() / (double)RAND_MAX - 0.5;
      for (int j = 0; j <= i; j++)
        h[(size_t)u * P + (size_t)i * (i + 1) / 2 + j] = i == j ? 1.0 + 0.01 * D : 0.01 * (rand() / (double)RAND_MAX - 0.5);
    }
  double *L, *L0, *b, *phi, *ld, *bp;
  int* st;
  cudaMalloc(&L, sizeof(double) * U * P);
  cudaMalloc(&L0, sizeof(double) * U * P);
  cudaMalloc(&b, sizeof(double) * U * D);
  cudaMalloc(&phi, sizeof(double) * U * D);
  cudaMalloc(&ld, sizeof(double) * U);
  cudaMalloc(&bp, sizeof(double) * U);
  cudaMalloc(&st, sizeof(int) * U);
  cudaMemcpy(L0, h.data(), sizeof(double) * U * P, cudaMemcpyHostToDevice);
  cudaMemcpy(b, hb.data(), sizeof(double) * U * D, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; rep++) {
    cudaMemcpy(L, L0, sizeof(double) * U * P, cudaMemcpyDeviceToDevice);
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(tvk::g_sweep_prof, z, sizeof(z));
    cudaEventRecord(e0);
    int rc = 0;
    if (grid > 0) {
      cudaFuncSetAttribute(tvk::sweep_posterior_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tvk::sw::smem_bytes());
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(tvk::sw::NT);
      cfg.dynamicSmemBytes = tvk::sw::smem_bytes();
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = tvk::sw::CL;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, tvk::sweep_posterior_kernel, (const double*)L, L, (const double*)b, U, D, 3, phi, ld, bp, st);
    } else {
      rc = tvk_posterior(L, b, U, D, 3, phi, L, ld, bp, st, nullptr, 0, nullptr);
    }
    if (rc) printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
    unsigned long long pr[8];
    cudaMemcpyFromSymbol(pr, tvk::g_sweep_prof, sizeof(pr));
    double tot = 0;
    for (int i = 0; i < 6; i++) tot += pr[i];
    printf("rc=%d %.3f ms (%.2f TF)  per-matrix cycles: load %.0f pivot %.0f B %.0f vr %.0f tiles %.0f other %.0f\n", rc,
           ms, (double)U * D * D * D / ms / 1e9, pr[0] / (double)U, pr[1] / (double)U, pr[2] / (double)U,
           pr[3] / (double)U, pr[4] / (double)U, pr[5] / (double)U);
  }
  return 0;
}
