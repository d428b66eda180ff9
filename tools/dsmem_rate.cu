// DSMEM store bandwidth probe: clusters of CL CTAs; every CTA writes a 64 KB block into each peer's
// shared memory (float4 stores), R rounds, cluster.sync() between rounds.  Reports bytes per SM cycle.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
template <int CL, int NB>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(512, 1) probe(int R, long long* out) {
  extern __shared__ float4 buf[];  // per source CTA slot: [CL][NB] float4
  cg::cluster_group cl = cg::this_cluster();
  const int me = cl.block_rank();
  for (int i = threadIdx.x; i < CL * NB; i += blockDim.x) buf[i] = make_float4(me, 0, 0, 0);
  cl.sync();
  long long t0 = clock64();
  for (int r = 0; r < R; r++) {
    for (int p = 0; p < CL; p++) {
      const int dst = (me + p) % CL;
      float4* remote = cl.map_shared_rank(buf, dst) + me * NB;
      for (int i = threadIdx.x; i < NB; i += blockDim.x) remote[i] = make_float4(r, i, me, p);
    }
    cl.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
}
template <int CL, int NB>
void run() {
  long long* d;
  cudaMalloc(&d, 8);
  const size_t sm = (size_t)CL * NB * 16;
  cudaFuncSetAttribute(probe<CL, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(probe<CL, NB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int R = 200;
  probe<CL, NB><<<CL * (144 / CL), 512, sm>>>(R, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)R * CL * NB * 16;  // written by one CTA (incl. its own slot)
  printf("cluster %d: %s  %.1f B/cycle/SM written (%lld cycles)\n", CL, cudaGetErrorString(e), bytes / c, c);
}
int main() { run<2, 4096>(); run<4, 2048>(); run<8, 1024>(); }
