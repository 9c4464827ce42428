// Cost of cluster-wide barriers (cluster of 16 / 8 CTAs) vs block size; dev microbenchmark.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned long long gt(){unsigned long long t;asm volatile("mov.u64 %0,%globaltimer;":"=l"(t));return t;}
__global__ void k(int iters, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = gt() - t0;
}
__global__ void k2(int iters, unsigned long long* out) {  // arrive/wait split, only warp 0 participates per CTA after a named CTA barrier
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x < 32) {
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = gt() - t0;
}
int main() {
  unsigned long long* o; cudaMalloc(&o, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {8, 16}) for (int bs : {128, 512, 1024}) for (int var = 0; var < 1; ++var) {
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(bs); cfg.attrs = a; cfg.numAttrs = 1;
    int iters = 20000;
    cudaError_t e = var ? cudaLaunchKernelEx(&cfg, k2, iters, o) : cudaLaunchKernelEx(&cfg, k, iters, o);
    cudaDeviceSynchronize();
    unsigned long long h = 0; cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("cluster %2d block %4d %s: %s %.3f us per barrier\n", cs, bs, var ? "warp0 arrive/wait" : "cluster.sync()   ", cudaGetErrorString(e), h / 1e3 / iters);
  }
}
