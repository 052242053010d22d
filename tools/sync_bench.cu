// Microbenchmark: cost of cluster.sync() / __syncthreads() / DSMEM push per iteration.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_cluster(int iters, int mode, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double slot[16][32];
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    if (mode & 1) __syncthreads();
    if (mode & 2) {
      if (threadIdx.x < 32)
        for (int c = 0; c < (int)cl.num_blocks(); ++c) *cl.map_shared_rank(&slot[cl.block_rank()][threadIdx.x], c) = acc;
    }
    if (mode & 4) cl.sync();
    if (mode & 8) { __syncthreads(); }
    acc += slot[i & 15][threadIdx.x & 31];
  }
  if (acc == 1.2345) out[0] = acc;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C : {1, 4, 8, 16}) for (int mode : {1, 4, 5, 7, 15}) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(C); cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int iters = 10000;
    cudaLaunchKernelEx(&cfg, k_cluster, iters, mode, out); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); cudaLaunchKernelEx(&cfg, k_cluster, iters, mode, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("C=%2d mode=%2d (1=sync,2=push,4=cluster.sync,8=sync2): %.3f us/iter  err=%s\n", C, mode, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
