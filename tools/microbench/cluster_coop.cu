// Can a cooperative launch carry a cluster dimension?  Latency of
// cluster.sync() vs grid.sync() in the same kernel.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k(int iters, unsigned long long *out) {
  cg::grid_group grid = cg::this_grid();
  cg::cluster_group cl = cg::this_cluster();
  unsigned long long t0, t1, t2;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (blockIdx.x < cl.num_blocks())
    for (int i = 0; i < iters; ++i) cl.sync();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  for (int i = 0; i < iters; ++i) grid.sync();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0, out[1] = t2 - t1, out[2] = cl.num_blocks();
}

int main() {
  unsigned long long *d;
  cudaMalloc(&d, 24);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    for (int per : {1, 2}) {
      int iters = 1000;
      cudaLaunchConfig_t cfg{};
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      attr[1].id = cudaLaunchAttributeClusterDimension;
      attr[1].val.clusterDim.x = cs, attr[1].val.clusterDim.y = 1, attr[1].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      int maxc = 0;
      cfg.gridDim = dim3(cs);
      cudaOccupancyMaxActiveClusters(&maxc, k, &cfg);
      int nb = (sms * per / cs) * cs;
      if (maxc * cs < nb) nb = maxc * cs;
      cfg.gridDim = dim3(nb);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k, iters, d);
      cudaError_t e2 = cudaDeviceSynchronize();
      unsigned long long h[3] = {0, 0, 0};
      cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
      printf("cluster %2d blocks %3d (max clusters %d): launch %s / %s  cluster.sync %.3f us  grid.sync %.3f us (n=%llu)\n", cs,
             nb, maxc, cudaGetErrorString(e), cudaGetErrorString(e2), h[0] / 1000.0 / iters, h[1] / 1000.0 / iters, h[2]);
    }
  }
  return 0;
}
