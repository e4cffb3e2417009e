// Cost of one device-wide barrier inside a cooperative kernel: cg grid.sync()
// vs a hand-rolled sense-reversing barrier (one atomic per block), for grids
// of 1..3 blocks per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ unsigned int g_count, g_gen;

__device__ __forceinline__ void bar_custom(unsigned int nblocks, unsigned int &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = gen;
    __threadfence();
    if (atomicAdd(&g_count, 1u) == nblocks - 1) {
      g_count = 0;
      __threadfence();
      atomicExch(&g_gen, g + 1);
    } else {
      unsigned int cur;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(&g_gen));
      } while (cur == g);
    }
    gen = g + 1;
  }
  __syncthreads();
}

__global__ void k_cg(int iters, unsigned long long *out) {
  cg::grid_group grid = cg::this_grid();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) grid.sync();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

__global__ void k_custom(int iters, unsigned long long *out) {
  __shared__ unsigned int gen;
  if (threadIdx.x == 0) gen = *(volatile unsigned int *)&g_gen;
  __syncthreads();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) bar_custom(gridDim.x, gen);
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

int main() {
  unsigned long long *d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 1000;
  for (int per = 1; per <= 3; ++per) {
    for (int threads : {128, 256}) {
      int nb = sms * per;
      for (int which = 0; which < 2; ++which) {
        void *args[] = {(void *)&iters, (void *)&d};
        unsigned long long ns = 0;
        for (int rep = 0; rep < 3; ++rep) {
          cudaError_t e = cudaLaunchCooperativeKernel(which ? (void *)k_custom : (void *)k_cg, nb, threads, args, 0, 0);
          if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
          cudaDeviceSynchronize();
          cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-7s blocks %4d threads %3d: %.3f us per barrier\n", which ? "custom" : "cg", nb, threads, ns / 1000.0 / iters);
      }
    }
  }
  return 0;
}
