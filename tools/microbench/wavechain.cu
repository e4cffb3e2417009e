// Floor of one dependency wave in a cooperative kernel: barrier only, barrier
// + dependent L2 load/store by a few blocks, + a 36-step fold per cell.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void chain(int waves, int mode, int active, double *buf, int n, unsigned long long *out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double A[16][129];
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int w = 0; w < waves; ++w) {
    const double *src = buf + (size_t)(w & 1) * n;
    double *dst = buf + (size_t)((w + 1) & 1) * n;
    if (mode > 0 && blockIdx.x < active) {
      const int r = threadIdx.x >> 4, c = threadIdx.x & 15;
      double v0 = src[(blockIdx.x * 16 + r) * 36 + c], v1 = src[(blockIdx.x * 16 + r) * 36 + c + 16];
      double v2 = c < 4 ? src[(blockIdx.x * 16 + r) * 36 + c + 32] : 0.0;
      if (mode == 1) {
        dst[(blockIdx.x * 16 + r) * 36 + c] = v0 + v1 + v2;
      } else {
        A[r][c] = v0, A[r][c + 16] = v1;
        if (c < 4) A[r][c + 32] = v2;
        __syncthreads();
        double be = 0, bo = 0;
        int je = 0, jo = -1;
        for (int j = 0; j + 1 < 36; j += 2) {
          const double c0 = A[r][j] + A[c][j], c1 = A[r][j + 1] + A[c][j + 1];
          if (j == 0 || c0 < be) be = c0, je = j;
          if (jo < 0 || c1 < bo) bo = c1, jo = j + 1;
        }
        dst[(blockIdx.x * 16 + r) * 36 + c] = (bo < be ? bo : be) + je;
        __syncthreads();
      }
    }
    grid.sync();
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n = 1 << 20;
  double *buf;
  unsigned long long *d;
  cudaMalloc(&buf, 2 * n * sizeof(double));
  cudaMemset(buf, 0, 2 * n * sizeof(double));
  cudaMalloc(&d, 8);
  const int waves = 200;
  for (int per : {1, 2})
    for (int mode = 0; mode < 3; ++mode)
      for (int active : {1, 9, 100}) {
        int nb = sms * per;
        void *args[] = {(void *)&waves, (void *)&mode, (void *)&active, (void *)&buf, (void *)&n, (void *)&d};
        unsigned long long ns = 0;
        for (int rep = 0; rep < 3; ++rep) {
          cudaLaunchCooperativeKernel((void *)chain, nb, 256, args, 0, 0);
          cudaDeviceSynchronize();
          cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        }
        printf("blocks %3d mode %d (%s) active %3d: %.3f us per wave\n", nb, mode,
               mode == 0 ? "barrier" : mode == 1 ? "load+store" : "load+fold+store", active, ns / 1000.0 / waves);
      }
  return 0;
}
