// cp.async.bulk + mbarrier round trips (kernels.cuh helpers), growing toward chain_item's use.
#include "kernels.cuh"
#include <cstdio>
using namespace pp;
__global__ void k(const double *src, int n, double *out, int mode) {
  extern __shared__ __align__(16) unsigned char dsm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(dsm);
  double *buf = reinterpret_cast<double *>(dsm + 16 + 1376 + 2064 + 12288);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_proxy_async();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode == 0) {
      mbar_expect_tx(&bar[0], n * 8);
      bulk_g2s(buf, src, n * 8, &bar[0]);
    } else if (mode == 1) {
      mbar_expect_tx(&bar[0], bulk_bytes(src + 1, n - 2));
      bulk_range(buf, src + 1, n - 2, &bar[0]);
    } else {
      fence_proxy_async();
      mbar_expect_tx(&bar[0], bulk_bytes(src, n) + bulk_bytes(src + n, 16));
      bulk_range(buf, src, n, &bar[0]);
      bulk_range(buf + n + 16, src + n, 16, &bar[0]);
    }
  }
  mbar_wait(&bar[0], 0);
  out[threadIdx.x] = buf[threadIdx.x];
}
int main() {
  double *s, *o;
  cudaMalloc(&s, 65536); cudaMalloc(&o, 8192);
  static double h[8192];
  for (int i = 0; i < 8192; ++i) h[i] = i;
  cudaMemcpy(s, h, 65536, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {64, 256, 6400}) {
      k<<<1, 128, 120000>>>(s, n, o, mode);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, o, 1024, cudaMemcpyDeviceToHost);
      printf("mode %d n %d: %s  %g %g %g\n", mode, n, cudaGetErrorString(e), h[0], h[1], h[63]);
      fflush(stdout);
    }
  return 0;
}
