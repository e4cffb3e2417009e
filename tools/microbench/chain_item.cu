// One chain item (kernels.cuh chain_item) in isolation: a VGG-like chain of
// n folds (nu x nw x nv doubles), one row per item, cycles per fold.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++20 -I../../paper_1802_04924_b200/csrc -I../../include
#include "kernels.cuh"
#include <cstdio>
#include <vector>
#include <cstring>
#include <unistd.h>
using namespace pp;

__global__ void k(const ChainDesc *chains, const FoldDesc<double> *cf, int items, long long *cyc, uint64_t *tr, size_t stage) {
  extern __shared__ __align__(16) unsigned char smem[];
  long long t0 = clock64();
  for (int it = blockIdx.x; it < items; it += gridDim.x) chain_item<double>(chains, 1, cf, it, smem, stage, blockIdx.x == 0 ? tr : nullptr);
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main(int argc, char **argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 1;
  const int n = argc > 2 ? atoi(argv[2]) : 19, nu = 53;
  const int nw = argc > 3 ? atoi(argv[3]) : 80, nv = nw;
  std::vector<double> h(static_cast<size_t>(n) * (nw * nv + nw) + nu * nw);
  for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 7919) % 1000) * 0.001;
  double *d, *out;
  uint16_t *am;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&out, nu * nv * 8);
  cudaMalloc(&am, static_cast<size_t>(n) * nu * nv * 2);
  std::vector<FoldDesc<double>> f(n);
  for (int q = 0; q < n; ++q) {
    f[q] = FoldDesc<double>{};
    f[q].t1 = d + static_cast<size_t>(n) * (nw * nv + nw);
    f[q].t2 = d + static_cast<size_t>(q) * (nw * nv + nw);
    f[q].w = f[q].t2 + nw * nv;
    f[q].out = out;
    f[q].am = am + static_cast<size_t>(q) * nu * nv;
    f[q].nu = nu, f[q].nw = nw, f[q].nv = nv;
  }
  FoldDesc<double> *df;
  cudaMalloc(&df, n * sizeof(FoldDesc<double>));
  cudaMemcpy(df, f.data(), n * sizeof(FoldDesc<double>), cudaMemcpyHostToDevice);
  ChainDesc c{0, n, nu, rows, 0};
  ChainDesc *dc;
  cudaMalloc(&dc, sizeof(c));
  cudaMemcpy(dc, &c, sizeof(c), cudaMemcpyHostToDevice);
  const size_t stage = chain_stage_bytes<double>(nw, nv);
  const size_t sm = chain_smem_bytes<double>(rows, n, stage, false);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  long long *cyc;
  cudaMalloc(&cyc, 8);
  const int items = (nu + rows - 1) / rows;
  uint64_t *tr;
  cudaHostAlloc(&tr, 32 * 8, cudaHostAllocMapped);
  memset(tr, 0, 256);
  k<<<items, 256, sm>>>(dc, df, items, cyc, tr, stage);
  for (int spin = 0; spin < 20 && cudaStreamQuery(0) == cudaErrorNotReady; ++spin) usleep(100000);
  if (cudaStreamQuery(0) == cudaErrorNotReady) {
    printf("HANG: stamps");
    for (int q = 0; q < 16; ++q) printf(" %llu", (unsigned long long)((volatile uint64_t *)tr)[q]);
    printf("\n");
    fflush(stdout);
    _exit(3);
  }
  for (int r = 0; r < 2; ++r) k<<<items, 256, sm>>>(dc, df, items, cyc, tr, stage);
  cudaError_t e = cudaDeviceSynchronize();
  long long hc;
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("rows %d smem %zu: %s, %.0f cycles per fold (%.2f us at 1.9 GHz)\n", rows, sm, cudaGetErrorString(e), hc / double(n),
         hc / double(n) / 1900.0);
  uint64_t t[32];
  memcpy(t, tr, 256);
  printf("stage issue: %lld %lld cycles; merge phase ends %lld after scan\n", (long long)(t[19] - t[18]), (long long)(t[21] - t[20]),
         (long long)(t[8] - t[7]));
  for (int q = 1; q < 3; ++q)
    printf("fold %d: wait %lld  A' %lld  scan %lld  (total %lld cycles)\n", q, (long long)(t[4 * q + 1] - t[4 * q]),
           (long long)(t[4 * q + 2] - t[4 * q + 1]), (long long)(t[4 * q + 3] - t[4 * q + 2]), (long long)(t[4 * (q + 1)] - t[4 * q]));
  return 0;
}
