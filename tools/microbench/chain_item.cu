// One chain item (kernels.cuh chain_item) in isolation: a VGG-like chain of
// n folds (nu x nw x nv doubles), one row per item, cycles per fold.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++20 -I../../paper_1802_04924_b200/csrc -I../../include
#include "kernels.cuh"
#include <cstdio>
#include <vector>
using namespace pp;

__global__ void k(const ChainDesc *chains, const FoldDesc<double> *cf, int items, long long *cyc, uint64_t *tr) {
  extern __shared__ __align__(16) unsigned char smem[];
  long long t0 = clock64();
  for (int it = blockIdx.x; it < items; it += gridDim.x) chain_item<double>(chains, 1, cf, it, smem, blockIdx.x == 0 ? tr : nullptr);
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main(int argc, char **argv) {
  const int n = 19, nu = 53, nw = 80, nv = 80;
  const int rows = argc > 1 ? atoi(argv[1]) : 1;
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
  const int buf = (nw * (nv + 2) + 3) & ~3;
  ChainDesc c{0, n, nu, rows, 0, buf, 0};
  ChainDesc *dc;
  cudaMalloc(&dc, sizeof(c));
  cudaMemcpy(dc, &c, sizeof(c), cudaMemcpyHostToDevice);
  const size_t sm = chain_smem_bytes<double>(rows, buf, n);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  long long *cyc;
  cudaMalloc(&cyc, 8);
  const int items = (nu + rows - 1) / rows;
  uint64_t *tr;
  cudaMalloc(&tr, 16 * 8);
  for (int r = 0; r < 3; ++r) k<<<items, 256, sm>>>(dc, df, items, cyc, tr);
  cudaError_t e = cudaDeviceSynchronize();
  long long hc;
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("rows %d smem %zu: %s, %.0f cycles per fold (%.2f us at 1.9 GHz)\n", rows, sm, cudaGetErrorString(e), hc / double(n),
         hc / double(n) / 1900.0);
  uint64_t t[16];
  cudaMemcpy(t, tr, 128, cudaMemcpyDeviceToHost);
  for (int q = 1; q < 4; ++q)
    printf("fold %d: stage+wait %lld  A' %lld  scan %lld  (total %lld cycles)\n", q, (long long)(t[4 * q + 1] - t[4 * q]),
           (long long)(t[4 * q + 2] - t[4 * q + 1]), (long long)(t[4 * q + 3] - t[4 * q + 2]), (long long)(t[4 * q + 3] - t[4 * q]));
  return 0;
}
