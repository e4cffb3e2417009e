// Latency of one panel tile (kernels.cuh panel_tile_r) in isolation: one
// block, stamps after each phase, repeated.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I../../paper_1802_04924_b200/csrc -I../../include
#include "kernels.cuh"
#include <cstdio>
#include <vector>
using namespace pp;

__device__ long long g_clk[2];
__device__ unsigned long long g_ns[2];

template <int R>
__global__ void k(FoldDesc<double> f, int reps, uint64_t *tr) {
  __shared__ WaveSmem<double> sm;
  if (threadIdx.x == 0) g_clk[0] = clock64(), g_ns[0] = trace_ns();
  for (int r = 0; r < reps; ++r) {
    uint64_t *t = tr + 8 * r;
    if (threadIdx.x == 0) t[0] = trace_ns();
    panel_tile_r<double, R>(f, 0, 0, sm.p, t);
  }
  if (threadIdx.x == 0) g_clk[1] = clock64(), g_ns[1] = trace_ns();
}

int main() {
  const int nu = 35, nw = 36, nv = 36;
  std::vector<double> h(nu * nw + nw * nv + nw, 1.0);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (i * 7919 % 1000) * 0.001;
  double *d;
  cudaMalloc(&d, (h.size() + nu * nv) * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  uint16_t *am;
  cudaMalloc(&am, nu * nv * 2);
  uint64_t *tr;
  const int reps = 20;
  cudaMalloc(&tr, reps * 8 * 8);
  FoldDesc<double> f{};
  f.t1 = d, f.t2 = d + nu * nw, f.w = d + nu * nw + nw * nv, f.out = d + h.size(), f.am = am;
  f.nu = nu, f.nw = nw, f.nv = nv, f.late = 0;
  for (int R : {16, 8, 4}) {
    f.small = R == 16 ? kPanel16 : R == 8 ? kPanel8 : kPanel4;
    f.tiles_k = (nv + R - 1) / R;
    for (int it = 0; it < 2; ++it) {
      if (R == 16) k<16><<<1, 256>>>(f, reps, tr);
      if (R == 8) k<8><<<1, 256>>>(f, reps, tr);
      if (R == 4) k<4><<<1, 256>>>(f, reps, tr);
      cudaDeviceSynchronize();
    }
    long long clk[2];
    unsigned long long ns[2];
    cudaMemcpyFromSymbol(clk, g_clk, 16);
    cudaMemcpyFromSymbol(ns, g_ns, 16);
    printf("R=%d SM clock over the run: %.0f MHz\n", R, 1e3 * double(clk[1] - clk[0]) / double(ns[1] - ns[0]));
    std::vector<uint64_t> t(reps * 8);
    cudaMemcpy(t.data(), tr, t.size() * 8, cudaMemcpyDeviceToHost);
    for (int r : {0, 1, 10, 19}) {
      const uint64_t *x = &t[8 * r];
      printf("R=%2d rep %2d: tile %5lld loaded %5lld scanned %5lld merged %5lld stored %5lld ns\n", R, r,
             (long long)(x[7] - x[0]), (long long)(x[1] - x[0]), (long long)(x[5] - x[0]), (long long)(x[6] - x[0]),
             (long long)(x[2] - x[0]));
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
