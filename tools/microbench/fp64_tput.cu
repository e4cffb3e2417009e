// Throughput of DADD / DSETP / FADD with 8 independent chains per thread.
#include <cstdio>
template <int V>
__global__ void k(double x, float y, long long *cyc, double *o) {
  double a[8];
  float f[8];
  for (int u = 0; u < 8; ++u) a[u] = x + u, f[u] = y + u;
  long long t0 = clock64();
  int cnt = 0;
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (V == 0) a[u] = a[u] + 1e-300;
      if (V == 1) f[u] = f[u] + 1e-30f;
      if (V == 2) cnt += a[u] < x + i ? 1 : 0;
      if (V == 3) a[u] = fmin(a[u], a[(u + 1) & 7] + 1e-300);
    }
  }
  long long t1 = clock64();
  double s = cnt;
  for (int u = 0; u < 8; ++u) s += a[u] + f[u];
  o[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  long long *c; double *o;
  cudaMalloc(&c, 8); cudaMalloc(&o, 8 * 1024);
  const char *name[] = {"DADD", "FADD", "DSETP", "fmin(d)+DADD"};
  for (int threads : {32, 128, 256, 1024})
    for (int V = 0; V < 4; ++V) {
      for (int r = 0; r < 2; ++r) {
        if (V == 0) k<0><<<1, threads>>>(0.5, 0.5f, c, o);
        if (V == 1) k<1><<<1, threads>>>(0.5, 0.5f, c, o);
        if (V == 2) k<2><<<1, threads>>>(0.5, 0.5f, c, o);
        if (V == 3) k<3><<<1, threads>>>(0.5, 0.5f, c, o);
      }
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      const double ops = 256.0 * 8 * threads;
      printf("threads %4d %-14s %.2f lane-ops/cycle/SM\n", threads, name[V], ops / h);
    }
  return 0;
}
