// Dependent-chain latency (cycles) of a few sm_100a instructions.
#include <cstdio>
__global__ void k(double *od, long long *ol, float *of, long long *cyc, int n, double x, float y) {
  __shared__ double sd[256];
  sd[threadIdx.x] = x;
  __syncthreads();
  double d = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) d = d + 1e-30;
  long long t1 = clock64();
  float f = y;
  for (int i = 0; i < n; ++i) f = f + 1e-30f;
  long long t2 = clock64();
  double e = x;
  for (int i = 0; i < n; ++i) e = e < 1.0 ? e + 1e-30 : e;  // DSETP + DADD + select
  long long t3 = clock64();
  int idx = threadIdx.x;
  double s = 0;
  for (int i = 0; i < n; ++i) { s = sd[idx]; idx = (int)(s) & 0; }  // LDS chain
  long long t4 = clock64();
  long long kk = (long long)x;
  for (int i = 0; i < n; ++i) kk = kk < 5 ? kk + 3 : kk - 1;  // int64 compare-select
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0, cyc[1] = t2 - t1, cyc[2] = t3 - t2, cyc[3] = t4 - t3, cyc[4] = t5 - t4;
  }
  od[threadIdx.x] = d + e + s;
  of[threadIdx.x] = f;
  ol[threadIdx.x] = kk;
}
int main() {
  double *od; long long *ol, *cyc; float *of;
  cudaMalloc(&od, 4096); cudaMalloc(&ol, 4096); cudaMalloc(&of, 4096); cudaMalloc(&cyc, 64);
  const int n = 1000;
  for (int threads : {32, 256}) {
    k<<<1, threads>>>(od, ol, of, cyc, n, 0.5, 0.5f);
    k<<<1, threads>>>(od, ol, of, cyc, n, 0.5, 0.5f);
    long long c[5];
    cudaMemcpy(c, cyc, 40, cudaMemcpyDeviceToHost);
    printf("threads %d: DADD %.1f  FADD %.1f  DSETP+DADD+SEL %.1f  LDS.64 %.1f  I64 cmp-sel %.1f cycles/step\n", threads,
           c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n);
  }
  return 0;
}
