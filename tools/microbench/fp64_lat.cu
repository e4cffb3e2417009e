// Latency (cycles per dependent step, one warp) of the operations on the
// chain scan's critical path: DADD, the (value, j) compare-select of
// keep_min, and one full candidate step (a + x, compare, select) with x read
// from shared memory; FP32 / INT64 variants for comparison.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_lat.cu -o fp64_lat
#include <cstdio>

template <int V>
__global__ void k(double x, long long *cyc, double *o, int *oj) {
  __shared__ double t2[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) t2[i] = 1.0 + (i * 7919 % 1024) * 1e-3;
  __syncthreads();
  double b = x, a = x;
  float f = static_cast<float>(x);
  long long ib = 1LL << 40;
  int j = 0;
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    if (V == 0) a = a + 1e-300;                                     // DADD chain
    if (V == 1) f = f + 1e-30f;                                     // FADD chain
    if (V == 2) {                                                   // keep_min: compare-select on (b, j)
      const double c = t2[i & 1023];
      const bool t = c < b || (c == b && i < j);
      b = t ? c : b, j = t ? i : j;
    }
    if (V == 3) {                                                   // candidate step: (a + x) then keep_min
      const double c = a + t2[(i * 33) & 1023];
      if (c < b) b = c, j = i;
    }
    if (V == 4) {                                                   // same with int64 keys
      const long long c = static_cast<long long>(t2[(i * 33) & 1023] * 1e6) + ib;
      if (c < ib) ib = c, j = i;
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  o[threadIdx.x] = a + b + f + static_cast<double>(ib);
  oj[threadIdx.x] = j;
}

int main() {
  long long *cyc;
  double *o;
  int *oj;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&o, 32 * 8);
  cudaMalloc(&oj, 32 * 4);
  const char *names[] = {"DADD chain", "FADD chain", "keep_min (value, j) from smem", "a + x, compare-select",
                         "int64 key compare-select"};
  for (int v = 0; v < 5; ++v) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      if (v == 0) k<0><<<1, 32>>>(1.0, cyc, o, oj);
      if (v == 1) k<1><<<1, 32>>>(1.0, cyc, o, oj);
      if (v == 2) k<2><<<1, 32>>>(1.0, cyc, o, oj);
      if (v == 3) k<3><<<1, 32>>>(1.0, cyc, o, oj);
      if (v == 4) k<4><<<1, 32>>>(1.0, cyc, o, oj);
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-32s %6.1f cycles / step\n", names[v], h / 1024.0);
  }
  return 0;
}
