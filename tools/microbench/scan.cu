// Cycles per candidate of an argmin scan over shared memory, by variant.
#include <climits>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ long long key(double x) {
  long long b = __double_as_longlong(x);
  b = b == LLONG_MIN ? 0 : b;
  return b ^ ((b >> 63) & LLONG_MAX);
}

template <int V>
__global__ void k(int nw, int G, long long *cyc, double *out, int *oj) {
  __shared__ double A[128], B[128 * 17];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) A[i] = (i * 37 % 101) * 0.01;
  for (int i = threadIdx.x; i < 128 * 17; i += blockDim.x) B[i] = (i * 53 % 97) * 0.01;
  __syncthreads();
  const int g = threadIdx.x % G, tx = (threadIdx.x / G) % 16;
  long long t0 = clock64();
  double bv = 0;
  int bj = -1;
  if (V == 0) { // doubles, plain loop
    for (int j = g; j < nw; j += G) {
      const double c = A[j] + B[j * 17 + tx];
      if (bj < 0 || c < bv) bv = c, bj = j;
    }
  } else if (V == 1) { // keys, unrolled x4, two chains
    long long k0 = LLONG_MAX, k1 = LLONG_MAX;
    int j0 = INT_MAX, j1 = INT_MAX;
    int j = g;
    for (; j + 3 * G < nw; j += 4 * G) {
      long long cc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) cc[u] = key(A[j + u * G] + B[(j + u * G) * 17 + tx]);
#pragma unroll
      for (int u = 0; u < 4; u += 2) {
        if (cc[u] < k0) k0 = cc[u], j0 = j + u * G;
        if (cc[u + 1] < k1) k1 = cc[u + 1], j1 = j + (u + 1) * G;
      }
    }
    for (; j < nw; j += G) {
      const long long c = key(A[j] + B[j * 17 + tx]);
      if (c < k0) k0 = c, j0 = j;
    }
    if (k1 < k0 || (k1 == k0 && j1 < j0)) k0 = k1, j0 = j1;
    bv = __longlong_as_double(k0), bj = j0;
  } else if (V == 2) { // doubles, unrolled x4 two chains
    double b0 = 0, b1 = 0;
    int j0 = -1, j1 = -1;
    int j = g;
    for (; j + 3 * G < nw; j += 4 * G) {
      double cc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) cc[u] = A[j + u * G] + B[(j + u * G) * 17 + tx];
#pragma unroll
      for (int u = 0; u < 4; u += 2) {
        if (j0 < 0 || cc[u] < b0) b0 = cc[u], j0 = j + u * G;
        if (j1 < 0 || cc[u + 1] < b1) b1 = cc[u + 1], j1 = j + (u + 1) * G;
      }
    }
    bv = b0 < b1 ? b0 : b1, bj = j0;
  } else if (V == 4) { // doubles, 8 independent (value, j) chains
    double b[8];
    int jb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) b[u] = __longlong_as_double(0x7ff0000000000000LL), jb[u] = INT_MAX;
    int j = g;
    for (; j + 7 * G < nw; j += 8 * G) {
      double cc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cc[u] = A[j + u * G] + B[(j + u * G) * 17 + tx];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (cc[u] < b[u]) b[u] = cc[u], jb[u] = j + u * G;
    }
    for (; j < nw; j += G) {
      const double c = A[j] + B[j * 17 + tx];
      if (c < b[0] || (c == b[0] && j < jb[0])) b[0] = c, jb[0] = j;
    }
    double bvv = b[0];
    int bjj = jb[0];
#pragma unroll
    for (int u = 1; u < 8; ++u)
      if (b[u] < bvv || (b[u] == bvv && jb[u] < bjj)) bvv = b[u], bjj = jb[u];
    bv = bvv, bj = bjj;
  } else if (V == 5) { // two passes: fmin with 8 accumulators, then first j equal to the min
    double m[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) m[u] = __longlong_as_double(0x7ff0000000000000LL);
    int j = g;
    for (; j + 7 * G < nw; j += 8 * G) {
#pragma unroll
      for (int u = 0; u < 8; ++u) m[u] = fmin(m[u], A[j + u * G] + B[(j + u * G) * 17 + tx]);
    }
    for (; j < nw; j += G) m[0] = fmin(m[0], A[j] + B[j * 17 + tx]);
#pragma unroll
    for (int u = 1; u < 8; ++u) m[0] = fmin(m[0], m[u]);
    int jf = INT_MAX;
    for (j = g; j < nw; j += G)
      if (A[j] + B[j * 17 + tx] == m[0]) { jf = j; break; }
    bv = m[0], bj = jf;
  } else { // fixed bounds (nw = 64 known)
    double b0 = 0;
    int j0 = -1;
#pragma unroll 8
    for (int j = 0; j < 64; ++j) {
      const double c = A[j] + B[j * 17 + tx];
      if (j0 < 0 || c < b0) b0 = c, j0 = j;
    }
    bv = b0, bj = j0;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  out[threadIdx.x] = bv;
  oj[threadIdx.x] = bj;
}

int main() {
  long long *c; double *o; int *oj;
  cudaMalloc(&c, 8); cudaMalloc(&o, 8192); cudaMalloc(&oj, 4096);
  for (int threads : {32, 256})
    for (int V = 0; V < 6; ++V) {
      const int nw = 64, G = 1;
      for (int r = 0; r < 2; ++r) {
        if (V == 0) k<0><<<1, threads>>>(nw, G, c, o, oj);
        if (V == 1) k<1><<<1, threads>>>(nw, G, c, o, oj);
        if (V == 2) k<2><<<1, threads>>>(nw, G, c, o, oj);
        if (V == 3) k<3><<<1, threads>>>(nw, G, c, o, oj);
        if (V == 4) k<4><<<1, threads>>>(nw, G, c, o, oj);
        if (V == 5) k<5><<<1, threads>>>(nw, G, c, o, oj);
      }
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("threads %3d variant %d: %.1f cycles per candidate\n", threads, V, h / 64.0);
    }
  return 0;
}
