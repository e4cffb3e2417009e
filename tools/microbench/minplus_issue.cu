// Instruction-throughput microbenchmark for the Eq. 2 (min,+) inner loop on sm_100a.
// Each CTA keeps a 128x128 output tile in registers (8x8 per thread, 256 threads)
// and sweeps a shared-memory-resident K panel R times, so the measurement is the
// issue rate of the add+min instruction mix, not memory.  Variants:
//   f32      FADD + FMNMX            (2 instr / cell update)
//   f32x2    FADD2 + FMNMX3          (1 instr / cell update)
//   s32      VIADDMNMX               (1 instr / cell update)
//   ffma     FFMA                    (peak reference, 1 instr / "cell")
//   f64      DADD + DMNMX
//   f32x2a / s32a: as above plus the chunked lowest-index argmin bookkeeping.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define BK 32
#define TILE 128

__device__ __forceinline__ float min3f(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

__device__ unsigned long long g_clk[2];

template <int V>
__global__ void __launch_bounds__(256, 1) bench(const float *gA, const float *gB, float *out, int R) {
  if (blockIdx.x == 0 && threadIdx.x == 0) g_clk[0] = clock64();
  __shared__ __align__(16) float As[BK][TILE];
  __shared__ __align__(16) float Bs[BK][TILE];
  for (int t = threadIdx.x; t < BK * TILE; t += 256) {
    (&As[0][0])[t] = gA[t];
    (&Bs[0][0])[t] = gB[t];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ty = (w >> 1) * 4 + (lane >> 3), tx = (w & 1) * 8 + (lane & 7);
  float acc = 0.f;
  if constexpr (V == 0 || V == 3) {
    float best[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) best[r][c] = (V == 3) ? 0.f : 3.0e38f;
    for (int it = 0; it < R; ++it) {
      asm volatile("" ::: "memory");
#pragma unroll 4
      for (int j = 0; j < BK; ++j) {
        float a[8], b[8];
        *(float4 *)&a[0] = *(const float4 *)&As[j][ty * 8];
        *(float4 *)&a[4] = *(const float4 *)&As[j][ty * 8 + 4];
        *(float4 *)&b[0] = *(const float4 *)&Bs[j][tx * 8];
        *(float4 *)&b[4] = *(const float4 *)&Bs[j][tx * 8 + 4];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if constexpr (V == 0) best[r][c] = fminf(best[r][c], a[r] + b[c]);
            else best[r][c] = fmaf(a[r], b[c], best[r][c]);
          }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc += best[r][c];
  } else if constexpr (V == 1 || V == 5) {
    // pairs (j, j+1): As viewed as float2 [BK/2][TILE] with element (jp, i) = (a[i][2jp], a[i][2jp+1])
    const float2 *A2 = reinterpret_cast<const float2 *>(&As[0][0]);
    const float2 *B2 = reinterpret_cast<const float2 *>(&Bs[0][0]);
    float best[8][8];
    float m[8][8];
    int idx[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) { best[r][c] = 3.0e38f; idx[r][c] = 0; }
    for (int it = 0; it < R; ++it) {
      asm volatile("" ::: "memory");
#pragma unroll 2
      for (int jp = 0; jp < BK / 2; ++jp) {
        float2 a[8], b[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          *(float4 *)&a[2 * q] = *(const float4 *)&A2[jp * TILE + ty * 8 + 2 * q];
          *(float4 *)&b[2 * q] = *(const float4 *)&B2[jp * TILE + tx * 8 + 2 * q];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float2 s = __fadd2_rn(a[r], b[c]);
            if constexpr (V == 1) best[r][c] = min3f(best[r][c], s.x, s.y);
            else m[r][c] = (jp == 0) ? fminf(s.x, s.y) : min3f(m[r][c], s.x, s.y);
          }
      }
      if constexpr (V == 5) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (m[r][c] < best[r][c]) { best[r][c] = m[r][c]; idx[r][c] = it; }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc += best[r][c] + (float)idx[r][c];
  } else if constexpr (V == 2 || V == 6) {
    const int *Ai = reinterpret_cast<const int *>(&As[0][0]);
    const int *Bi = reinterpret_cast<const int *>(&Bs[0][0]);
    int best[8][8], m[8][8], idx[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) { best[r][c] = 0x3fffffff; idx[r][c] = 0; }
    for (int it = 0; it < R; ++it) {
      asm volatile("" ::: "memory");
#pragma unroll 4
      for (int j = 0; j < BK; ++j) {
        int a[8], b[8];
        *(int4 *)&a[0] = *(const int4 *)&Ai[j * TILE + ty * 8];
        *(int4 *)&a[4] = *(const int4 *)&Ai[j * TILE + ty * 8 + 4];
        *(int4 *)&b[0] = *(const int4 *)&Bi[j * TILE + tx * 8];
        *(int4 *)&b[4] = *(const int4 *)&Bi[j * TILE + tx * 8 + 4];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if constexpr (V == 2) best[r][c] = __viaddmin_s32(a[r], b[c], best[r][c]);
            else m[r][c] = (j == 0) ? a[r] + b[c] : __viaddmin_s32(a[r], b[c], m[r][c]);
          }
      }
      if constexpr (V == 6) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (m[r][c] < best[r][c]) { best[r][c] = m[r][c]; idx[r][c] = it; }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc += (float)(best[r][c] + idx[r][c]);
  } else if constexpr (V == 7 || V == 8) {
    // 16-bit pairs: a duplicated in both halves (int32 words), b = two adjacent columns per word
    const unsigned *Au = reinterpret_cast<const unsigned *>(&As[0][0]);
    const unsigned *Bu = reinterpret_cast<const unsigned *>(&Bs[0][0]);
    unsigned best[8][4], m[8][4], idx[8][4];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) best[r][c] = 0x7fff7fffu, idx[r][c] = 0;
    for (int it = 0; it < R; ++it) {
      asm volatile("" ::: "memory");
      const unsigned cid = (unsigned)it * 0x10001u;
#pragma unroll 4
      for (int j = 0; j < BK; ++j) {
        unsigned a[8], b[4];
        *(uint4 *)&a[0] = *(const uint4 *)&Au[j * TILE + ty * 8];
        *(uint4 *)&a[4] = *(const uint4 *)&Au[j * TILE + ty * 8 + 4];
        *(uint4 *)&b[0] = *(const uint4 *)&Bu[j * TILE + tx * 4];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if constexpr (V == 7) best[r][c] = __viaddmin_s16x2(a[r], b[c], best[r][c]);
            else m[r][c] = (j == 0) ? __vadd2(a[r], b[c]) : __viaddmin_s16x2(a[r], b[c], m[r][c]);
          }
      }
      if constexpr (V == 8) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const unsigned lt = __vcmplts2(m[r][c], best[r][c]);
            best[r][c] = __vmins2(best[r][c], m[r][c]);
            idx[r][c] = (idx[r][c] & ~lt) | (cid & lt);
          }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc += (float)(best[r][c] ^ idx[r][c]);
  } else if constexpr (V == 4) {
    double best[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) best[r][c] = 1e300;
    for (int it = 0; it < R; ++it) {
      asm volatile("" ::: "memory");
#pragma unroll 4
      for (int j = 0; j < BK; ++j) {
        double a[4], b[8];
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = As[j][ty * 8 + r];
#pragma unroll
        for (int c = 0; c < 8; ++c) b[c] = Bs[j][tx * 8 + c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) best[r][c] = fmin(best[r][c], a[r] + b[c]);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc += (float)best[r][c];
  }
  out[blockIdx.x * 256 + threadIdx.x] = acc;
  if (blockIdx.x == 0 && threadIdx.x == 0) g_clk[1] = clock64();
}

template <int V>
double run(const char *name, const float *dA, const float *dB, float *dO, int sms, int R, double cells_per_thread_per_j) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bench<V>, 256, 0);
  int grid = sms * occ;
  bench<V><<<grid, 256>>>(dA, dB, dO, 4);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  bench<V><<<grid, 256>>>(dA, dB, dO, R);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double cells = (double)grid * 256 * cells_per_thread_per_j * BK * R;
  double rate = cells / (ms * 1e-3);
  unsigned long long clk[2];
  cudaMemcpyFromSymbol(clk, g_clk, sizeof clk);
  const double cyc = (double)(clk[1] - clk[0]);  // block 0's span ~ whole kernel (one wave)
  const double mhz = cyc / (ms * 1e3);
  printf("{\"variant\": \"%s\", \"occ\": %d, \"ms\": %.3f, \"cells_per_s\": %.4e, \"sm_mhz_est\": %.0f, "
         "\"cells_per_clk_per_sm\": %.2f, \"err\": \"%s\"}\n",
         name, occ, ms, rate, mhz, cells / cyc / sms, cudaGetErrorString(cudaGetLastError()));
  return rate;
}

int main(int argc, char **argv) {
  int R = argc > 1 ? atoi(argv[1]) : 20000;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, sms, p.clockRate);
  float *dA, *dB, *dO;
  cudaMalloc(&dA, BK * TILE * 4);
  cudaMalloc(&dB, BK * TILE * 4);
  cudaMalloc(&dO, sms * 256 * 4 * 4);
  float h[BK * TILE];
  for (int i = 0; i < BK * TILE; ++i) h[i] = (float)(rand() % 641) / 64.0f;
  cudaMemcpy(dA, h, sizeof h, cudaMemcpyHostToDevice);
  for (int i = 0; i < BK * TILE; ++i) h[i] = (float)(rand() % 641) / 64.0f;
  cudaMemcpy(dB, h, sizeof h, cudaMemcpyHostToDevice);
  run<0>("f32 FADD+FMNMX", dA, dB, dO, sms, R, 64);
  run<1>("f32x2 FADD2+FMNMX3", dA, dB, dO, sms, R, 64);
  run<5>("f32x2 + chunk argmin", dA, dB, dO, sms, R, 64);
  run<2>("s32 VIADDMNMX", dA, dB, dO, sms, R, 64);
  run<6>("s32 VIADDMNMX + chunk argmin", dA, dB, dO, sms, R, 64);
  run<3>("ffma (peak ref)", dA, dB, dO, sms, R, 64);
  run<4>("f64 DADD+DMNMX", dA, dB, dO, sms, R / 4, 32);
  run<7>("s16x2 VIADDMNMX.S16x2", dA, dB, dO, sms, R, 64);
  run<8>("s16x2 + chunk argmin", dA, dB, dO, sms, R, 64);
  return 0;
}
