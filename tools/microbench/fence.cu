// Cost of __threadfence() at a grid barrier when blocks arrive staggered:
// each block spins for a block-dependent time (optionally issuing global loads
// or stores), then stamps arrival, fence, atomic and release with %globaltimer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fence.cu -o fence
#include <cstdio>
#include <vector>
#include <algorithm>

__device__ unsigned int g_bar;

__device__ __forceinline__ unsigned long long now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// mode 0: pure spin; 1: spin + loads; 2: spin + stores; 3: spin with the
// co-resident blocks storing while thread 0 fences
__global__ void k(int mode, double *buf, unsigned long long *ts) {
  const unsigned long long t0 = now();
  const unsigned long long until = t0 + 2000 + (blockIdx.x * 7919u % 16) * 1000;
  double acc = 0;
  int it = 0;
  while (now() < until) {
    const size_t i = (static_cast<size_t>(blockIdx.x) * 256 + threadIdx.x + static_cast<size_t>(it) * 296 * 256) % (1 << 22);
    if (mode == 1) acc += buf[i];
    if (mode == 2) buf[i] = acc + it;
    ++it;
  }
  if (acc == -1.0) buf[0] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long *t = ts + 4 * blockIdx.x;
    t[0] = now();
    __threadfence();
    t[1] = now();
    const unsigned int nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    const unsigned int old = atomicAdd(&g_bar, nb);
    t[2] = now();
    unsigned int cur;
    for (;;) {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&g_bar) : "memory");
      if ((old ^ cur) & 0x80000000u) break;
      __nanosleep(20);
    }
    __threadfence();
    t[3] = now();
  }
  __syncthreads();
}

int main() {
  const int nb = 296;
  double *buf;
  unsigned long long *ts;
  cudaMalloc(&buf, (1 << 22) * sizeof(double));
  cudaMemset(buf, 0, (1 << 22) * sizeof(double));
  cudaMalloc(&ts, nb * 4 * sizeof(unsigned long long));
  for (int mode = 0; mode < 3; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      void *args[] = {&mode, &buf, &ts};
      cudaLaunchCooperativeKernel((void *)k, nb, 256, args, 0, 0);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
      std::vector<unsigned long long> h(nb * 4);
      cudaMemcpy(h.data(), ts, h.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long base = ~0ull, lastarr = 0, lastfence = 0, firstrel = ~0ull, maxrel = 0;
      double maxf = 0, sumf = 0;
      for (int b = 0; b < nb; ++b) {
        base = std::min(base, h[4 * b]);
        lastarr = std::max(lastarr, h[4 * b]);
        lastfence = std::max(lastfence, h[4 * b + 1]);
        firstrel = std::min(firstrel, h[4 * b + 3]);
        maxrel = std::max(maxrel, h[4 * b + 3]);
        const double f = double(h[4 * b + 1] - h[4 * b]);
        maxf = std::max(maxf, f), sumf += f;
      }
      printf("mode %d: first arrive 0, last arrive %llu, last fence done %llu, release %llu..%llu ns; fence max %.0f mean %.0f ns\n",
             mode, lastarr - base, lastfence - base, firstrel - base, maxrel - base, maxf, sumf / nb);
    }
  return 0;
}
