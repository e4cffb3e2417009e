// Event-timed latency of an empty kernel: plain vs cooperative launch, and in a CUDA graph.
#include <cstdio>
__global__ void k(int *p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int *d; cudaMalloc(&d, 4);
  for (int coop = 0; coop < 2; ++coop) {
    for (int graph = 0; graph < 2; ++graph) {
      cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(296); cfg.blockDim = dim3(256); cfg.stream = s;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
      cfg.attrs = at; cfg.numAttrs = coop;
      cudaGraphExec_t ge = nullptr;
      if (graph) {
        cudaGraph_t gr; cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        cudaLaunchKernelEx(&cfg, k, d);
        cudaStreamEndCapture(s, &gr); cudaGraphInstantiate(&ge, gr, 0);
      }
      float best = 1e9, sum = 0; int n = 200;
      for (int i = 0; i < n + 10; ++i) {
        cudaEventRecord(a, s);
        if (graph) cudaGraphLaunch(ge, s); else cudaLaunchKernelEx(&cfg, k, d);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (i >= 10) { sum += ms; if (ms < best) best = ms; }
      }
      printf("coop %d graph %d: mean %.2f us, min %.2f us\n", coop, graph, sum / n * 1000, best * 1000);
    }
  }
  return 0;
}
