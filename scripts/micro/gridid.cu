// Is %gridid unique per launch, including CUDA-graph replays of one node?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* out, int* n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%gridid;" : "=l"(g));
    out[atomicAdd(n, 1)] = g;
  }
}
int main() {
  unsigned long long* out; int* n;
  cudaMalloc(&out, 64 * 8); cudaMalloc(&n, 4); cudaMemset(n, 0, 4);
  cudaStream_t s; cudaStreamCreate(&s);
  k<<<1, 32, 0, s>>>(out, n);
  k<<<1, 32, 0, s>>>(out, n);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  k<<<1, 32, 0, s>>>(out, n);
  k<<<1, 32, 0, s>>>(out, n);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int r = 0; r < 3; ++r) cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  unsigned long long h[64]; int hn;
  cudaMemcpy(&hn, n, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h, out, hn * 8, cudaMemcpyDeviceToHost);
  printf("%d launches, gridids:", hn);
  for (int i = 0; i < hn; ++i) printf(" %llu", h[i]);
  printf("\n%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
