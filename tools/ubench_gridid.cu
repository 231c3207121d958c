// Is %gridid unique per launch, including CUDA-graph replays?  nvcc -arch=sm_100a tools/ubench_gridid.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* out, int i) {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%gridid;" : "=l"(g));
  if (threadIdx.x == 0 && blockIdx.x == 0) out[i] = g;
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int i = 0; i < 3; ++i) k<<<2, 32, 0, s>>>(d, i);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  k<<<2, 32, 0, s>>>(d, 3);
  k<<<2, 32, 0, s>>>(d, 4);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  unsigned long long h[8];
  for (int r = 0; r < 3; ++r) {
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaMemcpy(h, d, 5 * 8, cudaMemcpyDeviceToHost);
    printf("replay %d: direct %llu %llu %llu  graph %llu %llu\n", r, h[0], h[1], h[2], h[3], h[4]);
  }
  return 0;
}
