// Cost of a chain of 11 tail launches from a kernel node (vs the same 11
// kernels as graph nodes), per step.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_small(int* flag, int v) {
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(flag, v);
}
__global__ void k_parent(int* flag, int go, int grid) {
  if (go) {
    for (int k = 0; k < 11; ++k) k_small<<<grid, 128, 0, cudaStreamTailLaunch>>>(flag, 1);
  }
}
__global__ void k_work(int* flag) {
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(flag, 1000);
}
int main() {
  int* flag;
  cudaMalloc(&flag, 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {1, 256, 8192}) {
    for (int variant = 0; variant < 3; ++variant) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < 200; ++i) {
        if (variant == 0) {  // 11 nodes + work
          for (int k = 0; k < 11; ++k) k_small<<<grid, 128, 0, s>>>(flag, 1);
        } else {
          k_parent<<<1, 1, 0, s>>>(flag, variant == 2, grid);
        }
        k_work<<<grid, 128, 0, s>>>(flag);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaMemset(flag, 0, 4);
      cudaGraphLaunch(ge, s);
      cudaStreamSynchronize(s);
      int h = 0;
      cudaMemcpy(&h, flag, 4, cudaMemcpyDeviceToHost);
      cudaEventRecord(a, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const char* nm[] = {"11 graph nodes", "parent, no launch", "parent + 11 tail launches"};
      printf("grid %5d %-26s: %.2f us per step (flag %d)\n", grid, nm[variant], ms * 1e3 / 200, h);
    }
  }
  return 0;
}
