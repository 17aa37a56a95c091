// Does a tail launch from a kernel node complete before the next graph node?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_child(int* flag, int v) {
  long long t0 = clock64();
  while (clock64() - t0 < 200000) {}  // ~100 us
  *flag = v;
}
__global__ void k_child2(int* flag, int v) { *flag = *flag * 10 + v; }
__global__ void k_parent(int* flag, int go, int v) {
  if (go) {
    k_child<<<1, 1, 0, cudaStreamTailLaunch>>>(flag, v);
    k_child2<<<1, 1, 0, cudaStreamTailLaunch>>>(flag, 7);
  }
}
__global__ void k_check(int* flag, int* seen, int idx) { seen[idx] = *flag; }
int main() {
  int *flag, *seen;
  cudaMalloc(&flag, 4); cudaMalloc(&seen, 64 * 4);
  cudaMemset(flag, 0, 4); cudaMemset(seen, 0, 256);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 8; ++i) {
    k_parent<<<1, 1, 0, s>>>(flag, i % 2, i + 1);
    k_check<<<1, 1, 0, s>>>(flag, seen, i);
  }
  cudaError_t e = cudaStreamEndCapture(s, &g);
  printf("capture: %s\n", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&ge, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  e = cudaGraphLaunch(ge, s);
  printf("launch: %s\n", cudaGetErrorString(e));
  e = cudaStreamSynchronize(s);
  printf("sync: %s\n", cudaGetErrorString(e));
  int h[8]; cudaMemcpy(h, seen, 32, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 8; ++i) printf("step %d go=%d seen=%d\n", i, i % 2, h[i]);
  // timing: graph of 1000 (parent go=0 -> check) pairs vs 1000 checks
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int variant = 0; variant < 2; ++variant) {
    cudaGraph_t g2; cudaGraphExec_t ge2;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 1000; ++i) {
      if (variant) k_parent<<<1, 1, 0, s>>>(flag, 0, 0);
      k_check<<<1, 1, 0, s>>>(flag, seen, 0);
    }
    cudaStreamEndCapture(s, &g2);
    cudaGraphInstantiate(&ge2, g2, 0);
    cudaGraphLaunch(ge2, s); cudaStreamSynchronize(s);
    cudaEventRecord(a, s); cudaGraphLaunch(ge2, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("variant %d: %.3f us per step\n", variant, ms);
  }
  return 0;
}
