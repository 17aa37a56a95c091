// Cost of a conditional IF node (condition false) by body size, vs none.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_set(cudaGraphConditionalHandle h, int v) { cudaGraphSetConditional(h, v); }
__global__ void k_small(int* flag) { if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(flag, 1); }
__global__ void k_work(int* flag, int grid) { if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(flag, 1000); }
int main() {
  int* flag; cudaMalloc(&flag, 4);
  cudaStream_t s, side; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int steps = 200;
  for (int body : {-1, 0, 1, 12}) {
    for (int nested : {0, 1}) {
      if (body <= 0 && nested) continue;
      cudaGraph_t g; cudaGraphCreate(&g, 0);
      cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < steps; ++i) {
        if (body >= 0) {
          cudaGraphConditionalHandle h;
          cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault);
          k_set<<<1, 1, 0, s>>>(h, 0);
          cudaStreamCaptureStatus st; const cudaGraphNode_t* deps; size_t nd;
          cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd);
          cudaGraphNodeParams cp = {};
          cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
          cp.conditional.type = cudaGraphCondTypeIf; cp.conditional.size = 1;
          cudaGraphNode_t cn; cudaGraphAddNode(&cn, g, deps, nd, &cp);
          if (nested) {  // the body's kernels inside one child-graph node
            cudaGraph_t child; cudaGraphCreate(&child, 0);
            cudaStreamBeginCaptureToGraph(side, child, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
            for (int k = 0; k < body; ++k) k_small<<<256, 128, 0, side>>>(flag);
            cudaStreamEndCapture(side, &child);
            cudaGraphNode_t cnode; cudaGraphAddChildGraphNode(&cnode, cp.conditional.phGraph_out[0], nullptr, 0, child);
          } else {
            cudaStreamBeginCaptureToGraph(side, cp.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
            for (int k = 0; k < body; ++k) k_small<<<256, 128, 0, side>>>(flag);
            cudaGraph_t bg; cudaStreamEndCapture(side, &bg);
          }
          cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies);
        } else {
          k_small<<<1, 1, 0, s>>>(flag);  // in place of the decide kernel
        }
        k_work<<<1000, 128, 0, s>>>(flag, 1000);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphExec_t ge; cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
      if (e != cudaSuccess) { printf("instantiate body %d nested %d: %s\n", body, nested, cudaGetErrorString(e)); continue; }
      cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
      cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("body %3d nested %d: %.2f us per step\n", body, nested, ms * 1e3 / steps);
    }
  }
  return 0;
}
