// Cross-process CUDA IPC on one GPU: ./ipc_probe export FILE | ./ipc_probe import FILE
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <unistd.h>
int main(int argc, char** argv) {
  if (argc < 3) return 2;
  cudaSetDevice(0);
  if (!strcmp(argv[1], "export")) {
    void* p = nullptr;
    size_t bytes = argc > 3 ? atol(argv[3]) : (64 << 20);
    cudaMalloc(&p, bytes);
    cudaMemset(p, 7, bytes);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, p);
    printf("export get=%s ptr=%p\n", cudaGetErrorString(e), p);
    FILE* f = fopen(argv[2], "wb"); fwrite(&h, sizeof h, 1, f); fclose(f);
    sleep(6);
    unsigned char b = 0; cudaMemcpy(&b, p, 1, cudaMemcpyDeviceToHost);
    printf("export sees byte %d after import wrote\n", b);
    return 0;
  }
  sleep(2);
  cudaIpcMemHandle_t h;
  FILE* f = fopen(argv[2], "rb"); fread(&h, sizeof h, 1, f); fclose(f);
  for (int flag = 0; flag < 2; ++flag) {
    void* q = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&q, h, flag ? cudaIpcMemLazyEnablePeerAccess : 0);
    printf("import flag=%d open=%s ptr=%p\n", flag, cudaGetErrorString(e), q);
    if (e == cudaSuccess) { cudaMemset(q, 42, 1); cudaDeviceSynchronize(); cudaIpcCloseMemHandle(q); }
    cudaGetLastError();
  }
  return 0;
}
