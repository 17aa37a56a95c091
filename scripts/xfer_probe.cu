// Host<->device copy strategies for the engine's upload/download of caller
// arrays (pageable memory), 64 MB: plain pageable cudaMemcpy, with the
// destination freshly allocated (first touch) or warm, cudaHostRegister
// around the copy, and a pinned staging buffer filled/drained by T threads.
// nvcc -O2 -std=c++17 scripts/xfer_probe.cu -o /tmp/xfer_probe && /tmp/xfer_probe
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

static void par_memcpy(void* dst, const void* src, size_t bytes, int threads) {
  std::vector<std::thread> ts;
  const size_t per = (bytes / threads + 4095) & ~size_t(4095);
  for (int t = 0; t < threads; ++t) {
    const size_t b = t * per;
    if (b >= bytes) break;
    const size_t e = std::min(bytes, b + per);
    ts.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + b,
                                      static_cast<const char*>(src) + b, e - b); });
  }
  for (auto& t : ts) t.join();
}

int main() {
  const size_t bytes = 64ull << 20;
  void* d = nullptr;
  cudaMalloc(&d, bytes);
  cudaFree(0);
  std::vector<char> warm(bytes, 1);
  void* pinned = nullptr;
  double t0 = now_ms();
  cudaHostAlloc(&pinned, bytes, cudaHostAllocDefault);
  printf("cudaHostAlloc 64 MB: %.2f ms\n", now_ms() - t0);
  for (int rep = 0; rep < 2; ++rep) {
    t0 = now_ms();
    cudaMemcpy(d, warm.data(), bytes, cudaMemcpyHostToDevice);
    printf("H2D pageable warm: %.2f ms\n", now_ms() - t0);
    t0 = now_ms();
    cudaMemcpy(d, pinned, bytes, cudaMemcpyHostToDevice);
    printf("H2D pinned: %.2f ms\n", now_ms() - t0);
    t0 = now_ms();
    cudaHostRegister(warm.data(), bytes, cudaHostRegisterDefault);
    double t1 = now_ms();
    cudaMemcpy(d, warm.data(), bytes, cudaMemcpyHostToDevice);
    double t2 = now_ms();
    cudaHostUnregister(warm.data());
    printf("H2D register %.2f + copy %.2f + unregister %.2f ms\n", t1 - t0, t2 - t1,
           now_ms() - t2);
    for (int th : {1, 4, 8, 16}) {
      t0 = now_ms();
      par_memcpy(pinned, warm.data(), bytes, th);
      cudaMemcpy(d, pinned, bytes, cudaMemcpyHostToDevice);
      printf("H2D staged %2d threads: %.2f ms\n", th, now_ms() - t0);
    }
    // D2H into fresh (first-touch) memory
    {
      char* fresh = static_cast<char*>(malloc(bytes));
      t0 = now_ms();
      cudaMemcpy(fresh, d, bytes, cudaMemcpyDeviceToHost);
      printf("D2H pageable fresh: %.2f ms\n", now_ms() - t0);
      t0 = now_ms();
      cudaMemcpy(fresh, d, bytes, cudaMemcpyDeviceToHost);
      printf("D2H pageable warm: %.2f ms\n", now_ms() - t0);
      free(fresh);
    }
    {
      char* fresh = static_cast<char*>(malloc(bytes));
      t0 = now_ms();
      cudaHostRegister(fresh, bytes, cudaHostRegisterDefault);
      double t1 = now_ms();
      cudaMemcpy(fresh, d, bytes, cudaMemcpyDeviceToHost);
      double t2 = now_ms();
      cudaHostUnregister(fresh);
      printf("D2H fresh register %.2f + copy %.2f + unregister %.2f ms\n", t1 - t0, t2 - t1,
             now_ms() - t2);
      free(fresh);
    }
    for (int th : {1, 4, 8, 16}) {
      char* fresh = static_cast<char*>(malloc(bytes));
      t0 = now_ms();
      cudaMemcpy(pinned, d, bytes, cudaMemcpyDeviceToHost);
      double t1 = now_ms();
      par_memcpy(fresh, pinned, bytes, th);
      printf("D2H fresh staged %2d threads: dma %.2f + memcpy %.2f ms\n", th, t1 - t0,
             now_ms() - t1);
      free(fresh);
    }
  }
  printf("hardware threads: %u\n", std::thread::hardware_concurrency());
  return 0;
}
