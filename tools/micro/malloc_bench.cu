// cudaMalloc cost probe: sequential vs threaded large allocations, cudaMallocAsync, VMM map.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  cudaFree(0);
  const size_t GB = 1ull << 30;
  for (size_t sz : {10 * GB, 40 * GB}) {
    void* p[3];
    double t0 = now();
    for (int i = 0; i < 3; ++i) cudaMalloc(&p[i], sz);
    double t1 = now();
    printf("3 x cudaMalloc(%zu GB) sequential: %.1f ms (%.2f ms/GB)\n", sz / GB, t1 - t0, (t1 - t0) / (3.0 * sz / GB));
    t0 = now();
    for (int i = 0; i < 3; ++i) cudaFree(p[i]);
    printf("  3 x cudaFree: %.1f ms\n", now() - t0);
    t0 = now();
    std::vector<std::thread> th;
    for (int i = 0; i < 3; ++i) th.emplace_back([&, i] { cudaMalloc(&p[i], sz); });
    for (auto& t : th) t.join();
    t1 = now();
    printf("3 x cudaMalloc(%zu GB) in 3 threads: %.1f ms\n", sz / GB, t1 - t0);
    for (int i = 0; i < 3; ++i) cudaFree(p[i]);
    cudaStream_t s;
    cudaStreamCreate(&s);
    t0 = now();
    for (int i = 0; i < 3; ++i) cudaMallocAsync(&p[i], sz, s);
    cudaStreamSynchronize(s);
    t1 = now();
    printf("3 x cudaMallocAsync(%zu GB): %.1f ms\n", sz / GB, t1 - t0);
    for (int i = 0; i < 3; ++i) cudaFreeAsync(p[i], s);
    cudaStreamSynchronize(s);
    cudaMemPool_t mp;
    cudaDeviceGetDefaultMemPool(&mp, 0);
    cudaMemPoolTrimTo(mp, 0);
  }
  return 0;
}
