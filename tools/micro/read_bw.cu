// Read-only HBM streaming ceiling (for the matvec roofline): sum of a large
// array with 16-byte streaming loads, grid = k x SMs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ a, size_t n, double* out) {
  double s = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * st < n; i += 4 * st) {
    double2 x0 = __ldcs(a + i), x1 = __ldcs(a + i + st), x2 = __ldcs(a + i + 2 * st), x3 = __ldcs(a + i + 3 * st);
    s += x0.x + x1.x + x2.x + x3.x + x0.y + x1.y + x2.y + x3.y;
  }
  for (; i < n; i += st) { double2 x = __ldcs(a + i); s += x.x + x.y; }
  if (s == 1.2345) out[0] = s;
}
int main() {
  size_t n = (size_t)10 << 30 >> 4;  // 10 GiB of double2
  double2* a; double* o;
  cudaMalloc(&a, n * 16); cudaMalloc(&o, 8); cudaMemset(a, 0, n * 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int k : {2, 4, 8, 16}) {
    rd<<<sms * k, 256>>>(a, n, o);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) rd<<<sms * k, 256>>>(a, n, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("read-only stream, %2d CTAs/SM: %.0f GB/s\n", k, 5.0 * n * 16 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
