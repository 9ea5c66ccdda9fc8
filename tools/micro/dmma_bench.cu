// FP64 tensor-core (mma.sync m8n8k4 f64) throughput probe vs DFMA.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = fma(a, b, c[k]);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {128, 256, 512}) {
    const int iters = 20000;
    dmma_loop<<<sms * 4, threads>>>(d, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms * 4, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 4 * (double)iters * (sms * 4) * (threads / 32);
    printf("DMMA m8n8k4  %d thr x %d CTAs: %.1f TFLOP/s\n", threads, sms * 4, flops / ms / 1e9);
    dfma_loop<<<sms * 4, threads>>>(d, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms * 4, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * (double)iters * (sms * 4) * threads;
    printf("DFMA         %d thr x %d CTAs: %.1f TFLOP/s\n", threads, sms * 4, flops / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
