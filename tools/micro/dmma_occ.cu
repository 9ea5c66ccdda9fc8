// DMMA (mma.sync m8n8k4 f64) throughput vs warps per SM and independent
// accumulator chains, plus the dependent-chain latency.  nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -o dmma_occ dmma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int NCH>
__global__ void loop(double* out, int iters, long long* cyc) {
  double c[NCH][2];
  for (int k = 0; k < NCH; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < NCH; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int NCH>
void run(int sms, int warps, int iters) {
  double* d; long long* cyc;
  cudaMalloc(&d, 8); cudaMalloc(&cyc, 8);
  loop<NCH><<<sms, 32 * warps>>>(d, 10, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  loop<NCH><<<sms, 32 * warps>>>(d, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long hc; cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  const double fl = 512.0 * NCH * (double)iters * warps * sms;
  printf("warps/SM %2d chains %2d: %6.2f TF/s, %6.1f cycles per DMMA per warp (chain step %5.1f cyc)\n", warps, NCH,
         fl / ms / 1e9, (double)hc / iters / NCH, (double)hc / iters);
  cudaFree(d); cudaFree(cyc);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {1, 4, 8, 16, 32}) {
    run<1>(sms, w, 20000);
    run<4>(sms, w, 5000);
    run<12>(sms, w, 2000);
  }
  return 0;
}
