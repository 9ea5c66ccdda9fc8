// Checks the m8n8k4 f64 fragment layout assumed by form_gemm / err_tiles:
// A[r][k] at lane = 4 r + k, B[k][n] at lane = 4 n + k, C[r][2 t + i] at lane = 4 r + t.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x;
  const double a = A[(lane >> 2) * 4 + (lane & 3)];   // A 8x4 row-major
  const double b = B[(lane & 3) * 8 + (lane >> 2)];   // B 4x8 row-major
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  C[(lane >> 2) * 8 + (lane & 3) * 2] = c0;
  C[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = c1;
}
int main() {
  double A[32], B[32], C[64], R[64];
  for (int i = 0; i < 32; ++i) { A[i] = 1 + i * 0.37; B[i] = 2 - i * 0.11; }
  for (int r = 0; r < 8; ++r) for (int n = 0; n < 8; ++n) { double s = 0; for (int q = 0; q < 4; ++q) s += A[r * 4 + q] * B[q * 8 + n]; R[r * 8 + n] = s; }
  double *dA, *dB, *dC; cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
  cudaMemcpy(dA, A, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, B, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dA, dB, dC); cudaMemcpy(C, dC, 512, cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < 64; ++i) err = fmax(err, fabs(C[i] - R[i]));
  printf("max err %.3e (%s)\n", err, err < 1e-12 ? "layout ok" : "LAYOUT MISMATCH");
  return 0;
}
