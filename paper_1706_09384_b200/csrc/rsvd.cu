// Randomized-SVD fallback of the vector ACA ("the
// randomized SVD ... is preferred"): when every sigma_3 pivot candidate of a leaf falls below the
// floor (aca_kernel status bit 3, e.g. coplanar traction blocks whose 3 x 3 sub-blocks all have
// rank 2), the leaf is regenerated densely on the device and compressed by an adaptive Gaussian
// range finder:
//
//   k = 8, 16, 32, ...:  Omega (n x (k + p)) complex Gaussian (counter-based, seeded per leaf
//                        and per round), Y = A Omega, Q = qr(Y), B = Q^H A,
//                        ||A - Q B||_F^2 = ||A||_F^2 - ||B||_F^2   (Q orthonormal)
//   stop when that residual is <= eps ||A||_F or the column cap is reached (flagged result)
//
// and returns U = Q, V = B^H with their Gram pair, ready for the same recompression as every
// ACA factor pair.  The dense products and the QR are plain library calls (cuBLAS ZGEMM /
// cuSOLVER ZGEQRF + ZUNGQR): this path runs only for the rare leaves ACA cannot compress.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cmath>
#include <vector>

#include "hmatrix.h"

namespace hmx {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Omega[i] = g1 + i g2, g1, g2 ~ N(0, 1) independent (Box-Muller on two 53-bit uniforms)
__global__ void gaussian_fill(double2* __restrict__ om, int64_t count, uint64_t key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = splitmix64(key ^ splitmix64(2 * (uint64_t)i));
    const uint64_t b = splitmix64(key ^ splitmix64(2 * (uint64_t)i + 1));
    const double u1 = ((a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = (b >> 11) * 0x1.0p-53;           // [0, 1)
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
    sincospi(2.0 * u2, &s, &c);
    om[i] = make_double2(r * c, r * s);
  }
}

const char* blas_msg(cublasStatus_t s) {
  switch (s) {
    case CUBLAS_STATUS_NOT_INITIALIZED: return "not initialized";
    case CUBLAS_STATUS_ALLOC_FAILED: return "alloc failed";
    case CUBLAS_STATUS_INVALID_VALUE: return "invalid value";
    case CUBLAS_STATUS_EXECUTION_FAILED: return "execution failed";
    default: return "error";
  }
}

#define RS_BLAS(x)                                                                \
  do {                                                                            \
    const cublasStatus_t s_ = (x);                                                \
    if (s_ != CUBLAS_STATUS_SUCCESS) {                                            \
      hmx_set_error("rsvd: %s failed (cuBLAS %s)", #x, blas_msg(s_));             \
      return HMX_ECUDA;                                                           \
    }                                                                             \
  } while (0)
#define RS_SOLVER(x)                                                              \
  do {                                                                            \
    const cusolverStatus_t s_ = (x);                                              \
    if (s_ != CUSOLVER_STATUS_SUCCESS) {                                          \
      hmx_set_error("rsvd: %s failed (cuSOLVER status %d)", #x, (int)s_);         \
      return HMX_ECUDA;                                                           \
    }                                                                             \
  } while (0)

// scratch owned by one rsvd call (returned to the context cache on exit)
struct Scratch {
  Ctx& c;
  std::vector<void*> p;
  explicit Scratch(Ctx& cc) : c(cc) {}
  ~Scratch() {
    for (void* q : p) dev_free(c, q);
  }
  template <class T>
  int get(T** out, int64_t count) {
    void* q = nullptr;
    if (dev_alloc(c, &q, sizeof(T) * (size_t)(count > 0 ? count : 1)) != cudaSuccess) {
      cudaGetLastError();
      hmx_set_error("rsvd: device allocation of %lld bytes failed", (long long)(sizeof(T) * count));
      return HMX_ENOMEM;
    }
    p.push_back(q);
    *out = static_cast<T*>(q);
    return HMX_OK;
  }
};

}  // namespace

int linalg_handles(Ctx& c, void** blas, void** solver) {
  std::lock_guard<std::mutex> lk(c.mem_mu);
  if (!c.blas) {
    cublasHandle_t h;
    RS_BLAS(cublasCreate(&h));
    c.blas = h;
  }
  if (!c.solver) {
    cusolverDnHandle_t h;
    RS_SOLVER(cusolverDnCreate(&h));
    c.solver = h;
  }
  *blas = c.blas;
  *solver = c.solver;
  return HMX_OK;
}

int launch_gaussian(Ctx& c, double2* out, int64_t count, uint64_t key) {
  if (count <= 0) return HMX_OK;
  gaussian_fill<<<(unsigned)std::min<int64_t>(hmx_cdiv(count, 256), 4 * c.num_sms), 256, 0, c.stream>>>(out, count,
                                                                                                       key);
  HMX_CUDA_TRY(cudaGetLastError());
  return HMX_OK;
}

void linalg_destroy(Ctx& c) {
  if (c.blas) cublasDestroy(static_cast<cublasHandle_t>(c.blas));
  if (c.solver) cusolverDnDestroy(static_cast<cusolverDnHandle_t>(c.solver));
  c.blas = c.solver = nullptr;
}

int rsvd_dense(Ctx& c, const double2* A, int64_t m, int64_t n, double eps, int oversample, int64_t cap, uint64_t seed,
               double2* U, double2* V, double2* G, int* K_out, int* converged) {
  *K_out = 0;
  *converged = 1;
  if (m <= 0 || n <= 0) return HMX_OK;
  cap = std::min<int64_t>(cap, std::min(m, n));
  void *hb, *hs;
  int rc = linalg_handles(c, &hb, &hs);
  if (rc) return rc;
  cublasHandle_t blas = static_cast<cublasHandle_t>(hb);
  cusolverDnHandle_t sol = static_cast<cusolverDnHandle_t>(hs);
  RS_BLAS(cublasSetStream(blas, c.stream));
  RS_SOLVER(cusolverDnSetStream(sol, c.stream));
  RS_BLAS(cublasSetPointerMode(blas, CUBLAS_POINTER_MODE_HOST));
  if (m * n > INT32_MAX) {  // cuBLAS / cuSOLVER 32-bit sizes
    hmx_set_error("rsvd: block of %lld entries too large", (long long)(m * n));
    return HMX_EINVAL;
  }
  double nA = 0.0;
  RS_BLAS(cublasDznrm2(blas, (int)(m * n), reinterpret_cast<const cuDoubleComplex*>(A), 1, &nA));
  if (nA == 0.0) return HMX_OK;  // zero block: rank 0
  Scratch s(c);
  double2 *Om, *B, *tau, *work;
  int* info;
  if ((rc = s.get(&Om, n * cap)) || (rc = s.get(&B, cap * n)) || (rc = s.get(&tau, cap)) || (rc = s.get(&info, 1)))
    return rc;
  int lwork = 0, lw2 = 0;
  RS_SOLVER(cusolverDnZgeqrf_bufferSize(sol, (int)m, (int)cap, reinterpret_cast<cuDoubleComplex*>(U), (int)m, &lwork));
  RS_SOLVER(cusolverDnZungqr_bufferSize(sol, (int)m, (int)cap, (int)cap, reinterpret_cast<cuDoubleComplex*>(U),
                                        (int)m, reinterpret_cast<cuDoubleComplex*>(tau), &lw2));
  lwork = std::max(lwork, lw2);
  if ((rc = s.get(&work, lwork))) return rc;
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  auto cz = [](const double2* p) { return reinterpret_cast<const cuDoubleComplex*>(p); };
  auto z = [](double2* p) { return reinterpret_cast<cuDoubleComplex*>(p); };
  int64_t k = std::min<int64_t>(8, cap);
  for (int round = 0;; ++round) {
    const int64_t kk = std::min<int64_t>(k + oversample, cap);
    const uint64_t key = seed * 0x100000001B3ull + (uint64_t)round * 0x9E3779B97F4A7C15ull + 1;
    gaussian_fill<<<(unsigned)std::min<int64_t>(hmx_cdiv(n * kk, 256), 4 * c.num_sms), 256, 0, c.stream>>>(
        Om, n * kk, key);
    HMX_CUDA_TRY(cudaGetLastError());
    // Y = A Omega into U, then U <- Q of its QR
    RS_BLAS(cublasZgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)m, (int)kk, (int)n, &one, cz(A), (int)m, cz(Om), (int)n,
                        &zero, z(U), (int)m));
    RS_SOLVER(cusolverDnZgeqrf(sol, (int)m, (int)kk, z(U), (int)m, z(tau), z(work), lwork, info));
    RS_SOLVER(cusolverDnZungqr(sol, (int)m, (int)kk, (int)kk, z(U), (int)m, z(tau), z(work), lwork, info));
    // B = Q^H A  (kk x n)
    RS_BLAS(cublasZgemm(blas, CUBLAS_OP_C, CUBLAS_OP_N, (int)kk, (int)n, (int)m, &one, cz(U), (int)m, cz(A), (int)m,
                        &zero, z(B), (int)kk));
    double nB = 0.0;
    RS_BLAS(cublasDznrm2(blas, (int)(kk * n), cz(B), 1, &nB));  // synchronises the stream
    int hinfo = 0;
    HMX_CUDA_TRY(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
    if (hinfo != 0) {
      hmx_set_error("rsvd: QR of the sketch failed (info %d)", hinfo);
      return HMX_ECUDA;
    }
    const double res2 = std::max(0.0, nA * nA - nB * nB);
    const bool ok = std::sqrt(res2) <= eps * nA;
    if (ok || kk >= cap) {
      *converged = ok ? 1 : 0;
      *K_out = (int)kk;
      // V = B^H (n x kk), Gram pair G_U = Q^H Q, G_V = V^H V = B B^H (ld = kk)
      RS_BLAS(cublasZgeam(blas, CUBLAS_OP_C, CUBLAS_OP_N, (int)n, (int)kk, &one, cz(B), (int)kk, &zero, cz(V), (int)n,
                          z(V), (int)n));
      RS_BLAS(cublasZgemm(blas, CUBLAS_OP_C, CUBLAS_OP_N, (int)kk, (int)kk, (int)m, &one, cz(U), (int)m, cz(U), (int)m,
                          &zero, z(G), (int)kk));
      RS_BLAS(cublasZgemm(blas, CUBLAS_OP_N, CUBLAS_OP_C, (int)kk, (int)kk, (int)n, &one, cz(B), (int)kk, cz(B),
                          (int)kk, &zero, z(G + kk * kk), (int)kk));
      HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));  // the scratch returns to the cache
      return HMX_OK;
    }
    k *= 2;
  }
}

}  // namespace hmx
