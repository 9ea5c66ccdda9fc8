// Device-resident restarted GMRES, same algorithm
// as the CPU oracle (oracle/solve.py): x0 = 0, modified Gram-Schmidt Arnoldi,
// complex Givens rotations, stop on the Arnoldi residual estimate
// |g_{j+1}| <= tol ||b||, iters = inner steps (= H-matvecs), explicit residual
// b - A x at each restart.
//
// The Krylov basis, w and x live in HBM; the MGS coefficients h_ij are
// produced and consumed on the device (dot -> device scalar -> axpy reads it),
// so the host sees one (j+2)-entry Hessenberg column per iteration for the
// Givens update.  Reductions are two-stage with a fixed grid -> deterministic.
#include <cmath>
#include <complex>
#include <vector>

#include "hmatrix.h"

namespace hmx {

namespace {

constexpr int kThreads = 256;
constexpr int kRedBlocks = 296;  // 2 x 148 SMs, fixed for determinism

__global__ void k_dot_partial(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n,
                              double2* __restrict__ part) {
  __shared__ double2 red[kThreads / 32];
  double2 acc = cmk(0, 0);
  for (int64_t k = blockIdx.x * (int64_t)kThreads + threadIdx.x; k < n; k += (int64_t)gridDim.x * kThreads)
    acc = cfma_ca(a[k], b[k], acc);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = red[0];
    for (int w = 1; w < kThreads / 32; ++w) t = cadd(t, red[w]);
    part[blockIdx.x] = t;
  }
}

// out = sum(part); if norm: out = (sqrt(re), 0)
__global__ void k_dot_final(const double2* __restrict__ part, int np, double2* __restrict__ out, int norm) {
  if (threadIdx.x == 0) {
    double2 t = cmk(0, 0);
    for (int i = 0; i < np; ++i) t = cadd(t, part[i]);
    if (norm) t = cmk(sqrt(fmax(t.x, 0.0)), 0.0);
    *out = t;
  }
}

// y -= (*h) x   (h on device)
__global__ void k_axpy_dev(double2* __restrict__ y, const double2* __restrict__ x, const double2* __restrict__ h,
                           int64_t n) {
  const double2 a = *h;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    y[k] = csub(y[k], cmul(a, x[k]));
}

// y += a x (a host scalar)
__global__ void k_axpy(double2* __restrict__ y, const double2* __restrict__ x, double2 a, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    y[k] = cadd(y[k], cmul(a, x[k]));
}

// y = x * s
__global__ void k_scale(double2* __restrict__ y, const double2* __restrict__ x, double s, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    y[k] = cscale(x[k], s);
}

// y = a - b
__global__ void k_sub(double2* __restrict__ y, const double2* __restrict__ a, const double2* __restrict__ b,
                      int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    y[k] = csub(a[k], b[k]);
}

struct Blas1 {
  Ctx* c;
  int64_t n;
  double2* part;
  int grid;
  int dot(const double2* a, const double2* b, double2* out, int norm) {
    k_dot_partial<<<kRedBlocks, kThreads, 0, c->stream>>>(a, b, n, part);
    k_dot_final<<<1, 32, 0, c->stream>>>(part, kRedBlocks, out, norm);
    return cudaGetLastError() == cudaSuccess ? HMX_OK : HMX_ECUDA;
  }
};

using cplx = std::complex<double>;

}  // namespace

void warm_gmres() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_dot_partial);
  cudaFuncGetAttributes(&a, k_dot_final);
  cudaFuncGetAttributes(&a, k_axpy_dev);
  cudaFuncGetAttributes(&a, k_axpy);
  cudaFuncGetAttributes(&a, k_scale);
  cudaFuncGetAttributes(&a, k_sub);
}

int gmres_device(DeviceH& H, const double2* b, double2* x, double tol, int restart, int64_t max_iters,
                 int64_t* iters_out, std::vector<double>& history, int* converged) {
  Ctx& c = *H.ctx;
  const int64_t n = H.n;
  const int m = restart;
  history.clear();
  *iters_out = 0;
  *converged = 0;
  double2 *Vb = nullptr, *w = nullptr, *tmp = nullptr, *part = nullptr, *hcol = nullptr;
  HMX_CUDA_TRY(dev_alloc_t(c, &Vb, (size_t)n * (m + 1)));
  HMX_CUDA_TRY(dev_alloc_t(c, &w, (size_t)n));
  HMX_CUDA_TRY(dev_alloc_t(c, &tmp, (size_t)n));
  HMX_CUDA_TRY(dev_alloc_t(c, &part, (size_t)kRedBlocks));
  HMX_CUDA_TRY(dev_alloc_t(c, &hcol, (size_t)(m + 2)));
  struct Guard {
    Ctx* c;
    std::vector<void*> p;
    ~Guard() {
      for (void* q : p) dev_free(*c, q);
    }
  } guard{&c, {Vb, w, tmp, part, hcol}};
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(hmx_cdiv(n, kThreads), 4 * c.num_sms));
  Blas1 B{&c, n, part, grid};
  HMX_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double2) * n, c.stream));
  double2 hb;
  if (B.dot(b, b, hcol, 1)) return HMX_ECUDA;
  HMX_CUDA_TRY(cudaMemcpyAsync(&hb, hcol, sizeof(double2), cudaMemcpyDeviceToHost, c.stream));
  HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  const double bnorm = hb.x;
  if (bnorm == 0.0) {
    *converged = 1;
    return HMX_OK;
  }
  int64_t iters = 0;
  double beta = bnorm;
  const double2* r = b;  // first cycle: r = b
  std::vector<cplx> Hm((size_t)(m + 1) * m), g(m + 1), sn(m);
  std::vector<double> cs(m);
  std::vector<double2> hh(m + 2);
  for (;;) {
    k_scale<<<grid, kThreads, 0, c.stream>>>(Vb, r, 1.0 / beta, n);
    std::fill(Hm.begin(), Hm.end(), cplx(0));
    std::fill(g.begin(), g.end(), cplx(0));
    g[0] = beta;
    int k = 0;
    bool done = false;
    for (int j = 0; j < m; ++j) {
      int rc = matvec_device(H, Vb + (int64_t)j * n, w, nullptr);
      if (rc) return rc;
      ++iters;
      for (int i = 0; i <= j; ++i) {
        if (B.dot(Vb + (int64_t)i * n, w, hcol + i, 0)) return HMX_ECUDA;
        k_axpy_dev<<<grid, kThreads, 0, c.stream>>>(w, Vb + (int64_t)i * n, hcol + i, n);
      }
      if (B.dot(w, w, hcol + j + 1, 1)) return HMX_ECUDA;
      HMX_CUDA_TRY(cudaMemcpyAsync(hh.data(), hcol, sizeof(double2) * (j + 2), cudaMemcpyDeviceToHost, c.stream));
      HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
      auto Hij = [&](int i, int jj) -> cplx& { return Hm[(size_t)i * m + jj]; };
      for (int i = 0; i <= j; ++i) Hij(i, j) = cplx(hh[i].x, hh[i].y);
      const double hn = hh[j + 1].x;
      Hij(j + 1, j) = hn;
      for (int i = 0; i < j; ++i) {
        const cplx t0 = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -std::conj(sn[i]) * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t0;
      }
      // Givens (oracle/solve.py givens)
      const cplx a = Hij(j, j), bb = Hij(j + 1, j);
      double cc;
      cplx ss, rr;
      if (bb == cplx(0)) {
        cc = 1.0;
        ss = 0.0;
        rr = a;
      } else if (a == cplx(0)) {
        cc = 0.0;
        ss = std::conj(bb) / std::abs(bb);
        rr = std::abs(bb);
      } else {
        const double t = std::hypot(std::abs(a), std::abs(bb));
        const cplx ph = a / std::abs(a);
        cc = std::abs(a) / t;
        ss = ph * std::conj(bb) / t;
        rr = ph * t;
      }
      cs[j] = cc;
      sn[j] = ss;
      Hij(j, j) = rr;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -std::conj(ss) * g[j];
      g[j] = cc * g[j];
      const double res = std::abs(g[j + 1]);
      history.push_back(res / bnorm);
      k = j + 1;
      if (res <= tol * bnorm) {
        done = true;
        break;
      }
      if (iters >= max_iters || hn == 0.0) break;
      k_scale<<<grid, kThreads, 0, c.stream>>>(Vb + (int64_t)(j + 1) * n, w, 1.0 / hn, n);
    }
    // y = H(0:k,0:k)^-1 g ; x += V y
    std::vector<cplx> y(k);
    for (int i = k - 1; i >= 0; --i) {
      cplx s = g[i];
      for (int l = i + 1; l < k; ++l) s -= Hm[(size_t)i * m + l] * y[l];
      y[i] = s / Hm[(size_t)i * m + i];
    }
    for (int i = 0; i < k; ++i)
      k_axpy<<<grid, kThreads, 0, c.stream>>>(x, Vb + (int64_t)i * n, cmk(y[i].real(), y[i].imag()), n);
    HMX_CUDA_TRY(cudaGetLastError());
    if (done) {
      *converged = 1;
      break;
    }
    if (iters >= max_iters) break;
    int rc = matvec_device(H, x, tmp, nullptr);
    if (rc) return rc;
    k_sub<<<grid, kThreads, 0, c.stream>>>(w, b, tmp, n);
    if (B.dot(w, w, hcol, 1)) return HMX_ECUDA;
    HMX_CUDA_TRY(cudaMemcpyAsync(&hb, hcol, sizeof(double2), cudaMemcpyDeviceToHost, c.stream));
    HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
    beta = hb.x;
    if (beta <= tol * bnorm) {
      *converged = 1;
      break;
    }
    // r = w (copy into tmp so the next cycle's V0 = r / beta does not alias w)
    HMX_CUDA_TRY(cudaMemcpyAsync(tmp, w, sizeof(double2) * n, cudaMemcpyDeviceToDevice, c.stream));
    r = tmp;
  }
  HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  *iters_out = iters;
  return HMX_OK;
}

}  // namespace hmx
