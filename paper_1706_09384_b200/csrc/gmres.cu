// Device-resident restarted GMRES, same algorithm
// as the CPU oracle (oracle/solve.py): x0 = 0, modified Gram-Schmidt Arnoldi,
// complex Givens rotations G = [[c, s], [-conj(s), c]] (c real), stop on the
// Arnoldi residual estimate |g_{j+1}| <= tol ||b||, iters = inner steps
// (= H-matvecs), explicit residual b - A x at each restart.
//
// Everything the iteration decides lives on the device (SURVEY 2 kernel 5:
// the host never round-trips per iteration):
//   * the Krylov basis, w, x in HBM;
//   * one cooperative kernel per Arnoldi step runs the whole MGS sweep
//     (dot -> grid barrier -> axpy per basis vector, then the norm), stores the
//     Hessenberg column, applies the previous rotations, forms the new Givens
//     rotation, updates g, appends |g_{j+1}|/||b|| to the history and decides
//     whether the cycle continues -- all in device memory (GmState);
//   * the end of a cycle (back substitution, x += V y, the explicit residual and
//     the restart) is a short chain of device kernels gated by the same state.
// The host only enqueues: it keeps at most kAhead Arnoldi steps queued beyond
// the device's progress (a counter the device writes to mapped host memory),
// so the GPU always has the next step queued and never waits for the host.
// Steps queued past convergence are skipped on the device: every launch
// (including the matvec's four kernels) is gated by a device flag.
//
// Reductions use a fixed grid of kGrid CTAs; every CTA sums the per-CTA
// partials in the same fixed order, so results are deterministic run to run.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "hmatrix.h"

namespace cg = cooperative_groups;

namespace hmx {

namespace {

constexpr int kThreads = 256;
constexpr int kGrid = 296;   // 2 CTAs x 148 SMs: co-resident for the cooperative launch, fixed for determinism
constexpr int kAhead = 2;    // Arnoldi steps the host keeps queued beyond the device's progress

struct GmState {
  double tol, bnorm, beta;
  int64_t max_iters;
  int64_t iters;   // inner steps so far
  int64_t nhist;
  int m;           // restart length
  int j;           // next inner step of the current cycle
  int k;           // completed inner steps of the current cycle
  int inner;       // 1 while the current cycle's Arnoldi loop runs (matvec / step gate)
  int open;        // 1 from a cycle's start until its x update is done
  int restart;     // 1 while the explicit residual of a restart is computed
  int scale0;      // 1 when V_0 = r / beta is due
  int finished;    // 1 once GMRES is done
  int converged;
  int cycles;      // completed cycles (x updates)
};

// progress word the host polls (mapped pinned memory): steps done, cycles closed, finished
struct GmProgress {
  volatile int64_t iters;
  volatile int cycles;
  volatile int inner;
  volatile int finished;
};

HMX_D void publish(const GmState* s, GmProgress* p) {
  p->iters = s->iters;
  p->cycles = s->cycles;
  p->inner = s->inner;
  p->finished = s->finished;
  __threadfence_system();
}

// ---- grid-wide deterministic reductions ----------------------------------------------------
// block partial of sum conj(a) b over this thread's grid-stride elements
HMX_D double2 block_dot(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n, double2* red) {
  double2 acc = cmk(0, 0);
  for (int64_t q = blockIdx.x * (int64_t)kThreads + threadIdx.x; q < n; q += (int64_t)gridDim.x * kThreads)
    acc = cfma_ca(a[q], b[q], acc);
  acc = warp_sum(acc);
  __syncthreads();  // red reused across calls
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double2 t = red[0];
  for (int w = 1; w < kThreads / 32; ++w) t = cadd(t, red[w]);
  return t;
}

// every CTA: sum of the kGrid partials in index order (same value everywhere)
HMX_D double2 grid_total(const double2* part) {
  __shared__ double2 tot;
  if (threadIdx.x < 32) {
    double2 t = cmk(0, 0);
    // fixed association: lane l sums partials l, l + 32, ...; then a fixed-order fold
    for (int i = threadIdx.x; i < kGrid; i += 32) t = cadd(t, part[i]);
    t = warp_sum(t);
    if (threadIdx.x == 0) tot = t;
  }
  __syncthreads();
  return tot;
}

__global__ void k_init(GmState* s, const double2* part, double2* g, GmProgress* prog) {
  if (threadIdx.x != 0) return;
  double2 t = cmk(0, 0);
  for (int i = 0; i < kGrid; ++i) t = cadd(t, part[i]);
  const double bn = sqrt(fmax(t.x, 0.0));
  s->bnorm = bn;
  s->beta = bn;
  s->iters = 0;
  s->nhist = 0;
  s->j = 0;
  s->k = 0;
  s->cycles = 0;
  s->restart = 0;
  if (bn == 0.0) {  // b = 0 -> x = 0, 0 iterations
    s->inner = 0;
    s->open = 0;
    s->scale0 = 0;
    s->finished = 1;
    s->converged = 1;
  } else {
    s->inner = 1;
    s->open = 1;
    s->scale0 = 1;
    s->finished = 0;
    s->converged = 0;
    for (int i = 0; i <= s->m; ++i) g[i] = cmk(0, 0);
    g[0] = cmk(bn, 0);
  }
  publish(s, prog);
}

// per-CTA partial of ||v||^2 into part (used for ||b|| and the restart residual), gated
__global__ void __launch_bounds__(kThreads) k_norm_part(const double2* __restrict__ v, int64_t n,
                                                        double2* __restrict__ part, const int* gate) {
  if (gate && *gate == 0) return;
  __shared__ double2 red[kThreads / 32];
  const double2 t = block_dot(v, v, n, red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// g := 0, g[0] = beta; start the next cycle (or finish when the residual is small)
__global__ void k_restart(GmState* s, const double2* part, double2* g, GmProgress* prog) {
  if (threadIdx.x != 0 || !s->restart) return;
  double2 t = cmk(0, 0);
  for (int i = 0; i < kGrid; ++i) t = cadd(t, part[i]);
  const double beta = sqrt(fmax(t.x, 0.0));
  s->restart = 0;
  s->beta = beta;
  if (beta <= s->tol * s->bnorm) {
    s->finished = 1;
    s->converged = 1;
  } else {
    for (int i = 0; i <= s->m; ++i) g[i] = cmk(0, 0);
    g[0] = cmk(beta, 0);
    s->j = 0;
    s->k = 0;
    s->inner = 1;
    s->open = 1;
    s->scale0 = 1;
  }
  publish(s, prog);
}

// V_0 = r / beta (gated by scale0)
__global__ void k_scale0(const GmState* s, double2* __restrict__ V0, const double2* __restrict__ r, int64_t n) {
  if (!s->scale0) return;
  const double inv = 1.0 / s->beta;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    V0[q] = cscale(r[q], inv);
}

__global__ void k_scale0_done(GmState* s) {
  if (threadIdx.x == 0) s->scale0 = 0;
}

// One Arnoldi step j = s->j (cooperative launch, kGrid x kThreads): MGS of w against V_0..V_j,
// h_{j+1,j} = ||w||, V_{j+1} = w / h_{j+1,j}; then (CTA 0, thread 0) the Givens update of
// oracle/solve.py and the stop decision.
__global__ void __launch_bounds__(kThreads) k_arnoldi(GmState* s, double2* __restrict__ Vb, double2* __restrict__ w,
                                                      int64_t n, double2* __restrict__ part, double2* __restrict__ Hm,
                                                      double* __restrict__ cs, double2* __restrict__ sn,
                                                      double2* __restrict__ g, double* __restrict__ hist,
                                                      int64_t hist_cap, GmProgress* prog) {
  if (!s->inner) return;  // uniform over the grid: written by an earlier launch
  cg::grid_group grid = cg::this_grid();
  __shared__ double2 red[kThreads / 32];
  const int j = s->j;
  const int m = s->m;
  for (int i = 0; i <= j; ++i) {
    const double2* vi = Vb + (int64_t)i * n;
    const double2 pb = block_dot(vi, w, n, red);
    double2* pbuf = part + (i & 1) * kGrid;  // double-buffered: no second barrier per vector
    if (threadIdx.x == 0) pbuf[blockIdx.x] = pb;
    grid.sync();
    const double2 h = grid_total(pbuf);
    // every thread updates exactly the elements its next dot reads: no barrier for w
    for (int64_t q = blockIdx.x * (int64_t)kThreads + threadIdx.x; q < n; q += (int64_t)gridDim.x * kThreads)
      w[q] = csub(w[q], cmul(h, vi[q]));
    if (blockIdx.x == 0 && threadIdx.x == 0) Hm[(int64_t)i * m + j] = h;
  }
  {
    const double2 pb = block_dot(w, w, n, red);
    double2* pbuf = part + ((j + 1) & 1) * kGrid;
    if (threadIdx.x == 0) pbuf[blockIdx.x] = pb;
    grid.sync();
    const double hn = sqrt(fmax(grid_total(pbuf).x, 0.0));
    if (hn != 0.0 && j + 1 <= m) {
      const double inv = 1.0 / hn;
      double2* vn = Vb + (int64_t)(j + 1) * n;
      for (int64_t q = blockIdx.x * (int64_t)kThreads + threadIdx.x; q < n; q += (int64_t)gridDim.x * kThreads)
        vn[q] = cscale(w[q], inv);
    }
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    auto H = [&](int r, int c) -> double2& { return Hm[(int64_t)r * m + c]; };
    H(j + 1, j) = cmk(hn, 0);
    for (int i = 0; i < j; ++i) {
      const double2 a = H(i, j), b = H(i + 1, j);
      const double2 t0 = cadd(cscale(a, cs[i]), cmul(sn[i], b));
      H(i + 1, j) = cadd(cscale(cmul(cconj(sn[i]), a), -1.0), cscale(b, cs[i]));
      H(i, j) = t0;
    }
    const double2 a = H(j, j), b = H(j + 1, j);
    double c;
    double2 sv, rr;
    if (b.x == 0.0 && b.y == 0.0) {
      c = 1.0;
      sv = cmk(0, 0);
      rr = a;
    } else if (a.x == 0.0 && a.y == 0.0) {
      const double ab = hypot(b.x, b.y);
      c = 0.0;
      sv = cscale(cconj(b), 1.0 / ab);
      rr = cmk(ab, 0);
    } else {
      const double aa = hypot(a.x, a.y), ab = hypot(b.x, b.y);
      const double t = hypot(aa, ab);
      const double2 ph = cscale(a, 1.0 / aa);
      c = aa / t;
      sv = cscale(cmul(ph, cconj(b)), 1.0 / t);
      rr = cscale(ph, t);
    }
    cs[j] = c;
    sn[j] = sv;
    H(j, j) = rr;
    H(j + 1, j) = cmk(0, 0);
    const double2 gj = g[j];
    g[j + 1] = cscale(cmul(cconj(sv), gj), -1.0);
    g[j] = cscale(gj, c);
    const double res = hypot(g[j + 1].x, g[j + 1].y);
    if (s->nhist < hist_cap) hist[s->nhist] = res / s->bnorm;
    s->nhist++;
    s->iters++;
    s->k = j + 1;
    s->j = j + 1;
    if (res <= s->tol * s->bnorm) {
      s->converged = 1;
      s->inner = 0;
    } else if (s->iters >= s->max_iters || hn == 0.0 || j + 1 >= m) {
      s->inner = 0;
    }
    publish(s, prog);
  }
}

// end of a cycle: y = H(0:k, 0:k)^{-1} g(0:k) by back substitution (one thread)
__global__ void k_backsolve(GmState* s, const double2* __restrict__ Hm, const double2* __restrict__ g,
                            double2* __restrict__ y) {
  if (threadIdx.x != 0 || !s->open || s->inner) return;
  const int k = s->k, m = s->m;
  for (int i = k - 1; i >= 0; --i) {
    double2 t = g[i];
    for (int l = i + 1; l < k; ++l) t = csub(t, cmul(Hm[(int64_t)i * m + l], y[l]));
    y[i] = cdiv(t, Hm[(int64_t)i * m + i]);
  }
}

// x += V(:, 0:k) y
__global__ void k_xupdate(const GmState* s, double2* __restrict__ x, const double2* __restrict__ Vb,
                          const double2* __restrict__ y, int64_t n) {
  if (!s->open || s->inner) return;
  const int k = s->k;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    double2 t = x[q];
    for (int i = 0; i < k; ++i) t = cadd(t, cmul(y[i], Vb[(int64_t)i * n + q]));
    x[q] = t;
  }
}

// close the cycle: finished (converged / out of iterations) or a restart is due
__global__ void k_close(GmState* s, GmProgress* prog) {
  if (threadIdx.x != 0 || !s->open || s->inner) return;
  s->open = 0;
  s->cycles++;
  if (s->converged || s->iters >= s->max_iters) {
    s->finished = 1;
  } else {
    s->restart = 1;
  }
  publish(s, prog);
}

// r = b - A x (A x already in ax), gated by the restart flag
__global__ void k_residual(const GmState* s, double2* __restrict__ r, const double2* __restrict__ b,
                           const double2* __restrict__ ax, int64_t n) {
  if (!s->restart) return;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    r[q] = csub(b[q], ax[q]);
}

}  // namespace

void warm_gmres() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_init);
  cudaFuncGetAttributes(&a, k_norm_part);
  cudaFuncGetAttributes(&a, k_restart);
  cudaFuncGetAttributes(&a, k_scale0);
  cudaFuncGetAttributes(&a, k_scale0_done);
  cudaFuncGetAttributes(&a, k_arnoldi);
  cudaFuncGetAttributes(&a, k_backsolve);
  cudaFuncGetAttributes(&a, k_xupdate);
  cudaFuncGetAttributes(&a, k_close);
  cudaFuncGetAttributes(&a, k_residual);
}

int gmres_device(DeviceH& H, const double2* b, double2* x, double tol, int restart, int64_t max_iters,
                 int64_t* iters_out, std::vector<double>& history, int* converged, cudaStream_t st) {
  Ctx& c = *H.ctx;
  const int64_t n = H.n;
  const int m = restart;
  history.clear();
  *iters_out = 0;
  *converged = 0;
  {
    int occ = 0;
    HMX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_arnoldi, kThreads, 0));
    if ((int64_t)occ * c.num_sms < kGrid) {
      hmx_set_error("GMRES step kernel: %d co-resident CTAs < %d", occ * c.num_sms, kGrid);
      return HMX_ECUDA;
    }
  }
  const int64_t hist_cap = std::max<int64_t>(1, max_iters);
  double2 *Vb = nullptr, *w = nullptr, *tmp = nullptr, *part = nullptr, *Hm = nullptr, *sn = nullptr, *g = nullptr,
          *y = nullptr;
  double *cs = nullptr, *hist = nullptr;
  GmState* s = nullptr;
  HMX_CUDA_TRY(dev_alloc_t(c, &Vb, (size_t)n * (m + 1)));
  HMX_CUDA_TRY(dev_alloc_t(c, &w, (size_t)n));
  HMX_CUDA_TRY(dev_alloc_t(c, &tmp, (size_t)n));
  HMX_CUDA_TRY(dev_alloc_t(c, &part, (size_t)2 * kGrid));
  HMX_CUDA_TRY(dev_alloc_t(c, &Hm, (size_t)(m + 1) * m));
  HMX_CUDA_TRY(dev_alloc_t(c, &sn, (size_t)m));
  HMX_CUDA_TRY(dev_alloc_t(c, &g, (size_t)(m + 1)));
  HMX_CUDA_TRY(dev_alloc_t(c, &y, (size_t)m));
  HMX_CUDA_TRY(dev_alloc_t(c, &cs, (size_t)m));
  HMX_CUDA_TRY(dev_alloc_t(c, &hist, (size_t)hist_cap));
  HMX_CUDA_TRY(dev_alloc_t(c, &s, 1));
  GmProgress* prog = nullptr;
  HMX_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&prog), sizeof(GmProgress), cudaHostAllocMapped));
  GmProgress* dprog = nullptr;
  struct Guard {
    Ctx* c;
    std::vector<void*> p;
    GmProgress* hp;
    ~Guard() {
      for (void* q : p) dev_free(*c, q);
      if (hp) cudaFreeHost(hp);
    }
  } guard{&c, {Vb, w, tmp, part, Hm, sn, g, y, cs, hist, s}, prog};
  HMX_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dprog), prog, 0));
  prog->iters = 0;
  prog->cycles = 0;
  prog->inner = 1;  // until k_init publishes
  prog->finished = 0;
  {
    GmState h{};
    h.tol = tol;
    h.max_iters = max_iters;
    h.m = m;
    HMX_CUDA_TRY(cudaMemcpyAsync(s, &h, sizeof(GmState), cudaMemcpyHostToDevice, st));
  }
  HMX_CUDA_TRY(cudaMemsetAsync(Hm, 0, sizeof(double2) * (m + 1) * m, st));
  HMX_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double2) * n, st));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(hmx_cdiv(n, kThreads), 4 * c.num_sms));
  k_norm_part<<<kGrid, kThreads, 0, st>>>(b, n, part, nullptr);
  k_init<<<1, 32, 0, st>>>(s, part, g, dprog);
  k_scale0<<<grid, kThreads, 0, st>>>(s, Vb, b, n);
  k_scale0_done<<<1, 32, 0, st>>>(s);
  HMX_CUDA_TRY(cudaGetLastError());
  // the inner-loop gate (s->inner) and the restart gate (s->restart) for the matvec launches
  const int* gate_inner = &s->inner;
  const int* gate_restart = &s->restart;
  int64_t nn = n, hc = hist_cap;
  int64_t queued = 0;  // Arnoldi steps enqueued so far
  int rc = HMX_OK;
  for (;;) {
    for (int j = 0; j < m; ++j) {
      // keep at most kAhead steps queued beyond what the device has finished (poll the mapped
      // progress word, no stream synchronisation); stop queueing once the device has left this
      // cycle's Arnoldi loop (converged / breakdown / iteration cap)
      while (!(prog->finished || !prog->inner || prog->iters >= queued - kAhead)) std::this_thread::yield();
      if (prog->finished || !prog->inner || queued >= max_iters) break;
      if ((rc = matvec_device(H, Vb + (int64_t)j * n, w, nullptr, st, gate_inner))) return rc;
      void* args[] = {&s, &Vb, &w, &nn, &part, &Hm, &cs, &sn, &g, &hist, &hc, &dprog};
      HMX_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_arnoldi, dim3(kGrid), dim3(kThreads), args, 0, st));
      ++queued;
    }
    // end of the cycle + the restart residual (all gated on the device)
    k_backsolve<<<1, 32, 0, st>>>(s, Hm, g, y);
    k_xupdate<<<grid, kThreads, 0, st>>>(s, x, Vb, y, n);
    k_close<<<1, 32, 0, st>>>(s, dprog);
    if ((rc = matvec_device(H, x, tmp, nullptr, st, gate_restart))) return rc;
    k_residual<<<grid, kThreads, 0, st>>>(s, w, b, tmp, n);
    k_norm_part<<<kGrid, kThreads, 0, st>>>(w, n, part, gate_restart);
    k_restart<<<1, 32, 0, st>>>(s, part, g, dprog);
    k_scale0<<<grid, kThreads, 0, st>>>(s, Vb, w, n);
    k_scale0_done<<<1, 32, 0, st>>>(s);
    HMX_CUDA_TRY(cudaGetLastError());
    // one host wait per cycle (every `restart` inner steps), never per iteration
    HMX_CUDA_TRY(cudaStreamSynchronize(st));
    if (prog->finished) break;
    queued = prog->iters;
  }
  HMX_CUDA_TRY(cudaStreamSynchronize(st));
  GmState h{};
  HMX_CUDA_TRY(cudaMemcpy(&h, s, sizeof(GmState), cudaMemcpyDeviceToHost));
  const int64_t nh = std::min<int64_t>(h.nhist, hist_cap);
  history.resize((size_t)nh);
  if (nh) HMX_CUDA_TRY(cudaMemcpy(history.data(), hist, sizeof(double) * nh, cudaMemcpyDeviceToHost));
  *iters_out = h.iters;
  *converged = h.converged;
  return HMX_OK;
}

}  // namespace hmx
