// H-matrix-vector product y = A_H x.
//
// One pass over the packed HBM streams (layout in hmatrix.h):
//   gather    x_tree[d k + a] = x[d perm[k] + a]                      (tree order)
//   phase 1   warp per job: s[slot..+4] = V_b(:, l..l+4)^H x_tree(cols of b)   (low-rank)
//             or s[slot..] = x_tree(cols of b)                        (dense)
//   phase 2   CTA per (row segment, 256-row tile): y_lev[level][rows] =
//             M_g(rows, :) s_g -- column-major M_g, lanes over rows so each
//             load instruction is a contiguous 512 B, columns split over up to
//             8 thread groups for short segments, reduced in shared memory
//   finalize  y[d perm[k] + a] = sum_level y_lev[level][d k + a]   (fixed order)
// Every (level, row) is written by exactly one phase-2 tile, so y is
// bit-reproducible run to run (no floating-point atomics).
// The pass is HBM-bound (complex128 GEMV = 0.5 flop/B); bytes per call are
// H.mv_bytes = 16 (sum dense d^2 m n + sum r d (m + n)) + 32 d N.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <numeric>

#include "hmatrix.h"

namespace hmx {

namespace {

constexpr int kThreads = 256;

// gate (optional): the launch does nothing when *gate == 0 (device-resident GMRES enqueues
// matvecs ahead of its convergence test; the ones past convergence are skipped on the device)
__global__ void mv_gather(const double2* __restrict__ x, const int64_t* __restrict__ perm, int d, int64_t np,
                          double2* __restrict__ xt, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < np * d; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = k / d, a = k - p * d;
    xt[k] = x[d * perm[p] + a];
  }
}

// Phase-1 job: kind 0 copies x pieces of a dense leaf into its slots; kind
// k = 1..4 computes k consecutive columns t_c = V(:, l + c)^H x of a low-rank
// leaf (x loaded once for the k columns, 2 k + 2 loads in flight per lane), then
// one butterfly reduce-scatter of the 2 x 4 partial sums over the warp.
constexpr int kColsPerJob = 4;  // 8 measured 13% slower (fewer, longer jobs)
__global__ void __launch_bounds__(kThreads) mv_phase1(const MvJob1* __restrict__ jobs, int64_t njobs,
                                                         const double2* __restrict__ V,
                                                         const double2* __restrict__ xt, double2* __restrict__ s,
                                                         const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = wid; j < njobs; j += nw) {
    const MvJob1 J = jobs[j];
    const double2* xp = xt + J.xoff;
    if (J.kind == 0) {
      for (int q = lane; q < J.len; q += 32) s[J.soff + q] = xp[q];
      continue;
    }
    const double2* vp = V + J.voff;
    const int64_t len = J.len;
    const int nc = J.kind;
    double2 acc[kColsPerJob];
#pragma unroll
    for (int c = 0; c < kColsPerJob; ++c) acc[c] = cmk(0, 0);
    int q = lane;
    if (nc == kColsPerJob) {
      for (; q + 32 < J.len; q += 64) {
        const double2 x0 = xp[q], x1 = xp[q + 32];
        double2 v0[kColsPerJob], v1[kColsPerJob];
#pragma unroll
        for (int c = 0; c < kColsPerJob; ++c) {
          v0[c] = __ldcs(vp + c * len + q);
          v1[c] = __ldcs(vp + c * len + q + 32);
        }
#pragma unroll
        for (int c = 0; c < kColsPerJob; ++c) acc[c] = cfma_ca(v1[c], x1, cfma_ca(v0[c], x0, acc[c]));
      }
      for (; q < J.len; q += 32) {
        const double2 x0 = xp[q];
#pragma unroll
        for (int c = 0; c < kColsPerJob; ++c) acc[c] = cfma_ca(__ldcs(vp + c * len + q), x0, acc[c]);
      }
    } else {
      for (; q < J.len; q += 32) {
        const double2 x0 = xp[q];
#pragma unroll
        for (int c = 0; c < kColsPerJob; ++c)
          if (c < nc) acc[c] = cfma_ca(__ldcs(vp + c * len + q), x0, acc[c]);
      }
    }
    // reduce-scatter of v[ri * C + c] over the 32 lanes: the first log2(2C)
    // xor stages halve the vector each lane carries, the rest finish the sum;
    // lane (q << kFin) holds value q = (ri, c) in bit-reversed-free order
    constexpr int NV = 2 * kColsPerJob;
    constexpr int kHalv = NV == 8 ? 3 : (NV == 16 ? 4 : 5);
    constexpr int kFin = 5 - kHalv;
    double v[NV];
#pragma unroll
    for (int c = 0; c < kColsPerJob; ++c) {
      v[c] = acc[c].x;
      v[kColsPerJob + c] = acc[c].y;
    }
#pragma unroll
    for (int st = 0; st < kHalv; ++st) {
      const int mask = 16 >> st, half = (NV / 2) >> st;
      const bool hi = (lane & mask) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const double send = hi ? v[i] : v[i + half];
        const double keep = hi ? v[i + half] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
      }
    }
#pragma unroll
    for (int st = 0; st < kFin; ++st) v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1 << st);
    if ((lane & ((1 << kFin) - 1)) == 0) {
      const int q = lane >> kFin;  // bits of q (MSB first) = the halving choices
      const int ri = q / kColsPerJob, c = q % kColsPerJob;
      if (c < nc) reinterpret_cast<double*>(s + J.soff + c)[ri] = v[0];
    }
  }
}

__global__ void __launch_bounds__(kThreads) mv_phase2(const MvTile2* __restrict__ tiles,
                                                      const double2* __restrict__ row,
                                                      const double2* __restrict__ s, double2* __restrict__ ylev,
                                                      const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ double2 red[kThreads];
  const MvTile2 T = tiles[blockIdx.x];
  const int tid = threadIdx.x;
  int r32 = ((T.nrows + 31) / 32) * 32;
  if (r32 > kThreads) r32 = kThreads;
  const int parts = kThreads / r32;
  const int rl = tid % r32, part = tid / r32;
  const bool valid = rl < T.nrows && part < parts;
  double2 a0 = cmk(0, 0), a1 = cmk(0, 0);
  if (valid) {
    const int64_t ld = T.ld;
    const double2* mp = row + T.moff + T.row0 + rl;
    const double2* sp = s + T.soff;
    int c = part;
    const int step = parts;
    for (; c + 3 * step < T.ncols; c += 4 * step) {
      const double2 m0 = mp[(int64_t)c * ld];
      const double2 m1 = mp[(int64_t)(c + step) * ld];
      const double2 m2 = mp[(int64_t)(c + 2 * step) * ld];
      const double2 m3 = mp[(int64_t)(c + 3 * step) * ld];
      const double2 s0 = sp[c], s1 = sp[c + step], s2 = sp[c + 2 * step], s3 = sp[c + 3 * step];
      a0 = cfma(m0, s0, a0);
      a1 = cfma(m1, s1, a1);
      a0 = cfma(m2, s2, a0);
      a1 = cfma(m3, s3, a1);
    }
    for (; c < T.ncols; c += step) a0 = cfma(mp[(int64_t)c * ld], sp[c], a0);
  }
  const double2 acc = cadd(a0, a1);
  if (parts == 1) {
    if (valid) ylev[T.yoff + T.row0 + rl] = acc;
    return;
  }
  red[tid] = acc;
  __syncthreads();
  if (part == 0 && rl < T.nrows) {
    double2 t = red[rl];
    for (int p = 1; p < parts; ++p) t = cadd(t, red[p * r32 + rl]);
    ylev[T.yoff + T.row0 + rl] = t;
  }
}

__global__ void mv_finalize(const double2* __restrict__ ylev, int64_t nlev, int64_t n, const int64_t* __restrict__ perm,
                            int d, double2* __restrict__ y, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double2 t = ylev[k];
    for (int64_t l = 1; l < nlev; ++l) t = cadd(t, ylev[l * n + k]);
    const int64_t p = k / d, a = k - p * d;
    y[d * perm[p] + a] = t;
  }
}

}  // namespace

void warm_matvec() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, mv_gather);
  cudaFuncGetAttributes(&a, mv_phase1);
  cudaFuncGetAttributes(&a, mv_phase2);
  cudaFuncGetAttributes(&a, mv_finalize);
}

void build_plan_pre(const DeviceH& H, PlanPre& pre) {
  const int64_t nb = H.nb;
  // row segments keyed by (r0, r1): leaves sorted by (r0 asc, r1 desc) = nesting order
  std::vector<int64_t> byrow(nb);
  std::iota(byrow.begin(), byrow.end(), int64_t(0));
  std::sort(byrow.begin(), byrow.end(), [&](int64_t a, int64_t b) {
    const int64_t a0 = H.table[5 * a + 1], b0 = H.table[5 * b + 1];
    if (a0 != b0) return a0 < b0;
    const int64_t a1 = H.table[5 * a + 2], b1 = H.table[5 * b + 2];
    return a1 != b1 ? a1 > b1 : a < b;
  });
  auto& segs = pre.segs;
  segs.clear();
  pre.bseg.assign(nb, 0);
  for (int64_t q = 0; q < nb; ++q) {
    const int64_t b = byrow[q];
    const std::pair<int64_t, int64_t> key(H.table[5 * b + 1], H.table[5 * b + 2]);
    if (segs.empty() || segs.back() != key) segs.push_back(key);
    pre.bseg[b] = (int64_t)segs.size() - 1;
  }
  const int64_t ns = (int64_t)segs.size();
  pre.level.assign(ns, 0);
  std::vector<int64_t> stack;
  int64_t maxlev = 0;
  for (int64_t g = 0; g < ns; ++g) {
    while (!stack.empty() && segs[stack.back()].second <= segs[g].first) stack.pop_back();
    pre.level[g] = (int64_t)stack.size();
    maxlev = std::max(maxlev, pre.level[g]);
    stack.push_back(g);
  }
  pre.nlevels = maxlev + 1;
}

// Builds segments, levels, stream offsets and the phase-1/phase-2 work lists.
// Requires H.table, H.rank_after (low-rank leaves), H.d, H.np.
int build_matvec_plan(DeviceH& H, const PlanPre* pre_in) {
  const auto t0 = std::chrono::steady_clock::now();
  const bool verbose = std::getenv("HMX_VERBOSE_PLAN") != nullptr;
  auto tick = [&](const char* what) {
    if (verbose)
      std::fprintf(stderr, "[hmx]   plan %-22s %9.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  const int d = H.d;
  const int64_t nb = H.nb;
  PlanPre own;
  const bool have = pre_in && !pre_in->segs.empty();  // e.g. no admissible leaf: no ACA pass built it
  if (!have) build_plan_pre(H, own);
  const PlanPre& pre = have ? *pre_in : own;
  const auto& segs = pre.segs;
  const auto& bseg = pre.bseg;
  const auto& level = pre.level;
  const int64_t ns = (int64_t)segs.size();
  H.nlevels = pre.nlevels;
  tick("segments");
  std::vector<int64_t> ncols(ns, 0), colstart(nb, 0);
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t g = bseg[b];
    colstart[b] = ncols[g];
    const int64_t n = H.table[5 * b + 4] - H.table[5 * b + 3];
    ncols[g] += H.table[5 * b] == 0 ? d * n : H.rank_after[b];
  }
  std::vector<int64_t> moff(ns), soff(ns);
  int64_t mo = 0, so = 0;
  for (int64_t g = 0; g < ns; ++g) {
    moff[g] = mo;
    soff[g] = so;
    mo += d * (segs[g].second - segs[g].first) * ncols[g];
    so += ncols[g];
  }
  H.row_elems = mo;
  H.s_elems = so;
  H.leaf_moff.assign(nb, 0);
  H.leaf_ld.assign(nb, 0);
  H.leaf_voff.assign(nb, -1);
  int64_t vo = 0;
  double dense_b = 0, lr_b = 0;
  // phase-1 jobs placed directly in longest-first order (counting sort on the
  // job length, stable in leaf order): one pass to count, one to place
  int32_t maxlen = 1;
  for (int64_t b = 0; b < nb; ++b) maxlen = std::max<int32_t>(maxlen, (int32_t)(d * (H.table[5 * b + 4] - H.table[5 * b + 3])));
  std::vector<int64_t> slot((size_t)maxlen + 2, 0);
  for (int64_t b = 0; b < nb; ++b) {
    const int32_t len = (int32_t)(d * (H.table[5 * b + 4] - H.table[5 * b + 3]));
    slot[(size_t)(maxlen - len) + 1] += H.table[5 * b] == 0 ? 1 : hmx_cdiv(H.rank_after[b], kColsPerJob);
  }
  for (size_t i = 1; i < slot.size(); ++i) slot[i] += slot[i - 1];
  std::vector<MvJob1> jobs((size_t)slot.back());
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t g = bseg[b];
    const int64_t m = H.table[5 * b + 2] - H.table[5 * b + 1];
    const int64_t n = H.table[5 * b + 4] - H.table[5 * b + 3];
    const int64_t ld = d * m;
    H.leaf_ld[b] = ld;
    H.leaf_moff[b] = moff[g] + colstart[b] * ld;
    const int64_t c0 = H.table[5 * b + 3];
    int64_t& pos = slot[(size_t)(maxlen - (int32_t)(d * n))];
    if (H.table[5 * b] == 0) {
      jobs[(size_t)pos++] = MvJob1{0, d * c0, soff[g] + colstart[b], (int32_t)(d * n), 0};
      dense_b += 16.0 * ld * d * n;
    } else {
      const int64_t r = H.rank_after[b];
      H.leaf_voff[b] = vo;
      for (int64_t l = 0; l < r; l += kColsPerJob)
        jobs[(size_t)pos++] = MvJob1{vo + l * d * n, d * c0, soff[g] + colstart[b] + l, (int32_t)(d * n),
                                     (int32_t)std::min<int64_t>(kColsPerJob, r - l)};
      vo += d * n * r;
      lr_b += 16.0 * r * d * (m + n);
    }
  }
  H.v_elems = vo;
  std::vector<MvTile2> tiles;
  // tile height: 256 rows (one thread per row), lowered to 128 / 64 / 32 rows for segments whose
  // 256-row tile would carry more than a fair share of the phase-2 bytes (the kernel then splits the
  // columns over 2 / 4 / 8 thread groups): the widest segments no longer leave one long CTA per
  // tile running after the rest (small configurations, few tiles per SM)
  double p2_total = 0.0;
  for (int64_t g = 0; g < ns; ++g) p2_total += 16.0 * (double)d * (segs[g].second - segs[g].first) * ncols[g];
  const double fair = p2_total / (4.0 * (double)std::max(1, H.ctx->num_sms));
  for (int64_t g = 0; g < ns; ++g) {
    if (ncols[g] == 0) continue;
    const int64_t rows = d * (segs[g].second - segs[g].first);
    int64_t th = kThreads;
    while (th > 32 && 16.0 * (double)std::min<int64_t>(th, rows) * ncols[g] > fair) th /= 2;
    for (int64_t r0 = 0; r0 < rows; r0 += th) {
      MvTile2 t;
      t.moff = moff[g];
      t.soff = soff[g];
      t.yoff = level[g] * H.n + d * segs[g].first;
      t.ld = (int32_t)rows;
      t.ncols = (int32_t)ncols[g];
      t.row0 = (int32_t)r0;
      t.nrows = (int32_t)std::min<int64_t>(th, rows - r0);
      tiles.push_back(t);
    }
  }
  std::stable_sort(tiles.begin(), tiles.end(), [](const MvTile2& a, const MvTile2& b) {
    return (int64_t)a.nrows * a.ncols > (int64_t)b.nrows * b.ncols;
  });
  H.njob1 = (int64_t)jobs.size();
  H.ntile2 = (int64_t)tiles.size();
  H.dense_bytes = dense_b;
  H.lr_bytes = lr_b;
  H.mv_bytes = dense_b + lr_b + 32.0 * H.n;
  // per-kernel algorithmic bytes: phase 1 streams V (+ x pieces -> dense slots),
  // phase 2 streams the row stream (dense leaves + U factors)
  {
    double copy_b = 0;
    for (const MvJob1& j : jobs)
      if (j.kind == 0) copy_b += 32.0 * j.len;
    H.phase1_bytes = 16.0 * H.v_elems + copy_b;
    H.phase2_bytes = 16.0 * H.row_elems;
  }
  tick("host layout");
  Ctx& c = *H.ctx;
  HMX_CUDA_TRY(dev_alloc_t(c, &H.d_row, (size_t)(std::max<int64_t>(H.row_elems, 1))));
  HMX_CUDA_TRY(dev_alloc_t(c, &H.d_v, (size_t)(std::max<int64_t>(H.v_elems, 1))));
  tick("malloc row + V");
  // the context stream's matvec workspace up front (other streams get theirs on first use)
  {
    int rc = HMX_OK;
    if (!mv_workspace(H, c.stream, &rc)) return rc;
  }
  HMX_CUDA_TRY(dev_alloc_t(c, &H.d_job1, (size_t)(std::max<int64_t>(H.njob1, 1))));
  HMX_CUDA_TRY(dev_alloc_t(c, &H.d_tile2, (size_t)(std::max<int64_t>(H.ntile2, 1))));
  if (H.njob1)
    HMX_CUDA_TRY(cudaMemcpyAsync(H.d_job1, jobs.data(), sizeof(MvJob1) * H.njob1, cudaMemcpyHostToDevice, c.stream));
  if (H.ntile2)
    HMX_CUDA_TRY(
        cudaMemcpyAsync(H.d_tile2, tiles.data(), sizeof(MvTile2) * H.ntile2, cudaMemcpyHostToDevice, c.stream));
  HMX_CUDA_TRY(cudaStreamSynchronize(c.stream));
  tick("rest");
  return HMX_OK;
}

MvWorkspace* mv_workspace(DeviceH& H, cudaStream_t s, int* rc) {
  std::lock_guard<std::mutex> lk(H.ws_mu);
  for (auto& w : H.ws)
    if (w->stream == s) return w.get();
  Ctx& c = *H.ctx;
  auto w = std::make_unique<MvWorkspace>();
  w->stream = s;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = dev_alloc_t(c, &w->d_s, (size_t)(std::max<int64_t>(H.s_elems, 1)));
  if (e == cudaSuccess) e = dev_alloc_t(c, &w->d_xt, (size_t)H.n);
  if (e == cudaSuccess) e = dev_alloc_t(c, &w->d_ylev, (size_t)(H.n * H.nlevels));
  if (e == cudaSuccess) e = cudaMemsetAsync(w->d_ylev, 0, sizeof(double2) * H.n * H.nlevels, s);
  if (e == cudaSuccess) e = dev_alloc_t(c, &w->d_xio, (size_t)H.n);
  if (e == cudaSuccess) e = dev_alloc_t(c, &w->d_yio, (size_t)H.n);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    hmx_set_error("matvec workspace: %s", cudaGetErrorString(e));
    cudaGetLastError();
    for (void* p : {(void*)w->d_s, (void*)w->d_xt, (void*)w->d_ylev, (void*)w->d_xio, (void*)w->d_yio})
      dev_free(c, p);
    *rc = e == cudaErrorMemoryAllocation ? HMX_ENOMEM : HMX_ECUDA;
    return nullptr;
  }
  H.ws.push_back(std::move(w));
  return H.ws.back().get();
}

void free_workspaces(DeviceH& H) {
  std::lock_guard<std::mutex> lk(H.ws_mu);
  for (auto& w : H.ws) {
    std::lock_guard<std::mutex> lw(w->mu);  // no call of another thread still enqueueing
    if (w->done) {
      cudaEventSynchronize(w->done);
      cudaEventDestroy(w->done);
    }
    for (void* p : {(void*)w->d_s, (void*)w->d_xt, (void*)w->d_ylev, (void*)w->d_xio, (void*)w->d_yio})
      dev_free(*H.ctx, p);
  }
  H.ws.clear();
}

int matvec_device(DeviceH& H, const double2* x, double2* y, float* phase_ms, cudaStream_t s, const int* gate) {
  int rc = HMX_OK;
  MvWorkspace* w = mv_workspace(H, s, &rc);
  if (!w) return rc;
  std::lock_guard<std::mutex> lk(w->mu);
  return matvec_enqueue(H, *w, x, y, phase_ms, gate);
}

int matvec_enqueue(DeviceH& H, MvWorkspace& W, const double2* x, double2* y, float* phase_ms, const int* gate) {
  Ctx& c = *H.ctx;
  const cudaStream_t st = W.stream;
  cudaEvent_t ev[5];
  const bool prof = H.profiling;  // diagnostic (hmx_profile_begin/end): one stream at a time
  const bool timed = phase_ms != nullptr || prof;
  if (timed) {
    for (int i = 0; i < 5; ++i) HMX_CUDA_TRY(cudaEventCreate(&ev[i]));
    HMX_CUDA_TRY(cudaEventRecord(ev[0], st));
  }
  const int eg = std::max<int64_t>(1, std::min<int64_t>(hmx_cdiv(H.n, kThreads), 4 * c.num_sms));
  mv_gather<<<eg, kThreads, 0, st>>>(x, H.d_perm, H.d, H.np, W.d_xt, gate);
  if (timed) HMX_CUDA_TRY(cudaEventRecord(ev[1], st));
  if (H.njob1) {
    const int64_t warps = std::min<int64_t>(H.njob1, (int64_t)c.num_sms * 64);  // 8 CTAs x 8 warps per SM
    mv_phase1<<<(unsigned)hmx_cdiv(warps * 32, kThreads), kThreads, 0, st>>>(H.d_job1, H.njob1, H.d_v, W.d_xt,
                                                                             W.d_s, gate);
  }
  if (timed) HMX_CUDA_TRY(cudaEventRecord(ev[2], st));
  if (H.ntile2) mv_phase2<<<(unsigned)H.ntile2, kThreads, 0, st>>>(H.d_tile2, H.d_row, W.d_s, W.d_ylev, gate);
  if (timed) HMX_CUDA_TRY(cudaEventRecord(ev[3], st));
  mv_finalize<<<eg, kThreads, 0, st>>>(W.d_ylev, H.nlevels, H.n, H.d_perm, H.d, y, gate);
  HMX_CUDA_TRY(cudaGetLastError());
  HMX_CUDA_TRY(cudaEventRecord(W.done, st));
  if (timed) HMX_CUDA_TRY(cudaEventRecord(ev[4], st));
  if (prof && !phase_ms) {
    std::lock_guard<std::mutex> lk(H.ws_mu);
    H.prof_events.insert(H.prof_events.end(), ev, ev + 5);
  } else if (phase_ms) {
    HMX_CUDA_TRY(cudaEventSynchronize(ev[4]));
    for (int i = 0; i < 4; ++i) HMX_CUDA_TRY(cudaEventElapsedTime(&phase_ms[i], ev[i], ev[i + 1]));
    for (int i = 0; i < 5; ++i) cudaEventDestroy(ev[i]);
  }
  return HMX_OK;
}

}  // namespace hmx
