// Batched recompression of every ACA factor pair (SPEC.md:318-326,
// PAPER.md:431-443): the reference does QR(U), QR(V), SVD(R_U R_V^H),
// truncation, U' = Q_U P S^1/2, V' = Q_V L S^1/2.
//
// B200 formulation (same singular values, same subspaces, no tall QR): the ACA
// kernel already accumulated the Gram matrices G_U = U^H U and G_V = V^H V.
//   R   = chol(G_V)            (diagonally scaled; Q_V = V R^{-1})
//   E   = R G_U R^H = Y^H Y    (Y = U R^H, so U V^H = Y Q_V^H)
//   E   = L S^2 L^H            (cyclic parallel Jacobi, Hermitian)
//   r   = truncation rank of s (oracle/lowrank.py decision 8)
//   W_U = R^H L_r S_r^{-1/2},  W_V = R^{-1} L_r S_r^{1/2}
//   U'  = U W_U,  V' = V W_V   (batched tiled complex GEMM, launch_form)
// so U' V'^H = U V^H Q_V L_r L_r^H Q_V^H: the rank-r truncated SVD of the ACA
// product, identical to the reference pipeline up to roundoff.
#include "hmatrix.h"

namespace hmx {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSmemEigenMax = 112;  // E kept in shared memory up to this K

struct Rot {
  int p, q;
  double cs, sn;
  double2 u;  // phase of E_pq
  int active;
};

HMX_D double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kWarps; ++w) t += red[w];
  return t;
}

// Hermitian Jacobi eigensolver on E (ld = lde) accumulating eigenvectors in
// L (K x K, ld K, global).  Pairs follow the round-robin (circle) schedule.
__device__ void jacobi_eigen(double2* E, int lde, double2* L, int K, Rot* rot, double* red) {
  const int tid = threadIdx.x;
  const int Kp = K + (K & 1);
  const int npairs = Kp / 2;
  for (int t = tid; t < K * K; t += kThreads) {
    const int i = t % K, j = t / K;
    L[i + (int64_t)j * K] = cmk(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int t = tid; t < K * K; t += kThreads) {
      const int i = t % K, j = t / K;
      const double a = cabs2(E[i + (int64_t)j * lde]);
      tot += a;
      if (i != j) off += a;
    }
    off = block_sum(off, red);
    tot = block_sum(tot, red);
    if (off <= 1e-30 * tot || K < 2) break;
    for (int rnd = 0; rnd < Kp - 1; ++rnd) {
      for (int k = tid; k < npairs; k += kThreads) {
        int a = (k == 0) ? 0 : ((rnd + k - 1) % (Kp - 1)) + 1;
        int b = ((rnd + Kp - 2 - k) % (Kp - 1)) + 1;
        int p = a < b ? a : b, q = a < b ? b : a;
        Rot R;
        R.p = p;
        R.q = q;
        R.active = 0;
        R.cs = 1.0;
        R.sn = 0.0;
        R.u = cmk(1.0, 0.0);
        if (q < K) {
          const double app = E[p + (int64_t)p * lde].x, aqq = E[q + (int64_t)q * lde].x;
          const double2 c = E[p + (int64_t)q * lde];
          const double ac = sqrt(cabs2(c));
          if (ac > 1e-300 && ac > 1e-17 * sqrt(fabs(app * aqq))) {
            const double tau = (aqq - app) / (2.0 * ac);
            const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            R.cs = 1.0 / sqrt(1.0 + tt * tt);
            R.sn = tt * R.cs;
            R.u = cscale(c, 1.0 / ac);
            R.active = 1;
          }
        }
        rot[k] = R;
      }
      __syncthreads();
      // columns: E[:,p], E[:,q] <- (E_p cs - E_q conj(u) sn, E_p sn + E_q conj(u) cs); same for L
      for (int t = tid; t < npairs * K; t += kThreads) {
        const int k = t / K, i = t - k * K;
        const Rot R = rot[k];
        if (!R.active) continue;
        const double2 cu = cconj(R.u);
        {
          const double2 ep = E[i + (int64_t)R.p * lde], eq = E[i + (int64_t)R.q * lde];
          const double2 equ = cmul(eq, cu);
          E[i + (int64_t)R.p * lde] = csub(cscale(ep, R.cs), cscale(equ, R.sn));
          E[i + (int64_t)R.q * lde] = cadd(cscale(ep, R.sn), cscale(equ, R.cs));
        }
        {
          const double2 lp = L[i + (int64_t)R.p * K], lq = L[i + (int64_t)R.q * K];
          const double2 lqu = cmul(lq, cu);
          L[i + (int64_t)R.p * K] = csub(cscale(lp, R.cs), cscale(lqu, R.sn));
          L[i + (int64_t)R.q * K] = cadd(cscale(lp, R.sn), cscale(lqu, R.cs));
        }
      }
      __syncthreads();
      // rows: E[p,:], E[q,:] <- (cs E_p - u sn E_q, sn E_p + u cs E_q)
      for (int t = tid; t < npairs * K; t += kThreads) {
        const int k = t / K, i = t - k * K;
        const Rot R = rot[k];
        if (!R.active) continue;
        const double2 ep = E[R.p + (int64_t)i * lde], eq = E[R.q + (int64_t)i * lde];
        const double2 ueq = cmul(R.u, eq);
        E[R.p + (int64_t)i * lde] = csub(cscale(ep, R.cs), cscale(ueq, R.sn));
        E[R.q + (int64_t)i * lde] = cadd(cscale(ep, R.sn), cscale(ueq, R.cs));
      }
      __syncthreads();
    }
  }
}

// One CTA per low-rank leaf.  Workspace per leaf (ld K): A = R, B = T then L,
// C = E (when not in shared memory), Wu | Wv (K x r each).
__global__ void __launch_bounds__(kThreads) recompress_core(const RecDesc* __restrict__ desc, double eps, int rule,
                                                            const double2* __restrict__ G, double2* __restrict__ W,
                                                            int32_t* __restrict__ rank_out,
                                                            int32_t* __restrict__ flags_out) {
  extern __shared__ double2 dyn[];
  __shared__ Rot rot[320];
  __shared__ double red[kWarps];
  __shared__ int s_r, s_flag;
  const int tid = threadIdx.x;
  const RecDesc ds = desc[blockIdx.x];
  const int K = ds.K, kcap = ds.kcap;
  if (K == 0) {
    if (tid == 0) {
      rank_out[blockIdx.x] = 0;
      flags_out[blockIdx.x] = 0;
    }
    return;
  }
  const double2* GU = G + ds.goff;
  const double2* GV = GU + (int64_t)kcap * kcap;
  const int64_t KK = (int64_t)K * K;
  double2* A = W + ds.woff;  // R (upper)
  double2* B = A + KK;       // T, then L
  double2* Cg = B + KK;      // E (global fallback)
  double2* Wuv = Cg + KK;    // Wu (K x r) then Wv (K x r)
  double* dscale = reinterpret_cast<double*>(dyn);  // K scale factors + K eigenvalues + K order
  double* lam = dscale + K;
  int* ordr = reinterpret_cast<int*>(lam + K);
  const bool smemE = K <= kSmemEigenMax;
  double2* E = smemE ? reinterpret_cast<double2*>(dyn) + (3 * K + 1) / 2 + 1 : Cg;
  const int lde = K;

  if (tid == 0) s_flag = 0;
  // ---- scaled Cholesky of G_V: A = D^-1 G_V D^-1, R^H R = A (upper R) ----------
  for (int i = tid; i < K; i += kThreads) {
    const double g = GV[i + (int64_t)i * kcap].x;
    dscale[i] = g > 0.0 ? sqrt(g) : 1.0;
  }
  __syncthreads();
  for (int t = tid; t < K * K; t += kThreads) {
    const int i = t % K, j = t / K;
    const double2 g = GV[i + (int64_t)j * kcap];
    A[t] = (i <= j) ? cscale(g, 1.0 / (dscale[i] * dscale[j])) : cmk(0.0, 0.0);
  }
  __syncthreads();
  // right-looking, row j of R finalised per step (A upper triangle in place)
  for (int j = 0; j < K; ++j) {
    __shared__ double s_piv;
    if (tid == 0) {
      double p = A[j + (int64_t)j * K].x;
      if (!(p > 1e-14)) {
        p = 1e-14;
        s_flag |= 1;  // regularised
      }
      s_piv = sqrt(p);
      A[j + (int64_t)j * K] = cmk(s_piv, 0.0);
    }
    __syncthreads();
    const double ip = 1.0 / s_piv;
    for (int i = j + 1 + tid; i < K; i += kThreads) A[j + (int64_t)i * K] = cscale(A[j + (int64_t)i * K], ip);
    __syncthreads();
    // trailing update A[i,l] -= conj(R[j,i]) R[j,l] for j < i <= l
    const int rem = K - j - 1;
    for (int t = tid; t < rem * rem; t += kThreads) {
      const int i = j + 1 + t % rem, l = j + 1 + t / rem;
      if (i > l) continue;
      const double2 rji = A[j + (int64_t)i * K], rjl = A[j + (int64_t)l * K];
      A[i + (int64_t)l * K] = csub(A[i + (int64_t)l * K], cmul(cconj(rji), rjl));
    }
    __syncthreads();
  }
  // undo the scaling: R = Rhat D
  for (int t = tid; t < K * K; t += kThreads) {
    const int i = t % K, j = t / K;
    A[t] = (i <= j) ? cscale(A[t], dscale[j]) : cmk(0.0, 0.0);
  }
  __syncthreads();
  // ---- T = R G_U (B), E = T R^H ---------------------------------------------
  for (int t = tid; t < K * K; t += kThreads) {
    const int i = t % K, j = t / K;
    double2 s = cmk(0.0, 0.0);
    for (int k = i; k < K; ++k) s = cfma(A[i + (int64_t)k * K], GU[k + (int64_t)j * kcap], s);
    B[t] = s;
  }
  __syncthreads();
  for (int t = tid; t < K * K; t += kThreads) {
    const int i = t % K, j = t / K;
    double2 s = cmk(0.0, 0.0);
    for (int k = j; k < K; ++k) s = cfma_cj(B[i + (int64_t)k * K], A[j + (int64_t)k * K], s);
    E[i + (int64_t)j * lde] = s;
  }
  __syncthreads();
  // Hermitian symmetrise (roundoff) before Jacobi
  for (int t = tid; t < K * K; t += kThreads) {
    const int i = t % K, j = t / K;
    if (i < j) {
      const double2 a = E[i + (int64_t)j * lde], b = E[j + (int64_t)i * lde];
      const double2 h = cscale(cadd(a, cconj(b)), 0.5);
      E[i + (int64_t)j * lde] = h;
      E[j + (int64_t)i * lde] = cconj(h);
    } else if (i == j) {
      E[i + (int64_t)i * lde].y = 0.0;
    }
  }
  __syncthreads();
  jacobi_eigen(E, lde, B, K, rot, red);
  // ---- eigenvalues, descending order (rank sort, ties by index) ------------------
  for (int i = tid; i < K; i += kThreads) lam[i] = fmax(E[i + (int64_t)i * lde].x, 0.0);
  __syncthreads();
  for (int i = tid; i < K; i += kThreads) {
    int rk = 0;
    const double li = lam[i];
    for (int j = 0; j < K; ++j) rk += (lam[j] > li) || (lam[j] == li && j < i);
    ordr[rk] = i;
  }
  __syncthreads();
  if (tid == 0) {
    // truncation (oracle/lowrank.py truncation_rank)
    int r = 0;
    const double l1 = lam[ordr[0]];
    if (l1 > 0.0) {
      if (rule == 1) {
        for (int k = 0; k < K; ++k) r += lam[ordr[k]] > eps * eps * l1;
      } else {
        double total = 0.0;
        for (int k = K - 1; k >= 0; --k) total += lam[ordr[k]];
        double tail = total;  // tail[r] = sum_{k >= r}
        r = K;
        double acc = 0.0;
        // smallest r with sum_{k >= r} lam <= eps^2 total
        for (int k = K - 1; k >= 0; --k) {
          acc += lam[ordr[k]];
          if (acc <= eps * eps * total) r = k;
        }
        (void)tail;
      }
    }
    s_r = r;
    rank_out[blockIdx.x] = r;
    flags_out[blockIdx.x] = s_flag;
  }
  __syncthreads();
  const int r = s_r;
  // ---- W_U = R^H L_r S^-1/2 ------------------------------------------------------
  double2* Wu = Wuv;
  double2* Wv = Wuv + (int64_t)K * r;
  for (int t = tid; t < K * r; t += kThreads) {
    const int i = t % K, c = t / K;
    const int e = ordr[c];
    double2 s = cmk(0.0, 0.0);
    for (int k = 0; k <= i; ++k) s = cfma_ca(A[k + (int64_t)i * K], B[k + (int64_t)e * K], s);
    Wu[t] = cscale(s, 1.0 / sqrt(sqrt(lam[e])));
  }
  // ---- W_V = R^{-1} L_r S^1/2 (back substitution, one thread per column) ----------
  for (int c = tid; c < r; c += kThreads) {
    const int e = ordr[c];
    const double sc = sqrt(sqrt(lam[e]));
    for (int i = K - 1; i >= 0; --i) {
      double2 s = B[i + (int64_t)e * K];
      for (int k = i + 1; k < K; ++k) s = csub(s, cmul(A[i + (int64_t)k * K], Wv[k + (int64_t)c * K]));
      Wv[i + (int64_t)c * K] = cdiv(s, A[i + (int64_t)i * K]);
    }
    for (int i = 0; i < K; ++i) Wv[i + (int64_t)c * K] = cscale(Wv[i + (int64_t)c * K], sc);
  }
}

// C (rows x r, ldc) = A (rows x K, lda) * W (K x r, ld K); one CTA = 64 x 32 tile.
constexpr int TM = 64, TN = 32, TK = 16;
__global__ void __launch_bounds__(kThreads) form_gemm(const FormDesc* __restrict__ desc,
                                                      const int64_t* __restrict__ tile_start, int64_t nitems,
                                                      const double2* __restrict__ Abase,
                                                      const double2* __restrict__ Wbase, double2* __restrict__ Cbase) {
  __shared__ double2 As[TK][TM + 1];
  __shared__ double2 Ws[TK][TN + 1];
  // locate item by binary search over tile_start
  const int64_t tile = blockIdx.x;
  int64_t lo = 0, hi = nitems - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= tile) lo = mid;
    else hi = mid - 1;
  }
  const FormDesc ds = desc[lo];
  const int64_t local = tile - tile_start[lo];
  const int ntm = (ds.rows + TM - 1) / TM;
  const int tm = (int)(local % ntm), tn = (int)(local / ntm);
  const double2* A = Abase + ds.aoff;
  const double2* W = Wbase + ds.woff;
  double2* C = Cbase + ds.coff;
  const int tid = threadIdx.x;
  const int tr = tid % 32, tc = tid / 32;  // thread computes rows tr, tr+32 ; cols tc, tc+8, tc+16, tc+24
  double2 acc[2][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = cmk(0.0, 0.0);
  const int row0 = tm * TM, col0 = tn * TN;
  for (int k0 = 0; k0 < ds.K; k0 += TK) {
    for (int t = tid; t < TK * TM; t += kThreads) {
      const int rr = t % TM, kk = t / TM;
      const int gr = row0 + rr, gk = k0 + kk;
      As[kk][rr] = (gr < ds.rows && gk < ds.K) ? A[gr + (int64_t)gk * ds.lda] : cmk(0.0, 0.0);
    }
    for (int t = tid; t < TK * TN; t += kThreads) {
      const int kk = t % TK, cc = t / TK;
      const int gk = k0 + kk, gc = col0 + cc;
      Ws[kk][cc] = (gk < ds.K && gc < ds.r) ? W[gk + (int64_t)gc * ds.K] : cmk(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < TK; ++kk) {
      const double2 a0 = As[kk][tr], a1 = As[kk][tr + 32];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double2 w = Ws[kk][tc + 8 * b];
        acc[0][b] = cfma(a0, w, acc[0][b]);
        acc[1][b] = cfma(a1, w, acc[1][b]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int gr = row0 + tr + 32 * a, gc = col0 + tc + 8 * b;
      if (gr < ds.rows && gc < ds.r) C[gr + (int64_t)gc * ds.ldc] = acc[a][b];
    }
}

}  // namespace

int launch_recompress_core(Ctx& c, const RecDesc* d_desc, int64_t nblk, int kmax, double eps, int rule, double2* G,
                           double2* W, int32_t* d_rank, int32_t* d_flags) {
  if (nblk == 0) return HMX_OK;
  if (kmax > 2 * 320) {
    hmx_set_error("recompress: ACA rank %d exceeds the Jacobi pair table", kmax);
    return HMX_EINVAL;
  }
  const int ke = kmax <= kSmemEigenMax ? kmax : 0;
  size_t smem = sizeof(double) * 3 * (size_t)kmax + 16 + sizeof(double2) * ((size_t)ke * ke + 2);
  HMX_CUDA_TRY(cudaFuncSetAttribute(recompress_core, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  recompress_core<<<(unsigned)nblk, kThreads, smem, c.stream>>>(d_desc, eps, rule, G, W, d_rank, d_flags);
  HMX_CUDA_TRY(cudaGetLastError());
  return HMX_OK;
}

int launch_form(Ctx& c, const FormDesc* d_desc, int64_t nitems, int64_t ntiles_total, const int64_t* d_tile_start,
                const double2* A, const double2* W, double2* C) {
  if (ntiles_total == 0) return HMX_OK;
  form_gemm<<<(unsigned)ntiles_total, kThreads, 0, c.stream>>>(d_desc, d_tile_start, nitems, A, W, C);
  HMX_CUDA_TRY(cudaGetLastError());
  return HMX_OK;
}

}  // namespace hmx
