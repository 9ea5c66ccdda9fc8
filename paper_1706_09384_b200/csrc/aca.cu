// Batched partially pivoted ACA over every admissible leaf at once.
//
// Algorithm: PAPER.md:261-280 (scalar, six steps) and PAPER.md:373-378 /
// SPEC.md:298-306 (vector, rank-d updates with sigma_3 pivoting), with the
// pinned decisions of oracle/lowrank.py (decisions 1-7) -- the CPU oracle and
// this kernel implement the same step sequence, so pivots agree except on
// roundoff-level near-ties (ranks compared +/-1 in tests/test_gpu_parity.py).
//
// Mapping: one CTA per admissible block (512 threads for large blocks, 128 for
// small ones), blocks taken in LPT order (largest first).  Per step:
//   row pass   thread per column point j: Green's d x d block of (i_piv, j)
//              minus U(i_piv,:) V(j,:)^H  -> written conjugated as the new V
//              columns (v_k = R_row^H), sigma_1 / sigma_3 per sub-block,
//              block argmax of sigma_3 (lowest index on ties)
//   pivot      gamma = R(i_piv, j_piv)^{-1}
//   col pass   thread per row point i: (i, j_piv) block minus U(i,:) V(j_piv,:)^H,
//              sigma_3 over unvisited rows -> next row pivot, u_k = R_col gamma
//   Gram pass  G_U(:, new) = U^H u_new, G_V(:, new) = V^H v_new, warp per
//              kGramGroup factor columns, lanes over rows (these Gram matrices
//              give the exact ||B_k||_F update of SPEC.md:338 and are reused by
//              the recompression)
//   decision   ||B_k||^2 update, stop test ||u|| ||v|| <= eps ||B_k||.
// The Gram pass re-streams both factor panels from HBM (they do not fit in a
// CTA's share of L2), so it is run once per kGramBatch steps for all their new
// columns together: the stop decisions of the batched steps are then taken in
// order, and a step after the one that stops is discarded (it was speculative:
// nothing the decision reads depends on it).  Where a step cannot run (column
// capacity, max rank, no unvisited row, zero residual row, sigma_3 fallback)
// the pending steps are resolved first, so every outcome is the one the
// sequential algorithm produces.
// The residual strips are written straight into the factor storage; U/V are
// column-major with ld = d m / d n, the U(i_piv,:) and V(j_piv,:) rows are
// staged in shared memory.
#include <cstdio>
#include <cstdlib>

#include "green.cuh"
#include "hmatrix.h"

namespace hmx {

namespace {

#ifndef HMX_GRAM_GROUP
#define HMX_GRAM_GROUP 4
#endif
constexpr int kGramGroup = HMX_GRAM_GROUP;  // factor columns per warp in the Gram pass
#ifndef HMX_GRAM_BATCH
#define HMX_GRAM_BATCH 1
#endif
constexpr int kGramBatch = HMX_GRAM_BATCH;  // steps per Gram pass (max)

// Reciprocal from the MUFU approximation refined by three Newton steps (full double precision):
// the sigma Newton iterations below are chains of divisions
HMX_D double rcp3(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
#pragma unroll
  for (int k = 0; k < 3; ++k) r = fma(r, fma(-q, r, 1.0), r);
  return r;
}

// sigma_1 and sigma_3 of a 3x3 complex matrix from the characteristic
// polynomial of R^H R: c2 = ||R||_F^2, c1 = sum |2x2 minors|^2 (Cauchy-Binet),
// c0 = |det R|^2.  Smallest root by Newton from c0/c1 (monotone from below on
// the concave branch), largest from c2 (monotone from above).
HMX_D void svals3(const double2* R, double& s1, double& s3) {
  double c2 = 0.0;
#pragma unroll
  for (int t = 0; t < 9; ++t) c2 += cabs2(R[t]);
  // minors M[ab][cd] for rows (a,b) cols (c,d)
  double c1 = 0.0;
  double2 cof0 = cmk(0, 0), cof1 = cmk(0, 0), cof2 = cmk(0, 0);
#pragma unroll
  for (int ra = 0; ra < 3; ++ra) {
    const int r1 = (ra + 1) % 3, r2 = (ra + 2) % 3;
#pragma unroll
    for (int ca = 0; ca < 3; ++ca) {
      const int k1 = (ca + 1) % 3, k2 = (ca + 2) % 3;
      const double2 mnr = csub(cmul(R[3 * r1 + k1], R[3 * r2 + k2]), cmul(R[3 * r1 + k2], R[3 * r2 + k1]));
      c1 += cabs2(mnr);
      if (ra == 0) {
        if (ca == 0) cof0 = mnr;
        if (ca == 1) cof1 = mnr;
        if (ca == 2) cof2 = mnr;
      }
    }
  }
  double2 det = cmul(R[0], cof0);
  det = cadd(det, cmul(R[1], cof1));
  det = cadd(det, cmul(R[2], cof2));
  const double c0 = cabs2(det);
  if (c2 <= 0.0) {
    s1 = s3 = 0.0;
    return;
  }
  // largest root
  double lam = c2;
#pragma unroll 1
  for (int it = 0; it < 60; ++it) {
    const double f = ((lam - c2) * lam + c1) * lam - c0;
    const double fp = (3.0 * lam - 2.0 * c2) * lam + c1;
    if (!(fp > 0.0)) break;
    const double nl = lam - f * rcp3(fp);
    if (!(nl < lam)) break;
    lam = nl;
  }
  s1 = sqrt(fmax(lam, 0.0));
  if (c0 <= 0.0 || c1 <= 0.0) {
    s3 = 0.0;
    return;
  }
  double mu = c0 * rcp3(c1);
#pragma unroll 1
  for (int it = 0; it < 60; ++it) {
    const double f = ((mu - c2) * mu + c1) * mu - c0;
    const double fp = (3.0 * mu - 2.0 * c2) * mu + c1;
    if (!(fp > 0.0)) break;
    const double nm = mu - f * rcp3(fp);
    if (!(nm > mu)) break;
    mu = nm;
  }
  s3 = sqrt(fmax(mu, 0.0));
}

template <int D>
HMX_D void svals(const double2* R, double& s1, double& s3) {
  if (D == 1) {
    s1 = s3 = sqrt(cabs2(R[0]));
  } else {
    svals3(R, s1, s3);
  }
}

// gamma = P^{-1}, row-major d x d
template <int D>
HMX_D void inverse(const double2* P, double2* G) {
  if (D == 1) {
    G[0] = cdiv(cmk(1.0, 0.0), P[0]);
    return;
  }
  double2 adj[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      // cofactor C_ab -> adj_ba
      const int r1 = (a + 1) % 3, r2 = (a + 2) % 3, k1 = (b + 1) % 3, k2 = (b + 2) % 3;
      adj[3 * b + a] = csub(cmul(P[3 * r1 + k1], P[3 * r2 + k2]), cmul(P[3 * r1 + k2], P[3 * r2 + k1]));
    }
  double2 det = cadd(cadd(cmul(P[0], adj[0]), cmul(P[1], adj[3])), cmul(P[2], adj[6]));
  const double2 idet = cdiv(cmk(1.0, 0.0), det);
#pragma unroll
  for (int t = 0; t < 9; ++t) G[t] = cmul(adj[t], idet);
}

constexpr int kMaxWarps = 32;
struct Shared {
  int ipiv, jpiv, K, steps, state, zero_rows, verdict, npend, rowout, nextrow, stop, bbi, kfinal, sfinal;
  double normB2, s1max, bbv;
  double2 gamma[9];
  double red_v[kMaxWarps];
  int red_i[kMaxWarps];
  double red_s[kMaxWarps];
  double red_a[kMaxWarps];
};

// state codes / row-pass outcomes
constexpr int kRun = 0, kZeroRow = 1, kDone = 2;
constexpr int kRowPivot = 0, kRowZero = 1, kRowFallback = 2;

// Gram columns G(:, Kc:Kc+NC) = F^H F(:, Kc:Kc+NC) for NC new columns, rows
// l < Kc + NC, both factor panels; warp per kGramGroup columns l, lanes over
// factor rows (contiguous 512 B per load instruction).
template <int NC, int NT>
HMX_D void gram_columns(const double2* __restrict__ Ub, const double2* __restrict__ Vb, int64_t ldu, int64_t ldv,
                        double2* __restrict__ GU, double2* __restrict__ GV, int kcap, int Kc, int sides = 3) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Kn = Kc + NC;
  const int ngroups = (Kn + kGramGroup - 1) / kGramGroup;
  for (int side = 0; side < 2; ++side) {
    if (!((sides >> side) & 1)) continue;
    const double2* F = side == 0 ? Ub : Vb;
    const int64_t ld = side == 0 ? ldu : ldv;
    double2* Gm = side == 0 ? GU : GV;
    for (int grp = warp; grp < ngroups; grp += NW) {
      double2 acc[kGramGroup][NC];
#pragma unroll
      for (int t = 0; t < kGramGroup; ++t)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[t][c] = cmk(0.0, 0.0);
      const int l0 = grp * kGramGroup;
#pragma unroll 2
      for (int64_t q = lane; q < ld; q += 32) {
        double2 nf[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) nf[c] = F[q + (int64_t)(Kc + c) * ld];
#pragma unroll
        for (int t = 0; t < kGramGroup; ++t) {
          if (l0 + t < Kn) {
            const double2 fl = F[q + (int64_t)(l0 + t) * ld];
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[t][c] = cfma_ca(fl, nf[c], acc[t][c]);
          }
        }
      }
      constexpr int NV = 2 * kGramGroup * NC;  // doubles to sum over the warp
      if constexpr (NV <= 32) {
        // butterfly reduce-scatter (as mv_phase1): each xor stage halves the vector a lane carries,
        // so NV values cost ~NV shuffles instead of 5 NV; lane (q << kFin) ends with value q =
        // 2 (t NC + c) + {re, im}, and the even ones write their complex Gram entry
        constexpr int P = NV <= 8 ? 8 : (NV <= 16 ? 16 : 32);
        constexpr int kHalv = P == 8 ? 3 : (P == 16 ? 4 : 5);
        constexpr int kFin = 5 - kHalv;
        double v[P];
#pragma unroll
        for (int t = 0; t < kGramGroup; ++t)
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            v[2 * (t * NC + c)] = acc[t][c].x;
            v[2 * (t * NC + c) + 1] = acc[t][c].y;
          }
#pragma unroll
        for (int q = NV; q < P; ++q) v[q] = 0.0;
#pragma unroll
        for (int st = 0; st < kHalv; ++st) {
          const int mask = 16 >> st, half = (P / 2) >> st;
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
        const double im = __shfl_down_sync(0xffffffffu, v[0], 1 << kFin);
        const int q = lane >> kFin;
        if ((lane & ((1 << kFin) - 1)) == 0 && (q & 1) == 0 && q < NV) {
          const int t = (q >> 1) / NC, c = (q >> 1) % NC;
          const int l = l0 + t, col = Kc + c;
          const double2 val = cmk(v[0], im);
          if (l < Kn) {
            if (l < Kc || l < col) {
              Gm[l + (int64_t)col * kcap] = val;
              Gm[col + (int64_t)l * kcap] = cconj(val);
            } else if (l == col) {
              Gm[l + (int64_t)col * kcap] = cmk(val.x, 0.0);
            }
          }
        }
        continue;
      }
#pragma unroll
      for (int t = 0; t < kGramGroup; ++t)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[t][c] = warp_sum(acc[t][c]);
      if (lane == 0) {
#pragma unroll
        for (int t = 0; t < kGramGroup; ++t) {
          const int l = l0 + t;
          if (l >= Kn) continue;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const int col = Kc + c;
            if (l < Kc || l < col) {
              Gm[l + (int64_t)col * kcap] = acc[t][c];
              Gm[col + (int64_t)l * kcap] = cconj(acc[t][c]);
            } else if (l == col) {
              Gm[l + (int64_t)col * kcap] = cmk(acc[t][c].x, 0.0);
            }
          }
        }
      }
    }
  }
}

// ||B||_F^2 update with the Gram columns Ks..Ks+D-1 and the stop test
// (oracle/lowrank.py decisions 4-5); result in sh.stop.
template <int D, int NT>
HMX_D void decide_step(const double2* __restrict__ GU, const double2* __restrict__ GV, int kcap, int Ks, double eps,
                       Shared& sh) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double cross = 0.0;
  for (int t = tid; t < Ks * D; t += NT) {
    const int l = t / D, c = t - l * D;
    const double2 gu = GU[l + (int64_t)(Ks + c) * kcap];
    const double2 gv = GV[l + (int64_t)(Ks + c) * kcap];
    cross += gu.x * gv.x + gu.y * gv.y;
  }
  cross = warp_sum(cross);
  if (lane == 0) sh.red_a[warp] = cross;
  __syncthreads();
  if (tid == 0) {
    double crs = 0.0;
    for (int w = 0; w < NW; ++w) crs += sh.red_a[w];
    double diag = 0.0, nu = 0.0, nv = 0.0;
    for (int c = 0; c < D; ++c) {
      nu += GU[(Ks + c) + (int64_t)(Ks + c) * kcap].x;
      nv += GV[(Ks + c) + (int64_t)(Ks + c) * kcap].x;
      for (int q = 0; q < D; ++q) {
        const double2 a = GU[(Ks + c) + (int64_t)(Ks + q) * kcap];
        const double2 bq = GV[(Ks + q) + (int64_t)(Ks + c) * kcap];
        diag += a.x * bq.x - a.y * bq.y;
      }
    }
    sh.normB2 = sh.normB2 + 2.0 * crs + diag;
    sh.stop = sqrt(nu) * sqrt(nv) <= eps * sqrt(fmax(sh.normB2, 0.0));
  }
  __syncthreads();
}

// Gram columns of the npend pending steps (one pass) and their stop decisions
// in order.  sh.kfinal / sh.sfinal = rank / step count at the first step that
// stops (sh.stop = 1), else the whole batch is accepted (sh.stop = 0).
template <int D, int NT, int BMAX>
HMX_D void resolve_pending(const double2* __restrict__ Ub, const double2* __restrict__ Vb, int64_t ldu, int64_t ldv,
                           double2* __restrict__ GU, double2* __restrict__ GV, int kcap, double eps, Shared& sh) {
  const int npend = sh.npend;
  const int K = sh.K;
  const int Kc = K - npend * D;
  if (BMAX == 1 || npend == 1)
    gram_columns<D, NT>(Ub, Vb, ldu, ldv, GU, GV, kcap, Kc);
  else
    gram_columns<D * (BMAX > 1 ? 2 : 1), NT>(Ub, Vb, ldu, ldv, GU, GV, kcap, Kc);
  __syncthreads();
  int stop = 0;
  for (int p = 0; p < npend && !stop; ++p) {
    decide_step<D, NT>(GU, GV, kcap, Kc + p * D, eps, sh);
    stop = sh.stop;
    if (stop && threadIdx.x == 0) {
      sh.kfinal = Kc + (p + 1) * D;
      sh.sfinal = sh.steps - (npend - 1 - p);
    }
  }
  if (threadIdx.x == 0) {
    sh.stop = stop;
    sh.npend = 0;
  }
  __syncthreads();
}

template <int D, int KIND, int NT, int MINB, int BMAX>
__global__ void __launch_bounds__(NT, MINB) aca_kernel(GreenParams P, PointsSoA pts, const AcaDesc* __restrict__ desc,
                                                       const int32_t* __restrict__ order, double eps, double floor,
                                                       double2* __restrict__ U, double2* __restrict__ V,
                                                       double2* __restrict__ G, AcaOut* __restrict__ out,
                                                       int kcap_max, int batch) {
  extern __shared__ double2 dyn[];
  __shared__ Shared sh;
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = order[blockIdx.x];
  const AcaDesc ds = desc[b];
  const int m = ds.m, n = ds.n, kcap = ds.kcap;
  const int64_t ldu = (int64_t)D * m, ldv = (int64_t)D * n;
  double2* __restrict__ Ub = U + ds.uoff;
  double2* __restrict__ Vb = V + ds.voff;
  double2* __restrict__ GU = G + ds.goff;
  double2* __restrict__ GV = GU + (int64_t)kcap * kcap;
  double2* Urow = dyn;                 // D x kcap_max
  double2* Vrow = dyn + D * kcap_max;  // D x kcap_max
  unsigned char* visited = reinterpret_cast<unsigned char*>(Vrow + D * kcap_max);
  if (batch < 1) batch = 1;
  if (batch > BMAX) batch = BMAX;

  for (int i = tid; i < m; i += NT) visited[i] = 0;
  if (tid == 0) {
    sh.ipiv = 0;
    sh.K = 0;
    sh.steps = 0;
    sh.state = kRun;
    sh.zero_rows = 0;
    sh.normB2 = 0.0;
    sh.s1max = 0.0;
    sh.npend = 0;
    sh.stop = 0;
  }
  __syncthreads();
  int status = 0;

  for (;;) {
    const int ipiv = sh.ipiv;
    const int K = sh.K;
    if (K + D > kcap) {
      if (sh.npend > 0) {  // the pending steps may already have converged
        resolve_pending<D, NT, BMAX>(Ub, Vb, ldu, ldv, GU, GV, kcap, eps, sh);
        if (sh.stop) {
          status = 1;
          break;
        }
      }
      status = 4;  // capacity overflow -> host reruns with a larger capacity
      break;
    }
    if (tid == 0) visited[ipiv] = 1;
    for (int t = tid; t < D * K; t += NT) {
      const int a = t / K, l = t - a * K;
      Urow[a * kcap_max + l] = Ub[(int64_t)(D * ipiv + a) + (int64_t)l * ldu];
    }
    __syncthreads();

    // ---- row pass -----------------------------------------------------------------
    ArgMax best{-1.0, 0x7fffffff};
    double rs1 = 0.0;
    for (int j = tid; j < n; j += NT) {
      double2 acc[D * D];
#pragma unroll
      for (int t = 0; t < D * D; ++t) acc[t] = cmk(0.0, 0.0);
      const double2* vp = Vb + (int64_t)D * j;
      // 4 factor columns per iteration: 4 D independent loads in flight
      int l = 0;
#pragma unroll 1
      for (; l + 3 < K; l += 4) {
        double2 vv[4][D];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < D; ++c) vv[u][c] = vp[(int64_t)(l + u) * ldv + c];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const double2 ua = Urow[a * kcap_max + l + u];
#pragma unroll
            for (int c = 0; c < D; ++c) acc[a * D + c] = cfma_cj(ua, vv[u][c], acc[a * D + c]);
          }
      }
#pragma unroll 1
      for (; l < K; ++l) {
        double2 vv[D];
#pragma unroll
        for (int c = 0; c < D; ++c) vv[c] = vp[(int64_t)l * ldv + c];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double2 ua = Urow[a * kcap_max + l];
#pragma unroll
          for (int c = 0; c < D; ++c) acc[a * D + c] = cfma_cj(ua, vv[c], acc[a * D + c]);
        }
      }
      // Green's block after the accumulation: fewer values live at once
      double2 R[D * D];
      green_xy_k<KIND>(P, pts, ds.r0 + ipiv, pts, ds.c0 + j, R);
#pragma unroll
      for (int t = 0; t < D * D; ++t) R[t] = csub(R[t], acc[t]);
      // v_k = R_row^H : V(D j + c, K + a) = conj(R[a][c])
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int c = 0; c < D; ++c) Vb[(int64_t)(D * j + c) + (int64_t)(K + a) * ldv] = cconj(R[a * D + c]);
      double s1, s3;
      svals<D>(R, s1, s3);
      rs1 = fmax(rs1, s1);
      best = argmax_pick(best, ArgMax{s3, j});
    }
    best = warp_argmax(best);
    rs1 = warp_max(rs1);
    if (lane == 0) {
      sh.red_v[warp] = best.v;
      sh.red_i[warp] = best.i;
      sh.red_s[warp] = rs1;
    }
    __syncthreads();
    if (tid == 0) {
      ArgMax bb{sh.red_v[0], sh.red_i[0]};
      double r1 = sh.red_s[0];
      for (int w = 1; w < NW; ++w) {
        bb = argmax_pick(bb, ArgMax{sh.red_v[w], sh.red_i[w]});
        r1 = fmax(r1, sh.red_s[w]);
      }
      sh.s1max = fmax(sh.s1max, r1);
      if (r1 <= floor * sh.s1max || sh.s1max == 0.0) {
        sh.rowout = kRowZero;  // zero residual row: lowest unvisited row, no rank added
        int nxt = -1;
        for (int i = 0; i < m; ++i)
          if (!visited[i]) {
            nxt = i;
            break;
          }
        sh.nextrow = nxt;
      } else if (bb.v <= floor * sh.s1max) {
        sh.rowout = kRowFallback;
      } else {
        sh.rowout = kRowPivot;
        sh.jpiv = bb.i;
        double2 Pv[D * D];
        for (int a = 0; a < D; ++a)
          for (int c = 0; c < D; ++c) Pv[a * D + c] = cconj(Vb[(int64_t)(D * bb.i + c) + (int64_t)(K + a) * ldv]);
        inverse<D>(Pv, sh.gamma);
      }
    }
    __syncthreads();
    if (sh.rowout != kRowPivot) {
      if (sh.npend > 0) {  // this step cannot complete: settle the pending ones first
        resolve_pending<D, NT, BMAX>(Ub, Vb, ldu, ldv, GU, GV, kcap, eps, sh);
        if (sh.stop) {
          status = 1;
          break;
        }
      }
      if (sh.rowout == kRowFallback) {
        status = 8;  // fallback needed
        break;
      }
      if (tid == 0) {
        sh.zero_rows++;
        if (sh.nextrow < 0) {
          sh.state = kDone;
          sh.verdict = 1;  // converged flag
        } else {
          sh.ipiv = sh.nextrow;
        }
      }
      __syncthreads();
      if (sh.state == kDone) {
        status = sh.verdict;
        break;
      }
      continue;
    }
    const int jpiv = sh.jpiv;
    for (int t = tid; t < D * K; t += NT) {
      const int c = t / K, l = t - c * K;
      Vrow[c * kcap_max + l] = Vb[(int64_t)(D * jpiv + c) + (int64_t)l * ldv];
    }
    double2 gam[D * D];
#pragma unroll
    for (int t = 0; t < D * D; ++t) gam[t] = sh.gamma[t];
    __syncthreads();

    // ---- column pass ------------------------------------------------------------------
    best = ArgMax{-1.0, 0x7fffffff};
    for (int i = tid; i < m; i += NT) {
      double2 acc[D * D];
#pragma unroll
      for (int t = 0; t < D * D; ++t) acc[t] = cmk(0.0, 0.0);
      const double2* up = Ub + (int64_t)D * i;
      int l = 0;
#pragma unroll 1
      for (; l + 3 < K; l += 4) {
        double2 uu[4][D];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int a = 0; a < D; ++a) uu[u][a] = up[(int64_t)(l + u) * ldu + a];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const double2 vc = Vrow[c * kcap_max + l + u];
#pragma unroll
            for (int a = 0; a < D; ++a) acc[a * D + c] = cfma_cj(uu[u][a], vc, acc[a * D + c]);
          }
      }
#pragma unroll 1
      for (; l < K; ++l) {
        double2 uu[D];
#pragma unroll
        for (int a = 0; a < D; ++a) uu[a] = up[(int64_t)l * ldu + a];
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double2 vc = Vrow[c * kcap_max + l];
#pragma unroll
          for (int a = 0; a < D; ++a) acc[a * D + c] = cfma_cj(uu[a], vc, acc[a * D + c]);
        }
      }
      double2 C[D * D];
      green_xy_k<KIND>(P, pts, ds.r0 + i, pts, ds.c0 + jpiv, C);
#pragma unroll
      for (int t = 0; t < D * D; ++t) C[t] = csub(C[t], acc[t]);
      if (!visited[i]) {
        double s1, s3;
        svals<D>(C, s1, s3);
        best = argmax_pick(best, ArgMax{s3, i});
      }
      // u_k = C gamma
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int c = 0; c < D; ++c) {
          double2 sacc = cmk(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < D; ++q) sacc = cfma(C[a * D + q], gam[q * D + c], sacc);
          Ub[(int64_t)(D * i + a) + (int64_t)(K + c) * ldu] = sacc;
        }
    }
    best = warp_argmax(best);
    if (lane == 0) {
      sh.red_v[warp] = best.v;
      sh.red_i[warp] = best.i;
    }
    __syncthreads();
    if (tid == 0) {
      ArgMax bb{sh.red_v[0], sh.red_i[0]};
      for (int w = 1; w < NW; ++w) bb = argmax_pick(bb, ArgMax{sh.red_v[w], sh.red_i[w]});
      sh.bbv = bb.v;
      sh.bbi = bb.i;
      // this step joins the pending batch
      sh.K = K + D;
      sh.steps += 1;
      sh.npend += 1;
    }
    __syncthreads();
    const int Kn = K + D;
    const bool no_row = sh.bbv < 0.0;  // no unvisited row left
    const bool at_max = Kn >= ds.max_rank;
    if (at_max || no_row || sh.npend >= batch) {
      resolve_pending<D, NT, BMAX>(Ub, Vb, ldu, ldv, GU, GV, kcap, eps, sh);
      if (sh.stop) {
        status = 1;
        break;
      }
      if (at_max) {
        const int dmin = D * (m < n ? m : n);
        status = 2 | (Kn >= dmin ? 1 : 0);
        break;
      }
      if (no_row) {
        status = 1;
        break;
      }
    }
    if (tid == 0) sh.ipiv = sh.bbi;
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    AcaOut o;
    const bool truncated = status == 1 && sh.stop;  // a batched step converged
    o.steps = truncated ? sh.sfinal : sh.steps;
    o.rank = truncated ? sh.kfinal : sh.K;
    o.status = status;
    o.zero_rows = sh.zero_rows;
    out[b] = o;
  }
}

// ===================================================================================
// Tensor-core ACA for large leaves (d = 3): every pass streams its factor panel
// F (rows x K, column-major) ONCE and feeds the same fragments to two FP64 MMA
// contractions (mma.sync m8n8k4 f64, 37 TF/s measured, 256 FMAs / instruction):
//   residual   res(q, a) = sum_l F(q, l)^(*) piv(a, l)   (m = rows, k = columns)
//   Gram       G(l, a')  = sum_q conj F(q, l) F(q, P + a') of the PENDING step's
//              columns P..P+2                        (m = columns, k = rows)
// so the separate Gram pass of aca_kernel (which re-streamed both panels from
// HBM every step) disappears.  The Gram columns of step s are therefore
// produced by step s+1's passes and step s's stop decision is taken then; if it
// says stop, step s+1 is discarded (speculative).  Where step s+1 cannot run the
// pending columns come from the standalone gram_columns first -- the decision
// sequence is exactly the sequential algorithm's (aca_kernel, oracle/lowrank.py).
//
// Complex products as two real MMAs with B = [X_re | X_im] (3 + 3 of 8 columns):
// C1 = F_re B, C2 = F_im B.  Warp w owns row blocks of kTcRows rows (16 points),
// loops over all column octets; Gram partials of its rows go to a per-warp
// scratch slice in global memory (L2) and are summed in fixed warp order.
#ifndef HMX_TC_ROWS
#define HMX_TC_ROWS 48
#endif
constexpr int kTcRows = HMX_TC_ROWS, kTcOct = kTcRows / 8, kTcKs = kTcRows / 4;
#ifndef HMX_TC_WARPS
#define HMX_TC_WARPS 8
#endif
constexpr int kTcWarps = HMX_TC_WARPS, kTcThreads = 32 * kTcWarps;
#ifndef HMX_TC_PF
#define HMX_TC_PF 1
#endif
constexpr int kTcPf = HMX_TC_PF;  // Gram-scratch prefetch distance (octets)
// per-warp cp.async ring: 2 stages of one column octet x kTcRows rows, columns
// padded to kTcCol rows (the Gram fragments read 8 columns x 4 rows: the pad
// spreads the 8 columns over all banks)
constexpr int kTcCol = kTcRows + 4, kTcStage = 8 * kTcCol;  // double2 units; ring = STAGES x kTcStage

// HMX_TC_PROF (experiment builds only): clock64 phase cycles of the
// tensor-core ACA (thread 0 per CTA for the step phases 0-6; lane 0 of every
// warp for 8 = streaming loop, 9 = epilogue), read by hmx_debug_tc_prof.
#ifdef HMX_TC_PROF
__device__ unsigned long long g_tc_prof[16];
__device__ unsigned long long g_tc_cta[4 * 8192];  // per launched CTA: globaltimer start, end, SM id, (m + n) << 32 | K
HMX_D unsigned long long tc_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TC_MARK(i)                                                                   \
  do {                                                                               \
    if (threadIdx.x == 0) {                                                          \
      const long long t_ = clock64();                                                \
      atomicAdd(&g_tc_prof[(i)], (unsigned long long)(t_ - tc_t0));                  \
      tc_t0 = t_;                                                                    \
    }                                                                                \
  } while (0)
#define TC_WMARK(i)                                                                  \
  do {                                                                               \
    if ((threadIdx.x & 31) == 0) {                                                   \
      const long long t_ = clock64();                                                \
      atomicAdd(&g_tc_prof[(i)], (unsigned long long)(t_ - tw_t0));                  \
      tw_t0 = t_;                                                                    \
    }                                                                                \
  } while (0)
#define TC_T0() const long long te0_ = clock64()
#define TC_TADD(i) \
  do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_tc_prof[(i)], (unsigned long long)(clock64() - te0_)); } while (0)
#else
#define TC_T0() \
  do {          \
  } while (0)
#define TC_TADD(i) \
  do {             \
  } while (0)
#define TC_MARK(i) \
  do {             \
  } while (0)
#define TC_WMARK(i) \
  do {              \
  } while (0)
#endif

HMX_D void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Fused pass over panel F (rows = 3 npts, ld = rows, K columns) for the row
// blocks of this warp.  Each column octet of a row block is brought into the
// warp's shared-memory ring by eight bulk copies (one 48-row column run each,
// issued by one elected lane on the stage's mbarrier) kTcStages - 1 octets ahead, then
// feeds both contractions from shared memory.  Residual fragments of each row
// block are left in resb (aliases the ring: kTcRows x 12 doubles, C1 n = 0..5
// then C2 n = 0..5) and `epi(rb_row0)` is called by the whole warp; with pend,
// the Gram partials of the pending columns [Pc, Pc + 3) go to scr (this warp's
// slice: noct x 32 lanes x 4); the pending columns of the row block ride on the
// first octet's mbarrier.  `phase` holds the parity of the next wait on each
// ring stage (bit s), carried across passes.  Rows past the panel's end (last
// row block) are zeroed in shared memory after the copy lands (the bulk copy
// writes only the valid rows, so the two proxies never touch the same bytes).
template <int kTcStages, class Epi>
HMX_D void tc_pass(const double2* __restrict__ F, int64_t rows, int K, const double2* piv, int lds, bool pend,
                   int Pc, double* __restrict__ scr, int noct, double2* ring, double2* nfs, unsigned bar_sa,
                   unsigned& phase, Epi&& epi) {
  // the warp index through a shuffle: the compiler then keeps everything derived from it (row
  // block, copy addresses) in uniform registers
  const int lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int fr = lane >> 2, fk = lane & 3;
  double* resb = reinterpret_cast<double*>(ring);
  constexpr unsigned kStageBytes = sizeof(double2) * kTcStage;
  const unsigned ring_sa = (unsigned)__cvta_generic_to_shared(ring);
  const unsigned nfs_sa = (unsigned)__cvta_generic_to_shared(nfs);
  // B fragment of the residual for column l (pivot row staged with zeros past K)
  const bool bre = fr < 3, bon = fr < 6;
  const int bcol = bre ? fr : (bon ? fr - 3 : 0);  // lanes fr >= 6 read row 0 and use 0
  const double2* pbase = piv + bcol * lds;
  bool first = true;
#ifdef HMX_TC_PROF
  long long tw_t0 = clock64();
#endif
  for (int64_t r0 = (int64_t)warp * kTcRows; r0 < rows; r0 += (int64_t)kTcWarps * kTcRows) {
    const int rlim = rows - r0 < (int64_t)kTcRows ? (int)(rows - r0) : kTcRows;  // valid rows of this block
    const unsigned run = (unsigned)rlim * (unsigned)sizeof(double2);
    const double2* Fr = F + r0;
    auto stage = [&](int co, int buf) {
      const int clim = min(8, K - co * 8);  // columns of this octet inside the panel
      const unsigned mb = bar_sa + 8u * (unsigned)buf;
      const bool with_pend = pend && co == 0;
      // one elected lane issues the octet's copies from warp-uniform operands (uniform datapath:
      // no per-lane address broadcast), the pending columns riding on the first octet's barrier
      if (elect_one()) {
        mbar_expect_tx(mb, run * (unsigned)(clim + (with_pend ? 3 : 0)));
        const double2* src = Fr + (int64_t)(co * 8) * rows;
        unsigned dst = ring_sa + (unsigned)buf * kStageBytes;
        for (int c = 0; c < clim; ++c) {
          bulk_g2s(dst, src, run, mb);
          src += rows;
          dst += (unsigned)kTcCol * (unsigned)sizeof(double2);
        }
        if (with_pend) {
          const double2* ps = Fr + (int64_t)Pc * rows;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            bulk_g2s(nfs_sa + (unsigned)(c * kTcRows) * (unsigned)sizeof(double2), ps + (int64_t)c * rows, run, mb);
        }
      }
    };
    auto wait = [&](int buf) {
      mbar_wait(bar_sa + 8u * (unsigned)buf, (phase >> buf) & 1u);
      phase ^= 1u << buf;
    };
#pragma unroll
    for (int sidx = 0; sidx < kTcStages - 1; ++sidx)
      if (sidx < noct) stage(sidx, sidx);
    double c1[kTcOct][2], c2[kTcOct][2];
#pragma unroll
    for (int o = 0; o < kTcOct; ++o) c1[o][0] = c1[o][1] = c2[o][0] = c2[o][1] = 0.0;
    double bj[kTcKs];  // Gram B fragments: pending column fr mod 3 (re / im) at row 4 j + fk
    // this warp's Gram partials of its earlier row blocks (global scratch, L2):
    // a register queue of kTcPf octets ahead hides the L2 round trip
    double nx[kTcPf][4];
#pragma unroll
    for (int q = 0; q < kTcPf; ++q) {
      nx[q][0] = nx[q][1] = nx[q][2] = nx[q][3] = 0.0;
      if (pend && !first && q < noct) {
        const double2* dq = reinterpret_cast<const double2*>(scr + ((int64_t)q * 32 + lane) * 4);
        const double2 q0 = dq[0], q1 = dq[1];
        nx[q][0] = q0.x;
        nx[q][1] = q0.y;
        nx[q][2] = q1.x;
        nx[q][3] = q1.y;
      }
    }
    for (int co = 0; co < noct; ++co) {
      if (co + kTcStages - 1 < noct) stage(co + kTcStages - 1, (co + kTcStages - 1) % kTcStages);
      double* d = scr + ((int64_t)co * 32 + lane) * 4;
      double g3[2] = {nx[0][0], nx[0][1]}, g4[2] = {nx[0][2], nx[0][3]};
#pragma unroll
      for (int q = 0; q + 1 < kTcPf; ++q)
#pragma unroll
        for (int t = 0; t < 4; ++t) nx[q][t] = nx[q + 1][t];
      if (pend && !first && co + kTcPf < noct) {
        const double2* dn = reinterpret_cast<const double2*>(d + 128 * kTcPf);
        const double2 q0 = dn[0], q1 = dn[1];
        nx[kTcPf - 1][0] = q0.x;
        nx[kTcPf - 1][1] = q0.y;
        nx[kTcPf - 1][2] = q1.x;
        nx[kTcPf - 1][3] = q1.y;
      }
      const int buf = co % kTcStages;
      wait(buf);
      double2* T = ring + buf * kTcStage;  // T[col * kTcCol + row]
      if (rlim < kTcRows) {  // rows past the panel: zeros (bytes the bulk copy did not write)
        for (int e = lane; e < 8 * (kTcRows - rlim); e += 32) {
          const int c = e / (kTcRows - rlim), row = rlim + e % (kTcRows - rlim);
          T[c * kTcCol + row] = cmk(0.0, 0.0);
        }
        if (pend && co == 0)
          for (int e = lane; e < 3 * (kTcRows - rlim); e += 32) {
            const int c = e / (kTcRows - rlim), row = rlim + e % (kTcRows - rlim);
            nfs[c * kTcRows + row] = cmk(0.0, 0.0);
          }
        __syncwarp();
      }
      if (pend && co == 0) {
#pragma unroll
        for (int j = 0; j < kTcKs; ++j) {
          const double2 x = nfs[bcol * kTcRows + 4 * j + fk];
          bj[j] = bon ? (bre ? x.x : x.y) : 0.0;
        }
      }
      const int l0 = co * 8;
      // residual: two k-steps of 4 columns
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double2 pv = pbase[l0 + 4 * h + fk];
        const double b = bon ? (bre ? pv.x : pv.y) : 0.0;
#pragma unroll
        for (int o = 0; o < kTcOct; ++o) {
          const double2 a = T[(4 * h + fk) * kTcCol + 8 * o + fr];
          dmma(c1[o][0], c1[o][1], a.x, b);
          dmma(c2[o][0], c2[o][1], a.y, b);
        }
      }
      if (pend) {
        // A' = F^T: m = column l0 + fr, k = row r0 + 4 j + fk.  One accumulator per product,
        // started from the earlier row blocks' partial: the re / im MMAs alternate, so each
        // chain's next MMA issues two issue slots (32 cycles) after its predecessor, beyond
        // the MMA latency (more chains only cost registers and adds: measured slower)
        double h3[2] = {g3[0], g3[1]}, h4[2] = {g4[0], g4[1]};
#pragma unroll
        for (int j = 0; j < kTcKs; ++j) {
          const double2 a = T[fr * kTcCol + 4 * j + fk];
          dmma(h3[0], h3[1], a.x, bj[j]);
          dmma(h4[0], h4[1], a.y, bj[j]);
        }
        reinterpret_cast<double2*>(d)[0] = cmk(h3[0], h3[1]);
        reinterpret_cast<double2*>(d)[1] = cmk(h4[0], h4[1]);
      }
      // this buffer is refilled by the next iteration's prefetch: every lane's reads of it have
      // been consumed by the MMAs above, and the warp barrier orders them before the elected
      // lane's copy (reads followed by an async-proxy write need no proxy fence)
      __syncwarp();
    }
    // residual fragments -> shared memory (rows of this block; the ring is idle now)
#pragma unroll
    for (int o = 0; o < kTcOct; ++o)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int nn = 2 * fk + i;
        if (nn < 6) {
          resb[(8 * o + fr) * 12 + nn] = c1[o][i];
          resb[(8 * o + fr) * 12 + 6 + nn] = c2[o][i];
        }
      }
    __syncwarp();
    TC_WMARK(8);
    epi(r0);
    // the epilogue's panel-column stores (generic proxy) are read back by later bulk copies;
    // its shared-memory accesses precede the next row block's copies into the ring
    fence_async_global();
    fence_async_smem();
    __syncwarp();
    TC_WMARK(9);
    first = false;
  }
}

// Sum the warp slices (fixed order) into G(:, Pc:Pc+3), rows l < Kend.
HMX_D void tc_gram_finalize(const double* __restrict__ scr, int noct, int nwork, double2* __restrict__ Gm, int kcap,
                            int Pc, int Kend) {
  for (int t = threadIdx.x; t < Kend * 3; t += kTcThreads) {
    const int l = t / 3, a = t - l * 3;
    const int co = l >> 3, r = l & 7;
    // C3[r][n] / C4[r][n] live at lane 4 r + n / 2, element n % 2 (+ 2 for C4)
    auto at = [&](int w, int nn, int e) {
      return scr[(((int64_t)w * noct + co) * 32 + 4 * r + nn / 2) * 4 + e + (nn & 1)];
    };
    double re = 0.0, im = 0.0;
    for (int w = 0; w < nwork; ++w) {
      re += at(w, a, 0) + at(w, 3 + a, 2);
      im += at(w, 3 + a, 0) - at(w, a, 2);
    }
    const double2 v = cmk(re, im);
    const int col = Pc + a;
    if (l < Pc || l < col) {
      Gm[l + (int64_t)col * kcap] = v;
      Gm[col + (int64_t)l * kcap] = cconj(v);
    } else if (l == col) {
      Gm[l + (int64_t)col * kcap] = cmk(v.x, 0.0);
    }
  }
}

#ifndef HMX_TC_MINB
#define HMX_TC_MINB 1
#endif
template <int KIND, int STAGES>
__global__ void __launch_bounds__(kTcThreads, HMX_TC_MINB)
    aca_tc_kernel(GreenParams P, PointsSoA pts, const AcaDesc* __restrict__ desc, const int32_t* __restrict__ order,
                  double eps, double floor, double2* __restrict__ U, double2* __restrict__ V,
                  double2* __restrict__ G, AcaOut* __restrict__ out, int kcap_max) {
  constexpr int D = 3, NT = kTcThreads, NW = kTcWarps;
  extern __shared__ double2 dyn[];
  __shared__ Shared sh;
  __shared__ int s_pend;
  __shared__ __align__(8) unsigned long long tc_bar[kTcWarps][STAGES];  // per-warp ring mbarriers
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = order[blockIdx.x];
  const AcaDesc ds = desc[b];
  const int m = ds.m, n = ds.n, kcap = ds.kcap;
  const int64_t ldu = (int64_t)D * m, ldv = (int64_t)D * n;
  double2* __restrict__ Ub = U + ds.uoff;
  double2* __restrict__ Vb = V + ds.voff;
  double2* __restrict__ GU = G + ds.goff;
  double2* __restrict__ GV = GU + (int64_t)kcap * kcap;
  const int noct_cap = (kcap + 7) / 8;
  double* __restrict__ scr = reinterpret_cast<double*>(GV + (int64_t)kcap * kcap);  // NW x noct_cap x 32 x 4
  double* __restrict__ wscr = scr + (int64_t)warp * noct_cap * 128;
  const int lds = kcap_max + 8;
  double2* Urow = dyn;                 // 3 x lds
  double2* Vrow = dyn + D * lds;       // 3 x lds
  constexpr int kTcRing = STAGES * kTcStage;
  double2* ring = Vrow + D * lds + warp * kTcRing;  // NW x kTcRing (residual buffer aliased)
  double2* nfw = Vrow + D * lds + NW * kTcRing + warp * 3 * kTcRows;  // NW x 3 x kTcRows pending columns
  unsigned char* visited = reinterpret_cast<unsigned char*>(Vrow + D * lds + NW * kTcRing + NW * 3 * kTcRows);
  const int nwork_v = min(NW, (int)((ldv + kTcRows - 1) / kTcRows));
  const int nwork_u = min(NW, (int)((ldu + kTcRows - 1) / kTcRows));

  for (int i = tid; i < m; i += NT) visited[i] = 0;
  // ring stages start zeroed (copies past a short last octet leave earlier, finite data)
  for (int t = lane; t < kTcRing; t += 32) ring[t] = cmk(0.0, 0.0);
  const unsigned bar_sa = (unsigned)__cvta_generic_to_shared(&tc_bar[warp][0]);
  if (lane == 0)
    for (int st = 0; st < STAGES; ++st) mbar_init(bar_sa + 8u * st, 1);
  unsigned phase = 0;
  fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (tid == 0) {
    sh.ipiv = 0;
    sh.K = 0;
    sh.steps = 0;
    sh.state = kRun;
    sh.zero_rows = 0;
    sh.normB2 = 0.0;
    sh.s1max = 0.0;
    sh.stop = 0;
    s_pend = 0;
  }
  __syncthreads();
  int status = 0;
#ifdef HMX_TC_PROF
  long long tc_t0 = clock64();
  if (tid == 0 && blockIdx.x < 8192) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_tc_cta[4 * blockIdx.x] = tc_gtime();
    g_tc_cta[4 * blockIdx.x + 2] = smid;
  }
#endif

  for (;;) {
    const int ipiv = sh.ipiv;
    const int K = sh.K;
    const bool pend = s_pend != 0;
    const int Pc = K - D;
    const int noct = (K + 7) / 8;
    if (K + D > kcap) {
      if (pend) {
        gram_columns<D, NT>(Ub, Vb, ldu, ldv, GU, GV, kcap, Pc);
        __syncthreads();
        decide_step<D, NT>(GU, GV, kcap, Pc, eps, sh);
        if (sh.stop) {
          status = 1;
          break;
        }
      }
      status = 4;
      break;
    }
    if (tid == 0) visited[ipiv] = 1;
    for (int t = tid; t < D * lds; t += NT) {
      const int a = t / lds, l = t - a * lds;
      Urow[t] = l < K ? Ub[(int64_t)(D * ipiv + a) + (int64_t)l * ldu] : cmk(0.0, 0.0);
    }
    __syncthreads();
    TC_MARK(0);

    // ---- row pass over V ----------------------------------------------------------------
    ArgMax best{-1.0, 0x7fffffff};
    double rs1 = 0.0;
    tc_pass<STAGES>(Vb, ldv, K, Urow, lds, pend, Pc, wscr, noct, ring, nfw, bar_sa, phase, [&](int64_t r0) {
      // lanes 0..15: point j = r0 / 3 + lane, rows 3 lane + c of the block
      const int p = lane;
      const int j = (int)(r0 / 3) + p;
      if (p < kTcRows / 3 && j < n) {
        double2 R[9];
        {
          TC_T0();
          green_xy_k<KIND>(P, pts, ds.r0 + ipiv, pts, ds.c0 + j, R);
          TC_TADD(10);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double* rr = reinterpret_cast<const double*>(ring) + (3 * p + c) * 12;  // V row 3 j + c
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            // sum_l Urow(a, l) conj V(q, l): re = C1[a] + C2[3 + a], im = C1[3 + a] - C2[a]
            const double2 acc = cmk(rr[a] + rr[6 + 3 + a], rr[3 + a] - rr[6 + a]);
            R[a * 3 + c] = csub(R[a * 3 + c], acc);
          }
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) Vb[(int64_t)(3 * j + c) + (int64_t)(K + a) * ldv] = cconj(R[a * 3 + c]);
        double s1, s3;
        {
          TC_T0();
          svals3(R, s1, s3);
          TC_TADD(11);
        }
        rs1 = fmax(rs1, s1);
        best = argmax_pick(best, ArgMax{s3, j});
      }
    });
    best = warp_argmax(best);
    rs1 = warp_max(rs1);
    if (lane == 0) {
      sh.red_v[warp] = best.v;
      sh.red_i[warp] = best.i;
      sh.red_s[warp] = rs1;
    }
    __syncthreads();
    TC_MARK(1);
    if (pend) tc_gram_finalize(scr, noct_cap, nwork_v, GV, kcap, Pc, K);
    if (tid == 0) {
      ArgMax bb{sh.red_v[0], sh.red_i[0]};
      double r1 = sh.red_s[0];
      for (int w = 1; w < NW; ++w) {
        bb = argmax_pick(bb, ArgMax{sh.red_v[w], sh.red_i[w]});
        r1 = fmax(r1, sh.red_s[w]);
      }
      sh.s1max = fmax(sh.s1max, r1);
      if (r1 <= floor * sh.s1max || sh.s1max == 0.0) {
        sh.rowout = kRowZero;
        int nxt = -1;
        for (int i = 0; i < m; ++i)
          if (!visited[i]) {
            nxt = i;
            break;
          }
        sh.nextrow = nxt;
      } else if (bb.v <= floor * sh.s1max) {
        sh.rowout = kRowFallback;
      } else {
        sh.rowout = kRowPivot;
        sh.jpiv = bb.i;
        double2 Pv[9];
        for (int a = 0; a < 3; ++a)
          for (int c = 0; c < 3; ++c) Pv[a * 3 + c] = cconj(Vb[(int64_t)(3 * bb.i + c) + (int64_t)(K + a) * ldv]);
        inverse<3>(Pv, sh.gamma);
      }
    }
    __syncthreads();
    if (sh.rowout != kRowPivot) {
      if (pend) {  // settle the pending step from a standalone G_U column first
        gram_columns<D, NT>(Ub, Vb, ldu, ldv, GU, GV, kcap, Pc, 1);
        __syncthreads();
        decide_step<D, NT>(GU, GV, kcap, Pc, eps, sh);
        if (sh.stop) {
          status = 1;
          break;
        }
        if (tid == 0) s_pend = 0;
      }
      if (sh.rowout == kRowFallback) {
        status = 8;
        break;
      }
      if (tid == 0) {
        sh.zero_rows++;
        if (sh.nextrow < 0) {
          sh.state = kDone;
          sh.verdict = 1;
        } else {
          sh.ipiv = sh.nextrow;
        }
      }
      __syncthreads();
      if (sh.state == kDone) {
        status = sh.verdict;
        break;
      }
      continue;
    }
    const int jpiv = sh.jpiv;
    for (int t = tid; t < D * lds; t += NT) {
      const int c = t / lds, l = t - c * lds;
      Vrow[t] = l < K ? Vb[(int64_t)(D * jpiv + c) + (int64_t)l * ldv] : cmk(0.0, 0.0);
    }
    double2 gam[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) gam[t] = sh.gamma[t];
    __syncthreads();
    TC_MARK(2);

    // ---- column pass over U ---------------------------------------------------------------
    best = ArgMax{-1.0, 0x7fffffff};
    tc_pass<STAGES>(Ub, ldu, K, Vrow, lds, pend, Pc, wscr, noct, ring, nfw, bar_sa, phase, [&](int64_t r0) {
      const int p = lane;
      const int i = (int)(r0 / 3) + p;
      if (p < kTcRows / 3 && i < m) {
        double2 C[9];
        green_xy_k<KIND>(P, pts, ds.r0 + i, pts, ds.c0 + jpiv, C);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double* rr = reinterpret_cast<const double*>(ring) + (3 * p + a) * 12;  // U row 3 i + a
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            // sum_l U(q, l) conj Vrow(c, l): re = C1[c] + C2[3 + c], im = C2[c] - C1[3 + c]
            const double2 acc = cmk(rr[c] + rr[6 + 3 + c], rr[6 + c] - rr[3 + c]);
            C[a * 3 + c] = csub(C[a * 3 + c], acc);
          }
        }
        if (!visited[i]) {
          double s1, s3;
          svals3(C, s1, s3);
          best = argmax_pick(best, ArgMax{s3, i});
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double2 sacc = cmk(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 3; ++q) sacc = cfma(C[a * 3 + q], gam[q * 3 + c], sacc);
            Ub[(int64_t)(3 * i + a) + (int64_t)(K + c) * ldu] = sacc;
          }
      }
    });
    best = warp_argmax(best);
    if (lane == 0) {
      sh.red_v[warp] = best.v;
      sh.red_i[warp] = best.i;
    }
    __syncthreads();
    TC_MARK(3);
    if (pend) tc_gram_finalize(scr, noct_cap, nwork_u, GU, kcap, Pc, K);
    if (tid == 0) {
      ArgMax bb{sh.red_v[0], sh.red_i[0]};
      for (int w = 1; w < NW; ++w) bb = argmax_pick(bb, ArgMax{sh.red_v[w], sh.red_i[w]});
      sh.bbv = bb.v;
      sh.bbi = bb.i;
    }
    __syncthreads();
    if (pend) {
      decide_step<D, NT>(GU, GV, kcap, Pc, eps, sh);
      if (sh.stop) {  // the pending step converged: this one is discarded
        status = 1;
        break;
      }
    }
    const int Kn = K + D;
    const bool no_row = sh.bbv < 0.0;
    if (Kn >= ds.max_rank || no_row) {
      gram_columns<D, NT>(Ub, Vb, ldu, ldv, GU, GV, kcap, K);
      __syncthreads();
      decide_step<D, NT>(GU, GV, kcap, K, eps, sh);
      if (tid == 0) {
        sh.K = Kn;
        sh.steps += 1;
      }
      const int dmin = D * (m < n ? m : n);
      status = sh.stop ? 1 : (Kn >= ds.max_rank ? (2 | (Kn >= dmin ? 1 : 0)) : 1);
      break;
    }
    if (tid == 0) {
      sh.K = Kn;
      sh.steps += 1;
      s_pend = 1;
      sh.ipiv = sh.bbi;
    }
    __syncthreads();
    TC_MARK(4);
  }
  __syncthreads();
  TC_MARK(5);
#ifdef HMX_TC_PROF
  if (tid == 0 && blockIdx.x < 8192) {
    g_tc_cta[4 * blockIdx.x + 1] = tc_gtime();
    g_tc_cta[4 * blockIdx.x + 3] = ((unsigned long long)(m + n) << 32) | (unsigned)sh.K;
  }
#endif
  if (tid == 0) {
    AcaOut o;
    o.steps = sh.steps;
    o.rank = sh.K;
    o.status = status;
    o.zero_rows = sh.zero_rows;
    out[b] = o;
  }
}

size_t aca_tc_smem(int kcap_max, int m_max, int stages) {
  return sizeof(double2) * (2 * 3 * (size_t)(kcap_max + 8) + (size_t)kTcWarps * (stages * kTcStage + 3 * kTcRows)) +
         (size_t)((m_max + 15) / 16) * 16;
}

}  // namespace

void warm_aca() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, aca_kernel<1, 0, 512, 1, kGramBatch>);
  cudaFuncGetAttributes(&a, aca_kernel<3, 1, 512, 1, kGramBatch>);
  cudaFuncGetAttributes(&a, aca_kernel<3, 2, 512, 1, kGramBatch>);
  cudaFuncGetAttributes(&a, aca_kernel<1, 0, 128, 4, kGramBatch>);
  cudaFuncGetAttributes(&a, aca_kernel<3, 1, 128, 4, kGramBatch>);
  cudaFuncGetAttributes(&a, aca_kernel<3, 2, 128, 4, kGramBatch>);
  cudaFuncGetAttributes(&a, aca_tc_kernel<1, 3>);
  cudaFuncGetAttributes(&a, aca_tc_kernel<2, 3>);
  cudaFuncGetAttributes(&a, aca_tc_kernel<1, 2>);
  cudaFuncGetAttributes(&a, aca_tc_kernel<2, 2>);
}

int launch_aca(Ctx& c, int d, const GreenParams& P, const PointsSoA& pts, const AcaDesc* d_desc, const int32_t* d_order,
               int64_t nblk, int kcap_max, int m_max, double eps, double sigma3_floor, double2* U, double2* V,
               double2* G, AcaOut* d_out, int variant, int tc_stages) {
  if (nblk == 0) return HMX_OK;
  // variant: kAcaWide (512 threads, one CTA per SM: 2-3 CTAs/SM measured
  // 1.4-1.8x slower), kAcaNarrow (128 threads, 4 CTAs per SM: small leaves
  // are latency bound and use few threads per step).
  const int nt = variant == kAcaNarrow ? 128 : 512;
  const int batch = kGramBatch;
  if (variant == kAcaTensor) {
    // 3-stage ring when it fits in shared memory, else 2 stages, else the CUDA-core kernel
    int smem_max = 0;
    HMX_CUDA_TRY(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
    {
      cudaFuncAttributes fa;  // static shared memory (Shared + mbarriers) shares the opt-in limit
      HMX_CUDA_TRY(cudaFuncGetAttributes(&fa, aca_tc_kernel<1, 3>));
      smem_max -= (int)fa.sharedSizeBytes;
    }
    const int want = tc_stages > 0 ? tc_stages : 3;
    const int stages = want >= 3 && aca_tc_smem(kcap_max, m_max, 3) <= (size_t)smem_max ? 3
                       : aca_tc_smem(kcap_max, m_max, 2) <= (size_t)smem_max ? 2
                                                                               : 0;
    if (stages) {
      const size_t smem_tc = aca_tc_smem(kcap_max, m_max, stages);
      auto go_tc = [&](auto kern) -> int {
        HMX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tc));
        kern<<<(unsigned)nblk, kTcThreads, smem_tc, c.stream>>>(P, pts, d_desc, d_order, eps, sigma3_floor, U, V,
                                                                 G, d_out, kcap_max);
        return HMX_OK;
      };
      const int rc = stages == 3 ? (P.kind == 1 ? go_tc(aca_tc_kernel<1, 3>) : go_tc(aca_tc_kernel<2, 3>))
                                 : (P.kind == 1 ? go_tc(aca_tc_kernel<1, 2>) : go_tc(aca_tc_kernel<2, 2>));
      if (rc) return rc;
      HMX_CUDA_TRY(cudaGetLastError());
      return HMX_OK;
    }
    variant = kAcaWide;
  }
  const size_t smem = sizeof(double2) * 2 * (size_t)d * kcap_max + (size_t)((m_max + 15) / 16) * 16;
  auto go = [&](auto kern) -> int {
    HMX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)nblk, nt, smem, c.stream>>>(P, pts, d_desc, d_order, eps, sigma3_floor, U, V, G, d_out,
                                                 kcap_max, batch);
    return HMX_OK;
  };
  int rc;
  if (variant == kAcaNarrow) {
    rc = P.kind == 0 ? go(aca_kernel<1, 0, 128, 4, kGramBatch>)
                     : (P.kind == 1 ? go(aca_kernel<3, 1, 128, 4, kGramBatch>)
                                    : go(aca_kernel<3, 2, 128, 4, kGramBatch>));
  } else {
    rc = P.kind == 0 ? go(aca_kernel<1, 0, 512, 1, kGramBatch>)
                     : (P.kind == 1 ? go(aca_kernel<3, 1, 512, 1, kGramBatch>)
                                    : go(aca_kernel<3, 2, 512, 1, kGramBatch>));
  }
  if (rc) return rc;
  HMX_CUDA_TRY(cudaGetLastError());
  return HMX_OK;
}

}  // namespace hmx

#ifdef HMX_TC_PROF
extern "C" int hmx_debug_tc_prof(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, hmx::g_tc_prof, sizeof(hmx::g_tc_prof)) != cudaSuccess) return 2;
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(hmx::g_tc_prof, z, sizeof(z));
  return 0;
}
extern "C" int hmx_debug_tc_cta(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, hmx::g_tc_cta, sizeof(hmx::g_tc_cta)) != cudaSuccess ? 2 : 0;
}
#endif
