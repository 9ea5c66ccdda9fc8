// Batched partially pivoted ACA over every admissible leaf at once.
//
// Algorithm: PAPER.md:261-280 (scalar, six steps) and PAPER.md:373-378 /
// SPEC.md:298-306 (vector, rank-d updates with sigma_3 pivoting), with the
// pinned decisions of oracle/lowrank.py (decisions 1-7) -- the CPU oracle and
// this kernel implement the same step sequence, so pivots agree except on
// roundoff-level near-ties (ranks compared +/-1 in tests/test_gpu_parity.py).
//
// Mapping: one CTA (256 threads) per admissible block, blocks taken in LPT
// order (largest first).  Per step:
//   row pass   thread per column point j: Green's d x d block of (i_piv, j)
//              minus U(i_piv,:) V(j,:)^H  -> written conjugated as the new V
//              columns (v_k = R_row^H), sigma_1 / sigma_3 per sub-block,
//              block argmax of sigma_3 (lowest index on ties)
//   pivot      gamma = R(i_piv, j_piv)^{-1}
//   col pass   thread per row point i: (i, j_piv) block minus U(i,:) V(j_piv,:)^H,
//              sigma_3 over unvisited rows -> next row pivot, u_k = R_col gamma
//   Gram pass  warp per 4 factor columns: G_U(:, K:K+d) = U^H u_k and
//              G_V(:, K:K+d) = V^H v_k (these Gram matrices are reused by the
//              recompression, so the exact ||B_k||_F update of SPEC.md:338
//              costs no extra pass over the factors)
//   decision   thread 0: ||B_k||^2 update, stop test ||u|| ||v|| <= eps ||B_k||.
// The residual strips are written straight into the factor storage; U/V are
// column-major with ld = d m / d n, the U(i_piv,:) and V(j_piv,:) rows are
// staged in shared memory.
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "green.cuh"
#include "hmatrix.h"

namespace cg = cooperative_groups;

namespace hmx {

namespace {

constexpr int kGramGroup = 4;

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
    const double nl = lam - f / fp;
    if (!(nl < lam)) break;
    lam = nl;
  }
  s1 = sqrt(fmax(lam, 0.0));
  if (c0 <= 0.0 || c1 <= 0.0) {
    s3 = 0.0;
    return;
  }
  double mu = c0 / c1;
#pragma unroll 1
  for (int it = 0; it < 60; ++it) {
    const double f = ((mu - c2) * mu + c1) * mu - c0;
    const double fp = (3.0 * mu - 2.0 * c2) * mu + c1;
    if (!(fp > 0.0)) break;
    const double nm = mu - f / fp;
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
  int ipiv, jpiv, K, steps, state, zero_rows, verdict;
  double normB2, s1max;
  double2 gamma[9];
  double red_v[kMaxWarps];
  int red_i[kMaxWarps];
  double red_s[kMaxWarps];
  double red_a[kMaxWarps];
};

// What each CTA of a cluster publishes for the cluster-wide reductions
// (read by the other CTAs through distributed shared memory).
struct Pub {
  double row_v, row_s1, col_v, cross;
  int row_i, col_i;
};

// state codes
constexpr int kRun = 0, kZeroRow = 1, kDone = 2;

template <int CS>
HMX_D void cluster_sync() {
  if constexpr (CS > 1) cg::this_cluster().sync();
}

template <int CS, class T>
HMX_D T* peer(T* p, int r) {
  if constexpr (CS > 1) return cg::this_cluster().map_shared_rank(p, r);
  return p;
}

// CS CTAs (a thread-block cluster, distributed shared memory for the
// reductions) cooperate on one admissible leaf; CS = 1 is one CTA per leaf.
// Every CTA keeps an identical copy of the ACA state (all decisions are made
// from the same reduced values in the same order -> deterministic).
// CTA rank cr owns column points [n cr/CS, n (cr+1)/CS) in the row pass and
// row points [m cr/CS, ...) in the column pass; its Gram partial sums run over
// exactly the factor rows it wrote, so no barrier is needed before the Gram pass.
template <int D, int KIND, int NT, int MINB, int CS>
__global__ void __launch_bounds__(NT, MINB) aca_kernel(GreenParams P, PointsSoA pts, const AcaDesc* __restrict__ desc,
                                                       const int32_t* __restrict__ order, double eps, double floor,
                                                       double2* __restrict__ U, double2* __restrict__ V,
                                                       double2* __restrict__ G, AcaOut* __restrict__ out,
                                                       int kcap_max) {
  extern __shared__ double2 dyn[];
  __shared__ Shared sh;
  __shared__ Pub pub;
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int cr = 0;
  if constexpr (CS > 1) cr = (int)cg::this_cluster().block_rank();
  const int b = order[blockIdx.x / CS];
  const AcaDesc ds = desc[b];
  const int m = ds.m, n = ds.n, kcap = ds.kcap;
  const int64_t ldu = (int64_t)D * m, ldv = (int64_t)D * n;
  double2* __restrict__ Ub = U + ds.uoff;
  double2* __restrict__ Vb = V + ds.voff;
  double2* __restrict__ GU = G + ds.goff;
  double2* __restrict__ GV = GU + (int64_t)kcap * kcap;
  const int j0 = (int)((int64_t)n * cr / CS), j1 = (int)((int64_t)n * (cr + 1) / CS);
  const int i0 = (int)((int64_t)m * cr / CS), i1 = (int)((int64_t)m * (cr + 1) / CS);
  double2* Urow = dyn;                 // D x kcap_max
  double2* Vrow = dyn + D * kcap_max;  // D x kcap_max
  double2* pubG = Vrow + D * kcap_max; // (CS > 1) 2 x D x kcap_max partial Gram columns
  unsigned char* visited = reinterpret_cast<unsigned char*>(pubG + (CS > 1 ? 2 * D * kcap_max : 0));

  for (int i = tid; i < m; i += NT) visited[i] = 0;
  if (tid == 0) {
    sh.ipiv = 0;
    sh.K = 0;
    sh.steps = 0;
    sh.state = kRun;
    sh.zero_rows = 0;
    sh.normB2 = 0.0;
    sh.s1max = 0.0;
  }
  __syncthreads();
  int status = 0;

  for (;;) {
    const int ipiv = sh.ipiv;
    const int K = sh.K;
    if (K + D > kcap) {
      status = 4;  // capacity overflow -> host reruns with a larger capacity
      break;
    }
    if (tid == 0) visited[ipiv] = 1;
    for (int t = tid; t < D * K; t += NT) {
      const int a = t / K, l = t - a * K;
      Urow[a * kcap_max + l] = Ub[(int64_t)(D * ipiv + a) + (int64_t)l * ldu];
    }
    __syncthreads();

    // ---- row pass (own column points) -----------------------------------------
    ArgMax best{-1.0, 0x7fffffff};
    double rs1 = 0.0;
    for (int j = j0 + tid; j < j1; j += NT) {
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
      pub.row_v = bb.v;
      pub.row_i = bb.i;
      pub.row_s1 = r1;
    }
    cluster_sync<CS>();  // row-pass results (and the new V columns) visible cluster-wide
    if (tid == 0) {
      ArgMax bb{-1.0, 0x7fffffff};
      double r1 = 0.0;
      for (int r = 0; r < CS; ++r) {
        const Pub* q = peer<CS>(&pub, r);
        bb = argmax_pick(bb, ArgMax{q->row_v, q->row_i});
        r1 = fmax(r1, q->row_s1);
      }
      sh.s1max = fmax(sh.s1max, r1);
      if (r1 <= floor * sh.s1max || sh.s1max == 0.0) {
        // zero residual row: lowest unvisited row, no rank added
        sh.zero_rows++;
        int nxt = -1;
        for (int i = 0; i < m; ++i)
          if (!visited[i]) {
            nxt = i;
            break;
          }
        if (nxt < 0) {
          sh.state = kDone;
          sh.verdict = 1;  // converged flag
        } else {
          sh.state = kZeroRow;
          sh.ipiv = nxt;
        }
      } else if (bb.v <= floor * sh.s1max) {
        sh.state = kDone;
        sh.verdict = 8;  // fallback needed
      } else {
        sh.jpiv = bb.i;
        double2 Pv[D * D];
        for (int a = 0; a < D; ++a)
          for (int c = 0; c < D; ++c) Pv[a * D + c] = cconj(Vb[(int64_t)(D * bb.i + c) + (int64_t)(K + a) * ldv]);
        inverse<D>(Pv, sh.gamma);
        sh.state = kRun;
      }
    }
    __syncthreads();
    if (sh.state == kZeroRow) {
      cluster_sync<CS>();  // everyone has read pub.row_* before it is rewritten
      continue;
    }
    if (sh.state == kDone) {
      status = sh.verdict;
      break;
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

    // ---- column pass (own row points) -------------------------------------------
    best = ArgMax{-1.0, 0x7fffffff};
    for (int i = i0 + tid; i < i1; i += NT) {
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
          double2 s = cmk(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < D; ++q) s = cfma(C[a * D + q], gam[q * D + c], s);
          Ub[(int64_t)(D * i + a) + (int64_t)(K + c) * ldu] = s;
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
      pub.col_v = bb.v;
      pub.col_i = bb.i;
    }

    // ---- Gram pass: G(:, K:K+D) = F^H f_new over this CTA's factor rows -----------
    const int Kn = K + D;
    const int ngroups = (Kn + kGramGroup - 1) / kGramGroup;
    for (int side = 0; side < 2; ++side) {
      const double2* F = side == 0 ? Ub : Vb;
      const int64_t ld = side == 0 ? ldu : ldv;
      const int64_t q0 = (int64_t)D * (side == 0 ? i0 : j0), q1 = (int64_t)D * (side == 0 ? i1 : j1);
      double2* Gm = side == 0 ? GU : GV;
      for (int grp = warp; grp < ngroups; grp += NW) {
        double2 acc[kGramGroup][D];
#pragma unroll
        for (int t = 0; t < kGramGroup; ++t)
#pragma unroll
          for (int c = 0; c < D; ++c) acc[t][c] = cmk(0.0, 0.0);
        const int l0 = grp * kGramGroup;
#pragma unroll 2
        for (int64_t q = q0 + lane; q < q1; q += 32) {
          double2 nf[D];
#pragma unroll
          for (int c = 0; c < D; ++c) nf[c] = F[q + (int64_t)(K + c) * ld];
#pragma unroll
          for (int t = 0; t < kGramGroup; ++t) {
            if (l0 + t < Kn) {
              const double2 fl = F[q + (int64_t)(l0 + t) * ld];
#pragma unroll
              for (int c = 0; c < D; ++c) acc[t][c] = cfma_ca(fl, nf[c], acc[t][c]);
            }
          }
        }
#pragma unroll
        for (int t = 0; t < kGramGroup; ++t)
#pragma unroll
          for (int c = 0; c < D; ++c) acc[t][c] = warp_sum(acc[t][c]);
        if (lane == 0) {
#pragma unroll
          for (int t = 0; t < kGramGroup; ++t) {
            const int l = l0 + t;
            if (l >= Kn) continue;
#pragma unroll
            for (int c = 0; c < D; ++c) {
              if constexpr (CS > 1) {
                pubG[(side * D + c) * kcap_max + l] = acc[t][c];
              } else {
                const int col = K + c;
                if (l < K || l < col) {
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
    if constexpr (CS > 1) {
      // combine the CS partial Gram columns (fixed rank order); CTA cr finalises
      // the entries l = cr, cr + CS, ... and writes them to global G
      cluster_sync<CS>();
      for (int t = tid; t < 2 * D * Kn; t += NT) {
        const int l = t % Kn, sc = t / Kn;  // sc = side * D + c
        if (l % CS != cr) continue;
        double2 v = cmk(0.0, 0.0);
        for (int r = 0; r < CS; ++r) v = cadd(v, peer<CS>(pubG, r)[sc * kcap_max + l]);
        const int side = sc / D, c = sc - side * D, col = K + c;
        double2* Gm = side == 0 ? GU : GV;
        if (l < K || l < col) {
          Gm[l + (int64_t)col * kcap] = v;
          Gm[col + (int64_t)l * kcap] = cconj(v);
        } else if (l == col) {
          Gm[l + (int64_t)col * kcap] = cmk(v.x, 0.0);
        }
      }
    }
    __syncthreads();

    // ---- ||B_k||_F update: cross = Re sum_{l<K,c} G_U(l,K+c) conj(G_V(l,K+c)) ----------
    double cross = 0.0;
    for (int t = tid; t < K * D; t += NT) {
      const int l = t / D, c = t - l * D;
      if (l % CS != cr) continue;  // this CTA's finalised entries
      const double2 gu = GU[l + (int64_t)(K + c) * kcap];
      const double2 gv = GV[l + (int64_t)(K + c) * kcap];
      cross += gu.x * gv.x + gu.y * gv.y;
    }
    cross = warp_sum(cross);
    if (lane == 0) sh.red_a[warp] = cross;
    __syncthreads();
    if (tid == 0) {
      double cr_sum = 0.0;
      for (int w = 0; w < NW; ++w) cr_sum += sh.red_a[w];
      pub.cross = cr_sum;
    }
    cluster_sync<CS>();  // cross partials, column argmax and G entries visible
    if (tid == 0) {
      double crs = 0.0;
      ArgMax bb{-1.0, 0x7fffffff};
      for (int r = 0; r < CS; ++r) {
        const Pub* q = peer<CS>(&pub, r);
        crs += q->cross;
        bb = argmax_pick(bb, ArgMax{q->col_v, q->col_i});
      }
      double diag = 0.0, nu = 0.0, nv = 0.0;
      for (int c = 0; c < D; ++c) {
        nu += GU[(K + c) + (int64_t)(K + c) * kcap].x;
        nv += GV[(K + c) + (int64_t)(K + c) * kcap].x;
        for (int q = 0; q < D; ++q) {
          const double2 a = GU[(K + c) + (int64_t)(K + q) * kcap];
          const double2 bq = GV[(K + q) + (int64_t)(K + c) * kcap];
          diag += a.x * bq.x - a.y * bq.y;
        }
      }
      sh.normB2 = sh.normB2 + 2.0 * crs + diag;
      sh.K = Kn;
      sh.steps += 1;
      const int dmin = D * (m < n ? m : n);
      if (sqrt(nu) * sqrt(nv) <= eps * sqrt(fmax(sh.normB2, 0.0))) {
        sh.state = kDone;
        sh.verdict = 1;
      } else if (Kn >= ds.max_rank) {
        sh.state = kDone;
        sh.verdict = 2 | (Kn >= dmin ? 1 : 0);
      } else if (bb.v < 0.0) {  // no unvisited row left
        sh.state = kDone;
        sh.verdict = 1;
      } else {
        sh.state = kRun;
        sh.ipiv = bb.i;
      }
    }
    __syncthreads();
    cluster_sync<CS>();  // all peers done reading pub before the next step rewrites it
    if (sh.state == kDone) {
      status = sh.verdict;
      break;
    }
  }
  if (tid == 0 && cr == 0) {
    AcaOut o;
    o.steps = sh.steps;
    o.rank = sh.K;
    o.status = status;
    o.zero_rows = sh.zero_rows;
    out[b] = o;
  }
}

}  // namespace

void warm_aca() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, aca_kernel<1, 0, 512, 1, 1>);
  cudaFuncGetAttributes(&a, aca_kernel<3, 1, 512, 1, 1>);
  cudaFuncGetAttributes(&a, aca_kernel<3, 2, 512, 1, 1>);
  cudaFuncGetAttributes(&a, aca_kernel<1, 0, 128, 4, 1>);
  cudaFuncGetAttributes(&a, aca_kernel<3, 1, 128, 4, 1>);
  cudaFuncGetAttributes(&a, aca_kernel<3, 2, 128, 4, 1>);
}

int launch_aca(Ctx& c, int d, const GreenParams& P, const PointsSoA& pts, const AcaDesc* d_desc, const int32_t* d_order,
               int64_t nblk, int kcap_max, int m_max, double eps, double sigma3_floor, double2* U, double2* V,
               double2* G, AcaOut* d_out, int variant) {
  if (nblk == 0) return HMX_OK;
  // variant: kAcaWide (512 threads, one CTA per SM: the factors of large
  // leaves stay hot in L1 / the SM's L2 share; 2-3 CTAs/SM measured 1.4-1.8x
  // slower), kAcaNarrow (128 threads, 4 CTAs per SM: small leaves are latency
  // bound and use few threads per step), >1: cluster of that many CTAs per leaf.
  const int CSv = variant > 1 ? variant : 1;
  const char* e_wnt = std::getenv("HMX_ACA_WIDE_NT");
  const int wide_nt = e_wnt && std::atoi(e_wnt) == 256 ? 256 : 512;
  const int nt = variant == kAcaNarrow ? 128 : (CSv > 1 ? 512 : wide_nt);
  size_t smem = sizeof(double2) * (CSv > 1 ? 4 : 2) * (size_t)d * kcap_max + (size_t)((m_max + 15) / 16) * 16;
  auto go = [&](auto kern) -> int {
    HMX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nblk * CSv));
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CSv;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HMX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, P, pts, d_desc, d_order, eps, sigma3_floor, U, V, G, d_out,
                                    kcap_max));
    return HMX_OK;
  };
  int rc;
  if (CSv == 8) {
    rc = P.kind == 0 ? go(aca_kernel<1, 0, 512, 1, 8>)
                     : (P.kind == 1 ? go(aca_kernel<3, 1, 512, 1, 8>) : go(aca_kernel<3, 2, 512, 1, 8>));
  } else if (CSv == 4) {
    rc = P.kind == 0 ? go(aca_kernel<1, 0, 512, 1, 4>)
                     : (P.kind == 1 ? go(aca_kernel<3, 1, 512, 1, 4>) : go(aca_kernel<3, 2, 512, 1, 4>));
  } else if (variant == kAcaNarrow) {
    rc = P.kind == 0 ? go(aca_kernel<1, 0, 128, 4, 1>)
                     : (P.kind == 1 ? go(aca_kernel<3, 1, 128, 4, 1>) : go(aca_kernel<3, 2, 128, 4, 1>));
  } else if (nt == 256) {
    rc = P.kind == 0 ? go(aca_kernel<1, 0, 256, 2, 1>)
                     : (P.kind == 1 ? go(aca_kernel<3, 1, 256, 2, 1>) : go(aca_kernel<3, 2, 256, 2, 1>));
  } else {
    rc = P.kind == 0 ? go(aca_kernel<1, 0, 512, 1, 1>)
                     : (P.kind == 1 ? go(aca_kernel<3, 1, 512, 1, 1>) : go(aca_kernel<3, 2, 512, 1, 1>));
  }
  if (rc) return rc;
  HMX_CUDA_TRY(cudaGetLastError());
  return HMX_OK;
}

}  // namespace hmx
