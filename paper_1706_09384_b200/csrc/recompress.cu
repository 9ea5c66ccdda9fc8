// Batched recompression of every ACA factor pair (SPEC.md:318-326,
// PAPER.md:431-443): the reference does QR(U), QR(V), SVD(R_U R_V^H),
// truncation, U' = Q_U P S^1/2, V' = Q_V L S^1/2.
//
// B200 formulation (same singular values, same subspaces, no tall QR): the ACA
// kernel already accumulated the Gram matrices G_U = U^H U and G_V = V^H V.
//   R   = chol(G_V)            (diagonally scaled; Q_V = V R^{-1})
//   E   = R G_U R^H = Y^H Y    (Y = U R^H, so U V^H = Y Q_V^H)
//   E   = L S^2 L^H            (Householder tridiagonalisation + implicit QL)
//   r   = truncation rank of s (oracle/lowrank.py decision 8)
//   W_U = R^H L_r S_r^{-1/2},  W_V = R^{-1} L_r S_r^{1/2}
//   U'  = U W_U,  V' = V W_V   (batched tiled complex GEMM, launch_form)
// so U' V'^H = U V^H Q_V L_r L_r^H Q_V^H: the rank-r truncated SVD of the ACA
// product, identical to the reference pipeline up to roundoff.
#include <cstdlib>

#include "hmatrix.h"

#ifndef HMX_RC_NT64_MAX
#define HMX_RC_NT64_MAX 0
#endif
constexpr int kRecompressNt64Max = HMX_RC_NT64_MAX;  // K classes run by 64-thread CTAs
#ifndef HMX_RC_MINB
#define HMX_RC_MINB 8
#endif
namespace hmx {

// HMX_RC_PROF (experiment builds only): per-phase clock64 cycles of thread 0,
// summed over CTAs, per MODE (16 slots each: 0-8 phases, 14 sum K, 15 CTAs);
// read back by hmx_debug_rc_prof.
#ifdef HMX_RC_PROF
__device__ unsigned long long g_rc_prof[3 * 16];
#define RC_MARK(i)                                                  \
  do {                                                              \
    __syncthreads();                                                \
    if (threadIdx.x == 0) {                                         \
      const long long t_ = clock64();                               \
      atomicAdd(&g_rc_prof[MODE * 16 + (i)], (unsigned long long)(t_ - rc_t0)); \
      rc_t0 = t_;                                                   \
    }                                                               \
  } while (0)
#else
#define RC_MARK(i) \
  do {             \
  } while (0)
#endif

namespace {



template <int NT>
HMX_D double block_sum(double v, double* red) {
  constexpr int kWarps = NT / 32;
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kWarps; ++w) t += red[w];
  return t;
}

template <int NT>
HMX_D double2 block_sum2(double2 v, double* red) {
  constexpr int kWarps = NT / 32;
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    red[2 * warp] = v.x;
    red[2 * warp + 1] = v.y;
  }
  __syncthreads();
  double2 t = cmk(0.0, 0.0);
  for (int w = 0; w < kWarps; ++w) t = cadd(t, cmk(red[2 * w], red[2 * w + 1]));
  return t;
}

struct Scalars {
  double2 tau, scale, a2;
  double beta;
  int done, istop, m, fail;
};

// CTA-wide complex GEMM through shared-memory tiles (32 x 32 outputs, k-chunks
// of 16): C (M x N, ldc) = op(A) (M x Kd) * op(B) (Kd x N), column-major, with
// op(A)(i,k) = ACT ? conj(A(k,i)) : A(i,k) and op(B)(k,j) = BCT ? conj(B(j,k)) : B(k,j).
// Each thread owns (32 / (NT/16)) x 2 outputs; tile holds 2 x 16 x 33 complex.
constexpr int kGemmTile = 2 * 16 * 33;
template <int NT, bool ACT, bool BCT>
__device__ void cta_zgemm(int M, int N, int Kd, const double2* A, int lda, const double2* B, int ldb, double2* C,
                          int ldc, double2* tile) {
  constexpr int NG = NT > 512 ? 512 : NT;  // threads that own outputs (all threads load tiles)
  constexpr int BM = 32, BN = 32, BK = 16, RS = NG / 16, RPT = BM / RS;
  double2* As = tile;              // [BK][BM + 1]
  double2* Bs = tile + BK * (BM + 1);  // [BK][BN + 1]
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  for (int i0 = 0; i0 < M; i0 += BM)
    for (int j0 = 0; j0 < N; j0 += BN) {
      double2 acc[RPT][2];
#pragma unroll
      for (int q = 0; q < RPT; ++q) acc[q][0] = acc[q][1] = cmk(0.0, 0.0);
      for (int k0 = 0; k0 < Kd; k0 += BK) {
        for (int t = tid; t < BM * BK; t += NT) {
          int ii, kk;
          if (ACT) {
            kk = t % BK;
            ii = t / BK;
          } else {
            ii = t % BM;
            kk = t / BM;
          }
          const int gi = i0 + ii, gk = k0 + kk;
          double2 v = cmk(0.0, 0.0);
          if (gi < M && gk < Kd) v = ACT ? cconj(A[gk + (int64_t)gi * lda]) : A[gi + (int64_t)gk * lda];
          As[kk * (BM + 1) + ii] = v;
        }
        for (int t = tid; t < BK * BN; t += NT) {
          int kk, jj;
          if (BCT) {
            jj = t % BN;
            kk = t / BN;
          } else {
            kk = t % BK;
            jj = t / BK;
          }
          const int gk = k0 + kk, gj = j0 + jj;
          double2 v = cmk(0.0, 0.0);
          if (gk < Kd && gj < N) v = BCT ? cconj(B[gj + (int64_t)gk * ldb]) : B[gk + (int64_t)gj * ldb];
          Bs[kk * (BN + 1) + jj] = v;
        }
        __syncthreads();
        if (tid < NG) {
#pragma unroll 4
          for (int kk = 0; kk < BK; ++kk) {
            const double2 b0 = Bs[kk * (BN + 1) + tx], b1 = Bs[kk * (BN + 1) + tx + 16];
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
              const double2 a = As[kk * (BM + 1) + ty + q * RS];
              acc[q][0] = cfma(a, b0, acc[q][0]);
              acc[q][1] = cfma(a, b1, acc[q][1]);
            }
          }
        }
        __syncthreads();
      }
      if (tid < NG) {
#pragma unroll
        for (int q = 0; q < RPT; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gi = i0 + ty + q * RS, gj = j0 + tx + 16 * h;
            if (gi < M && gj < N) C[gi + (int64_t)gj * ldc] = acc[q][h];
          }
      }
    }
  __syncthreads();
}

// The same product on the FP64 tensor cores for 512-thread CTAs (the large-K class): 16 warps,
// 64 x 64 complex output tiles, k chunks of 16 staged (conjugated / transposed as op() asks) in
// shared memory; each warp owns 32 rows x 8 complex columns as two real mma.sync m8n8k4 f64 per
// 8 x 4 block with B = [op(B)_re | op(B)_im] (the fragment layout of form_gemm below).
constexpr int kGemmTileTc = 2 * 16 * 66;
HMX_D void dmma_acc(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
template <bool ACT, bool BCT>
__device__ void cta_zgemm_tc(int M, int N, int Kd, const double2* A, int lda, const double2* B, int ldb, double2* C,
                             int ldc, double2* tile) {
  constexpr int NT = 512, BM = 64, BN = 64, BK = 16, LDS = BM + 2;
  double2* As = tile;             // [BK][LDS]: op(A)(i0 + ii, k0 + kk) at kk * LDS + ii
  double2* Bs = tile + BK * LDS;  // [BK][LDS]: op(B)(k0 + kk, j0 + jj) at kk * LDS + jj
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;  // warp tile: rows wm*32 + [0,32), cols wn*8 + [0,8)
  const int fr = lane >> 2, fk = lane & 3, t4 = lane & 3;
  for (int i0 = 0; i0 < M; i0 += BM)
    for (int j0 = 0; j0 < N; j0 += BN) {
      double c1[4][2][2], c2[4][2][2];
#pragma unroll
      for (int o = 0; o < 4; ++o)
#pragma unroll
        for (int g = 0; g < 2; ++g) c1[o][g][0] = c1[o][g][1] = c2[o][g][0] = c2[o][g][1] = 0.0;
      for (int k0 = 0; k0 < Kd; k0 += BK) {
        for (int t = tid; t < BM * BK; t += NT) {
          int ii, kk;
          if (ACT) {
            kk = t % BK;
            ii = t / BK;
          } else {
            ii = t % BM;
            kk = t / BM;
          }
          const int gi = i0 + ii, gk = k0 + kk;
          double2 v = cmk(0.0, 0.0);
          if (gi < M && gk < Kd) v = ACT ? cconj(A[gk + (int64_t)gi * lda]) : A[gi + (int64_t)gk * lda];
          As[kk * LDS + ii] = v;
        }
        for (int t = tid; t < BK * BN; t += NT) {
          int kk, jj;
          if (BCT) {
            jj = t % BN;
            kk = t / BN;
          } else {
            kk = t % BK;
            jj = t / BK;
          }
          const int gk = k0 + kk, gj = j0 + jj;
          double2 v = cmk(0.0, 0.0);
          if (gk < Kd && gj < N) v = BCT ? cconj(B[gj + (int64_t)gk * ldb]) : B[gk + (int64_t)gj * ldb];
          Bs[kk * LDS + jj] = v;
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < BK; ks += 4) {
          double2 av[4];
#pragma unroll
          for (int o = 0; o < 4; ++o) av[o] = As[(ks + fk) * LDS + wm * 32 + o * 8 + fr];
          double bv[2];
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            const double2 w = Bs[(ks + fk) * LDS + wn * 8 + g * 4 + (fr & 3)];
            bv[g] = fr < 4 ? w.x : w.y;
          }
#pragma unroll
          for (int o = 0; o < 4; ++o)
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              dmma_acc(c1[o][g][0], c1[o][g][1], av[o].x, bv[g]);
              dmma_acc(c2[o][g][0], c2[o][g][1], av[o].y, bv[g]);
            }
        }
        __syncthreads();
      }
#pragma unroll
      for (int o = 0; o < 4; ++o)
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const double p1 = __shfl_xor_sync(0xffffffffu, c1[o][g][i], 2);
            const double p2 = __shfl_xor_sync(0xffffffffu, c2[o][g][i], 2);
            if (t4 < 2) {
              const int gr = i0 + wm * 32 + o * 8 + fr, gc = j0 + wn * 8 + g * 4 + 2 * t4 + i;
              if (gr < M && gc < N) C[gr + (int64_t)gc * ldc] = cmk(c1[o][g][i] - p2, p1 + c2[o][g][i]);
            }
          }
    }
  __syncthreads();
}

// Householder reduction of the Hermitian E (K x K, ld K, full storage) to a
// real symmetric tridiagonal (d, e): E = Q T Q^H, Q = H_0 ... H_{K-2},
// H_k = I - tau_k v_k v_k^H (LAPACK zhetd2 / zlarfg conventions, beta real).
// v_k is left in E(k+1:, k) with v_k[0] = 1.
template <int NT>
__device__ void tridiagonalize(double2* E, int K, double* d, double* e, double2* tau, double2* vbuf, double2* pbuf,
                               Scalars& S, double* red) {
  const int tid = threadIdx.x;
  const int ld = K;
  for (int k = 0; k + 1 < K; ++k) {
    const int n = K - k - 1;
    double2* col = E + (k + 1) + (int64_t)k * ld;  // x, length n
    double xn2 = 0.0;
    for (int i = 1 + tid; i < n; i += NT) xn2 += cabs2(col[i]);
    xn2 = block_sum<NT>(xn2, red);
    if (tid == 0) {
      const double2 alpha = col[0];
      d[k] = E[k + (int64_t)k * ld].x;
      if (xn2 == 0.0 && alpha.y == 0.0) {
        S.tau = cmk(0.0, 0.0);
        S.beta = alpha.x;
      } else {
        const double nrm = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xn2);
        const double beta = alpha.x >= 0.0 ? -nrm : nrm;
        S.beta = beta;
        S.tau = cmk((beta - alpha.x) / beta, -alpha.y / beta);
        S.scale = cdiv(cmk(1.0, 0.0), csub(alpha, cmk(beta, 0.0)));
      }
      e[k] = S.beta;
      tau[k] = S.tau;
    }
    __syncthreads();
    const double2 tk = S.tau;
    if (tk.x == 0.0 && tk.y == 0.0) continue;
    const double2 sc = S.scale;
    for (int i = tid; i < n; i += NT) {
      const double2 vi = i == 0 ? cmk(1.0, 0.0) : cmul(col[i], sc);
      vbuf[i] = vi;
      col[i] = vi;
    }
    __syncthreads();
    // p = tau A' v, A' = E(k+1:, k+1:)
    const double2* Ap = E + (k + 1) + (int64_t)(k + 1) * ld;
    for (int i = tid; i < n; i += NT) {
      double2 s0 = cmk(0.0, 0.0), s1 = cmk(0.0, 0.0);
      int j = 0;
      for (; j + 1 < n; j += 2) {
        s0 = cfma(Ap[i + (int64_t)j * ld], vbuf[j], s0);
        s1 = cfma(Ap[i + (int64_t)(j + 1) * ld], vbuf[j + 1], s1);
      }
      if (j < n) s0 = cfma(Ap[i + (int64_t)j * ld], vbuf[j], s0);
      pbuf[i] = cmul(tk, cadd(s0, s1));
    }
    __syncthreads();
    double2 dot = cmk(0.0, 0.0);
    for (int i = tid; i < n; i += NT) dot = cfma_ca(pbuf[i], vbuf[i], dot);  // sum conj(p) v
    dot = block_sum2<NT>(dot, red);
    const double2 a2 = cscale(cmul(tk, dot), -0.5);
    for (int i = tid; i < n; i += NT) pbuf[i] = cadd(pbuf[i], cmul(a2, vbuf[i]));  // w
    __syncthreads();
    double2* Aw = E + (k + 1) + (int64_t)(k + 1) * ld;
    for (int t = tid; t < n * n; t += NT) {
      const int i = t % n, j = t / n;
      double2 a = Aw[i + (int64_t)j * ld];
      a = csub(a, cmul(vbuf[i], cconj(pbuf[j])));
      a = csub(a, cmul(pbuf[i], cconj(vbuf[j])));
      Aw[i + (int64_t)j * ld] = a;
    }
    __syncthreads();
  }
  if (tid == 0) {
    d[K - 1] = E[(K - 1) + (int64_t)(K - 1) * ld].x;
    e[K - 1] = 0.0;
  }
  __syncthreads();
}

// Packed lower-triangular Hermitian storage (column-major): element (i, j),
// i >= j, at pk_col(j, K) + (i - j).  Halves the shared memory of E, so twice
// as many leaves are resident per SM in the latency-bound small-K classes.
HMX_HD int pk_col(int j, int K) { return j * (2 * K - j + 1) / 2; }

// Same reduction as tridiagonalize, on packed lower storage; the Householder
// vectors end up in the strictly lower part of the packed columns.
template <int NT>
__device__ void tridiagonalize_packed(double2* E, int K, double* d, double* e, double2* tau, double2* vbuf,
                                      double2* pbuf, Scalars& S, double* red) {
  const int tid = threadIdx.x;
  for (int k = 0; k + 1 < K; ++k) {
    const int n = K - k - 1;
    double2* col = E + pk_col(k, K) + 1;  // x, length n
    double xn2 = 0.0;
    for (int i = 1 + tid; i < n; i += NT) xn2 += cabs2(col[i]);
    xn2 = block_sum<NT>(xn2, red);
    if (tid == 0) {
      const double2 alpha = col[0];
      d[k] = E[pk_col(k, K)].x;
      if (xn2 == 0.0 && alpha.y == 0.0) {
        S.tau = cmk(0.0, 0.0);
        S.beta = alpha.x;
      } else {
        const double nrm = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xn2);
        const double beta = alpha.x >= 0.0 ? -nrm : nrm;
        S.beta = beta;
        S.tau = cmk((beta - alpha.x) / beta, -alpha.y / beta);
        S.scale = cdiv(cmk(1.0, 0.0), csub(alpha, cmk(beta, 0.0)));
      }
      e[k] = S.beta;
      tau[k] = S.tau;
    }
    __syncthreads();
    const double2 tk = S.tau;
    if (tk.x == 0.0 && tk.y == 0.0) continue;
    const double2 sc = S.scale;
    for (int i = tid; i < n; i += NT) {
      const double2 vi = i == 0 ? cmk(1.0, 0.0) : cmul(col[i], sc);
      vbuf[i] = vi;
      col[i] = vi;
    }
    __syncthreads();
    // p = tau A' v, A' = E(k+1:, k+1:): row i of the Hermitian trailing block is
    // column gi below the diagonal and the conjugated row gi left of it
    const int g0 = k + 1;
    for (int i = tid; i < n; i += NT) {
      const int gi = g0 + i;
      double2 s0 = cmk(0.0, 0.0), s1 = cmk(0.0, 0.0);
      for (int j = 0; j < i; ++j) s0 = cfma(E[pk_col(g0 + j, K) + (i - j)], vbuf[j], s0);
      const double2* ci = E + pk_col(gi, K);  // column gi, rows gi..K-1
      for (int j = i; j < n; ++j) s1 = cfma_cj(vbuf[j], ci[j - i], s1);  // conj(A(j, i)) v_j
      // diagonal term: A(i, i) real; cfma_cj used conj(A(i, i)) = A(i, i)
      pbuf[i] = cmul(tk, cadd(s0, s1));
    }
    __syncthreads();
    double2 dot = cmk(0.0, 0.0);
    for (int i = tid; i < n; i += NT) dot = cfma_ca(pbuf[i], vbuf[i], dot);  // sum conj(p) v
    dot = block_sum2<NT>(dot, red);
    const double2 a2 = cscale(cmul(tk, dot), -0.5);
    for (int i = tid; i < n; i += NT) pbuf[i] = cadd(pbuf[i], cmul(a2, vbuf[i]));  // w
    __syncthreads();
    for (int t = tid; t < n * n; t += NT) {
      const int i = t % n, j = t / n;
      if (i < j) continue;
      double2* ap = E + pk_col(g0 + j, K) + (i - j);
      double2 a = *ap;
      a = csub(a, cmul(vbuf[i], cconj(pbuf[j])));
      a = csub(a, cmul(pbuf[i], cconj(vbuf[j])));
      *ap = a;
    }
    __syncthreads();
  }
  if (tid == 0) {
    d[K - 1] = E[pk_col(K - 1, K)].x;
    e[K - 1] = 0.0;
  }
  __syncthreads();
}

// Implicit QL with Wilkinson-type shift on the real symmetric tridiagonal
// (d, e); eigenvectors accumulated in Z (row-major, ld ldz, identity on
// entry).  The rotation chain of one QL iteration is generated by thread 0
// (a scalar recurrence) and applied by all threads, one Z row each.
template <int NT>
__device__ void tridiag_ql(double* d, double* e, double* Z, int ldz, int K, double* rc, double* rs, Scalars& S) {
  const int tid = threadIdx.x;
  for (int t = tid; t < K * K; t += NT) {
    const int r = t / K, c = t % K;
    Z[(int64_t)r * ldz + c] = r == c ? 1.0 : 0.0;
  }
  if (tid == 0) S.fail = 0;
  __syncthreads();
  for (int l = 0; l < K; ++l) {
    int iter = 0;
    for (;;) {
      if (tid == 0) {
        int m;
        for (m = l; m < K - 1; ++m) {
          const double dd = fabs(d[m]) + fabs(d[m + 1]);
          if (fabs(e[m]) + dd == dd) break;
        }
        S.m = m;
        if (m == l) {
          S.done = 1;
        } else if (iter++ >= 60) {
          S.done = 1;
          S.fail = 1;
        } else {
          S.done = 0;
          double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
          double r = hypot(g, 1.0);
          g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? fabs(r) : -fabs(r)));
          double s = 1.0, c = 1.0, p = 0.0;
          int i;
          bool under = false;
          // the chain only reads entries it has not written yet: d[i], e[i]
          // for the next rotation are fetched one step ahead, off the chain
          double ei = e[m - 1], di = d[m - 1], dip1 = d[m];
          for (i = m - 1; i >= l; --i) {
            const double e_nx = i > l ? e[i - 1] : 0.0;
            const double d_nx = i > l ? d[i - 1] : 0.0;
            const double f = s * ei, b = c * ei;
            const double r2 = fma(f, f, g * g);
            if (r2 == 0.0) {
              e[i + 1] = 0.0;
              d[i + 1] = dip1 - p;
              e[m] = 0.0;
              under = true;
              break;
            }
            // one rsqrt instead of hypot + two divisions on the serial chain
            const double rinv = rsqrt(r2);
            r = r2 * rinv;
            e[i + 1] = r;
            s = f * rinv;
            c = g * rinv;
            g = dip1 - p;
            r = (di - g) * s + 2.0 * c * b;
            p = s * r;
            d[i + 1] = g + p;
            g = c * r - b;
            rc[i] = c;
            rs[i] = s;
            dip1 = di;
            di = d_nx;
            ei = e_nx;
          }
          S.istop = under ? i : l - 1;
          if (!under) {
            d[l] -= p;
            e[l] = g;
            e[m] = 0.0;
          }
        }
      }
      __syncthreads();
      const int done = S.done, m = S.m, lo = S.istop + 1;
      __syncthreads();  // everyone has read S before thread 0 rewrites it
      if (done) break;
      for (int row = tid; row < K; row += NT) {
        double* z = Z + (int64_t)row * ldz;
        double zi1 = z[m];
        for (int i = m - 1; i >= lo; --i) {
          const double zi = z[i];
          const double c = rc[i], s = rs[i];
          z[i + 1] = s * zi + c * zi1;
          zi1 = c * zi - s * zi1;
        }
        z[lo] = zi1;
      }
      __syncthreads();
    }
  }
}

// ---- fast tridiagonal eigen-solver: bisection + twisted factorisations ----------
// All K eigenvalues of the real symmetric tridiagonal (d, e) by bisection on
// Sturm counts (thread t finds the t-th smallest; parallel, no serial chain);
// eigenvectors of the r kept eigenvalues from the twisted LDL^T / UDU^T
// factorisation of T - lambda I (one thread per vector, Dhillon's getvec
// without the RRR machinery), orthonormalised by classical Gram-Schmidt twice
// in descending-eigenvalue order.  A vector that is mostly in the span of the
// previous ones (near-degenerate cluster) makes the caller fall back to QL.
// three shifts at once (independent recurrences interleave in the pipeline)
// Reciprocal from the MUFU approximation (rcp.approx.ftz.f64, ~23 bits) refined by NR Newton steps
// (each squares the relative error: 2 steps ~2^-46, 3 steps full precision): the Sturm and twisted
// recurrences are chains of divisions, and a full IEEE division is a longer dependent sequence.
template <int NR>
HMX_D double rcp_nr(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
#pragma unroll
  for (int k = 0; k < NR; ++k) r = fma(r, fma(-q, r, 1.0), r);
  return r;
}

HMX_D void sturm_count3(const double* d, const double* e2, int K, double x1, double x2, double x3, double pivmin,
                        int& c1, int& c2, int& c3) {
  double q1 = d[0] - x1, q2 = d[0] - x2, q3 = d[0] - x3;
  if (fabs(q1) < pivmin) q1 = -pivmin;
  if (fabs(q2) < pivmin) q2 = -pivmin;
  if (fabs(q3) < pivmin) q3 = -pivmin;
  int n1 = q1 < 0.0, n2 = q2 < 0.0, n3 = q3 < 0.0;
  for (int i = 1; i < K; ++i) {
    const double di = d[i], ei = e2[i - 1];
    // a Sturm count is backward stable: the ~2^-46 reciprocal perturbs T by far less than dstebz's
    // absolute tolerance (ulp ||T||) the bisection stops at
    q1 = (di - x1) - ei * rcp_nr<2>(q1);
    q2 = (di - x2) - ei * rcp_nr<2>(q2);
    q3 = (di - x3) - ei * rcp_nr<2>(q3);
    if (fabs(q1) < pivmin) q1 = -pivmin;
    if (fabs(q2) < pivmin) q2 = -pivmin;
    if (fabs(q3) < pivmin) q3 = -pivmin;
    n1 += q1 < 0.0;
    n2 += q2 < 0.0;
    n3 += q3 < 0.0;
  }
  c1 = n1;
  c2 = n2;
  c3 = n3;
}

// lam_asc[j] = j-th smallest eigenvalue
template <int NT>
__device__ void bisect_all(const double* d, const double* e, double* e2, int K, double* lam_asc, double* red,
                           double& pivmin_out) {
  const int tid = threadIdx.x;
  double lo = INFINITY, hi = -INFINITY, emax2 = 0.0;
  for (int i = tid; i < K; i += NT) {
    const double ei = i + 1 < K ? fabs(e[i]) : 0.0, em = i > 0 ? fabs(e[i - 1]) : 0.0;
    lo = fmin(lo, d[i] - ei - em);
    hi = fmax(hi, d[i] + ei + em);
    if (i + 1 < K) {
      e2[i] = e[i] * e[i];
      emax2 = fmax(emax2, e2[i]);
    }
  }
  // block min / max via shared memory
  __shared__ double s_lo[NT / 32], s_hi[NT / 32], s_e2[NT / 32];
  {
    double a = lo, b = hi, c = emax2;
    for (int o = 16; o > 0; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
      c = fmax(c, __shfl_xor_sync(0xffffffffu, c, o));
    }
    if ((tid & 31) == 0) {
      s_lo[tid >> 5] = a;
      s_hi[tid >> 5] = b;
      s_e2[tid >> 5] = c;
    }
    __syncthreads();
    a = s_lo[0];
    b = s_hi[0];
    c = s_e2[0];
    for (int w = 1; w < NT / 32; ++w) {
      a = fmin(a, s_lo[w]);
      b = fmax(b, s_hi[w]);
      c = fmax(c, s_e2[w]);
    }
    lo = a;
    hi = b;
    emax2 = c;
  }
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax2) * 4.0;
  pivmin_out = pivmin;
  const double span = fmax(fabs(lo), fabs(hi));
  lo -= 2.2e-16 * span * K + pivmin;
  hi += 2.2e-16 * span * K + pivmin;
  // stop at max(2 ulp ||T||, 2 ulp |lambda|) + pivmin: LAPACK dstebz's default
  // absolute tolerance (abstol = ulp ||T||), so eigenvalues far below ||T||
  // (all truncated away) do not iterate down to their own relative precision
  const double atol = 4.4e-16 * span + pivmin;
  // multisection: 3 independent Sturm chains per thread (ILP); with K <= NT / 2
  // (NT / 4) a group of T = 2 (4) adjacent lanes shares one eigenvalue and
  // tests 3 T points per step -> log2(3 T + 1) bits per step instead of 2
  const int T = 4 * K <= NT ? 4 : (2 * K <= NT ? 2 : 1);
  if (T > 1) {
    const int j = tid / T, sub = tid % T, P = 3 * T;
    const int lane = tid & 31;
    const unsigned gmask = ((1u << T) - 1u) << (lane & ~(T - 1));
    if (j < K) {
      double a = lo, b = hi;
      for (int it = 0; it < 40; ++it) {
        if (b - a <= fmax(atol, 4.4e-16 * fmax(fabs(a), fabs(b)))) break;
        const double h = (b - a) / (double)(P + 1);
        const int p0 = 3 * sub;
        const double x1 = a + (double)(p0 + 1) * h, x2 = a + (double)(p0 + 2) * h, x3 = a + (double)(p0 + 3) * h;
        int c1, c2, c3;
        sturm_count3(d, e2, K, x1, x2, x3, pivmin, c1, c2, c3);
        int first = c1 > j ? p0 : (c2 > j ? p0 + 1 : (c3 > j ? p0 + 2 : P));
        for (int o = 1; o < T; o <<= 1) first = min(first, __shfl_xor_sync(gmask, first, o));
        const double na = first == 0 ? a : a + (double)first * h;
        const double nb = first == P ? b : a + (double)(first + 1) * h;
        a = na;
        b = nb;
      }
      if (sub == 0) lam_asc[j] = 0.5 * (a + b);
    }
    __syncthreads();
    return;
  }
  for (int j = tid; j < K; j += NT) {
    double a = lo, b = hi;
    for (int it = 0; it < 40; ++it) {
      if (b - a <= fmax(atol, 4.4e-16 * fmax(fabs(a), fabs(b)))) break;
      const double h = 0.25 * (b - a);
      const double x1 = a + h, x2 = a + 2.0 * h, x3 = b - h;
      int c1, c2, c3;
      sturm_count3(d, e2, K, x1, x2, x3, pivmin, c1, c2, c3);
      if (c1 > j) {
        b = x1;
      } else if (c2 > j) {
        a = x1;
        b = x2;
      } else if (c3 > j) {
        a = x2;
        b = x3;
      } else {
        a = x3;
      }
    }
    lam_asc[j] = 0.5 * (a + b);
  }
  __syncthreads();
}

// eigenvector of T for eigenvalue lam into Z column (real parts of zc[0..K)),
// scratch: K doubles (U multipliers)
HMX_D void twisted_vector(const double* d, const double* e, int K, double lam, double pivmin, double2* zc,
                          double* scratch) {
  // forward D+ / L, stored as (L_i, D+_i) in zc
  double dp = d[0] - lam;
  for (int i = 0; i + 1 < K; ++i) {
    if (fabs(dp) < pivmin) dp = dp < 0.0 ? -pivmin : pivmin;
    const double L = e[i] * rcp_nr<3>(dp);
    zc[i] = cmk(L, dp);
    dp = (d[i + 1] - lam) - L * e[i];
  }
  if (fabs(dp) < pivmin) dp = dp < 0.0 ? -pivmin : pivmin;
  zc[K - 1] = cmk(0.0, dp);
  // backward D- / U, twist index k = argmin |gamma_k|
  double dm = d[K - 1] - lam;
  double best = fabs(zc[K - 1].y);
  int k = K - 1;
  for (int i = K - 1; i >= 1; --i) {
    if (fabs(dm) < pivmin) dm = dm < 0.0 ? -pivmin : pivmin;
    const double U = e[i - 1] * rcp_nr<3>(dm);
    scratch[i] = U;
    dm = (d[i - 1] - lam) - U * e[i - 1];
    const double g = fabs(zc[i - 1].y + dm - (d[i - 1] - lam));
    if (g < best) {
      best = g;
      k = i - 1;
    }
  }
  // z_k = 1, z_i = -L_i z_{i+1} (i < k), z_i = -U_i z_{i-1} (i > k)
  double z = 1.0, nrm = 1.0;
  for (int i = k - 1; i >= 0; --i) {
    z = -zc[i].x * z;
    zc[i] = cmk(z, 0.0);
    nrm = fma(z, z, nrm);
  }
  zc[k] = cmk(1.0, 0.0);
  z = 1.0;
  for (int i = k + 1; i < K; ++i) {
    z = -scratch[i] * z;
    zc[i] = cmk(z, 0.0);
    nrm = fma(z, z, nrm);
  }
  const double inv = rsqrt(nrm);
  for (int i = 0; i < K; ++i) zc[i].x *= inv;
}

// classical Gram-Schmidt twice on the real parts of the r columns of Zr (ld K);
// returns false if a column is (numerically) in the span of its predecessors
template <int NT>
__device__ bool cgs2_columns(double2* Zr, int K, int r, double* h, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int s_bad;
  if (tid == 0) s_bad = 0;
  for (int c = 0; c < r; ++c) {
    double2* zc = Zr + (int64_t)c * K;
    for (int pass = 0; pass < 2; ++pass) {
      for (int j = warp; j < c; j += NT / 32) {
        const double2* zj = Zr + (int64_t)j * K;
        double acc = 0.0;
        for (int i = lane; i < K; i += 32) acc = fma(zj[i].x, zc[i].x, acc);
        acc = warp_sum(acc);
        if (lane == 0) h[j] = acc;
      }
      __syncthreads();
      double nrm = 0.0;
      for (int i = tid; i < K; i += NT) {
        double v = zc[i].x;
        for (int j = 0; j < c; ++j) v = fma(-h[j], Zr[i + (int64_t)j * K].x, v);
        zc[i].x = v;
        nrm = fma(v, v, nrm);
      }
      nrm = block_sum<NT>(nrm, red);
      if (pass == 0 && tid == 0 && !(nrm > 0.25)) s_bad = 1;  // lost > 87% to earlier vectors
      const double inv = nrm > 0.0 ? rsqrt(nrm) : 0.0;
      for (int i = tid; i < K; i += NT) zc[i].x *= inv;
      __syncthreads();
    }
  }
  return s_bad == 0;
}

// L_r = Q Z_r with Q = H_0 H_1 ... H_{K-2} (H_k = I - tau_k v_k v_k^H, v_k zero above row k + 1 and
// 1 there) applied to B (K x r) in blocks of NB reflectors as the compact WY form (LAPACK zlarft,
// forward / columnwise): Q_blk = I - V T V^H, B <- B - V (T (V^H B)), last block first.  A handful
// of barriers per block instead of two per reflector.  scr: 2 NB r + NB^2 complex (L2).
template <int NT, int NB>
__device__ void backxf_blocked(const double2* E, const double2* Hv, bool hv_packed, const double2* tau, int K, int r,
                               double2* B, double2* scr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2* Wm = scr;           // NB x r: V^H B
  double2* W2 = scr + NB * r;  // NB x r: T V^H B
  double2* S = W2 + NB * r;    // NB x NB: V^H V, overwritten by the strictly upper T
  auto vget = [&](int i, int k) -> double2 {  // v_k at global row i
    if (i <= k) return cmk(0.0, 0.0);
    if (i == k + 1) return cmk(1.0, 0.0);
    return hv_packed ? E[pk_col(k, K) + (i - k)] : Hv[i + (int64_t)k * K];
  };
  const int nref = K - 1;
  for (int k0 = ((nref - 1) / NB) * NB; k0 >= 0; k0 -= NB) {
    const int nb = min(NB, nref - k0);
    for (int t = tid; t < nb * nb + nb * r; t += NT) {
      if (t < nb * nb) {  // S(q, i) = v_q^H v_i, q < i
        const int q = t % nb, i = t / nb;
        if (q >= i) continue;
        double2 acc = cmk(0.0, 0.0);
        for (int row = k0 + i + 1; row < K; ++row) acc = cfma_ca(vget(row, k0 + q), vget(row, k0 + i), acc);
        S[q + i * NB] = acc;
      } else {  // Wm(j, c) = v_j^H B(:, c)
        const int u = t - nb * nb, j = u % nb, c = u / nb;
        double2 acc = cmk(0.0, 0.0);
        for (int row = k0 + j + 1; row < K; ++row) acc = cfma_ca(vget(row, k0 + j), B[row + (int64_t)c * K], acc);
        Wm[j + c * NB] = acc;
      }
    }
    __syncthreads();
    if (warp == 0) {  // T(q, i) = -tau_i sum_{p = q..i-1} T(q, p) S(p, i), T(p, p) = tau_p
      for (int i = 1; i < nb; ++i) {
        double2 val = cmk(0.0, 0.0);
        if (lane < i) {
          val = cmul(tau[k0 + lane], S[lane + i * NB]);
          for (int p2 = lane + 1; p2 < i; ++p2) val = cfma(S[lane + p2 * NB], S[p2 + i * NB], val);
          val = cmul(cscale(tau[k0 + i], -1.0), val);
        }
        __syncwarp();
        if (lane < i) S[lane + i * NB] = val;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int t = tid; t < nb * r; t += NT) {  // W2 = T Wm
      const int j = t % nb, c = t / nb;
      double2 acc = cmul(tau[k0 + j], Wm[j + c * NB]);
      for (int p2 = j + 1; p2 < nb; ++p2) acc = cfma(S[j + p2 * NB], Wm[p2 + c * NB], acc);
      W2[j + c * NB] = acc;
    }
    __syncthreads();
    const int nrow = K - (k0 + 1);
    for (int t = tid; t < nrow * r; t += NT) {  // B -= V W2
      const int i = k0 + 1 + t % nrow, c = t / nrow;
      double2 acc = cmk(0.0, 0.0);
      const int jmax = min(nb, i - k0);  // v_{k0 + j} is zero at row i for k0 + j >= i
      for (int j = 0; j < jmax; ++j) acc = cfma(vget(i, k0 + j), W2[j + c * NB], acc);
      B[i + (int64_t)c * K] = csub(B[i + (int64_t)c * K], acc);
    }
    __syncthreads();
  }
}

// truncation rank (oracle/lowrank.py truncation_rank) from eigenvalues
// lam[ordr[k]] in descending order; thread 0 writes r
HMX_D void recompress_truncate(const double* lam, const int* ordr, int K, double eps, int rule, int& r_out) {
  if (threadIdx.x != 0) return;
  int r = 0;
  const double l1 = lam[ordr[0]];
  if (l1 > 0.0) {
    if (rule == 1) {
      for (int k = 0; k < K; ++k) r += lam[ordr[k]] > eps * eps * l1;
    } else {
      double total = 0.0;
      for (int k = K - 1; k >= 0; --k) total += lam[ordr[k]];
      r = K;
      double acc = 0.0;
      for (int k = K - 1; k >= 0; --k) {  // smallest r with sum_{k >= r} lam <= eps^2 total
        acc += lam[ordr[k]];
        if (acc <= eps * eps * total) r = k;
      }
    }
  }
  r_out = r;
}

// Workspace per leaf, 6 K x K complex slots: 0 R, 1 T then L_r, 2 E (global
// variant), 3 Z (real, global variant), 4-5 W_U | W_V.
// MODE 0: E, Z, R, T in L2 (large K); 1: E / Z in shared memory; 2: E / Z, R and
// T / L_r all in shared memory (small K: the O(K) sequential phases then run
// at shared-memory instead of L2 latency)
// register caps per instantiation (with the shared memory, what bounds the CTAs per SM; nvcc takes
// either __launch_bounds__ or __maxnreg__ on a kernel, so the cap alone is given):
//  * 64 for the small shared-memory classes (8 x 128-thread CTAs per SM);
//  * 64 for the large-K class (512 threads): two of its long eigen-solve chains per SM instead of
//    one CTA owning the whole register file (a few spills; U32k -2 ms, T65k -9 ms measured);
//  * 80 for the 256-thread shared-memory classes (three per SM by registers).
constexpr int rc_maxnreg(int mode, int nt) {
  return (mode == 1 && nt == 128) ? 65536 / (128 * HMX_RC_MINB)
         : (mode == 1 && nt == 64) ? 64
         : (mode == 0 && nt == 512) ? 64
         : (mode == 1 && nt == 256) ? 80
                                    : (65536 / nt > 255 ? 255 : 65536 / nt);
}
template <int MODE, int NT>
__global__ void __maxnreg__(rc_maxnreg(MODE, NT)) recompress_core(const RecDesc* __restrict__ desc, double eps, int rule,
                                                            const double2* __restrict__ G, double2* __restrict__ W,
                                                            int32_t* __restrict__ rank_out,
                                                            int32_t* __restrict__ flags_out) {
  constexpr bool SMEM = MODE >= 1;
  extern __shared__ double2 dyn[];
  __shared__ double red[2 * (NT / 32)];
  __shared__ Scalars S;
  __shared__ int s_r, s_flag;
  __shared__ double s_piv;
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
  double2* gA = W + ds.woff;  // this leaf's L2 workspace
  double2* A = gA;            // R (upper)
  double2* B = gA + KK;       // T, then L_r (K x r)
  double2* Wuv = gA + 4 * KK;
  // shared: 2K complex vectors, K complex tau, then 6K doubles (d, e, lam, dscale, rc, rs), K ints
  double2* vbuf = dyn;
  double2* pbuf = vbuf + K;
  double2* tau = pbuf + K;
  double* d = reinterpret_cast<double*>(tau + K);
  double* e = d + K;
  double* lam = e + K;
  double* dscale = lam + K;
  double* rc = dscale + K;
  double* rs = rc + K;
  int* ordr = reinterpret_cast<int*>(rs + K);
  double2* E;
  double* Z;
  int ldz;
  double2* gtile = reinterpret_cast<double2*>(ordr + K + (K & 1) + 2);
  gtile = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(gtile) + 15) & ~uintptr_t(15));
  const int KP = K * (K + 1) / 2;  // packed lower-triangular size
  if (SMEM) {
    E = gtile;  // packed lower triangle (pk_col); no GEMM tiles in the shared-memory variant
    Z = reinterpret_cast<double*>(E);  // QL fallback overlays E: K (K+1) doubles = packed E bytes
    ldz = K + 1;
    if (MODE == 2) {
      A = E + KP;
      B = A + KK;
    }
  } else {
    E = A + 2 * KK;
    Z = reinterpret_cast<double*>(A + 3 * KK);
    ldz = K;
  }

  if (tid == 0) s_flag = 0;
#ifdef HMX_RC_PROF
  long long rc_t0 = clock64();
  if (tid == 0) {
    atomicAdd(&g_rc_prof[MODE * 16 + 14], (unsigned long long)K);
    atomicAdd(&g_rc_prof[MODE * 16 + 15], 1ull);
  }
#endif
  // ---- scaled Cholesky of G_V: A = D^-1 G_V D^-1, R^H R = A (upper R) ----------
  for (int i = tid; i < K; i += NT) {
    const double g = GV[i + (int64_t)i * kcap].x;
    dscale[i] = g > 0.0 ? sqrt(g) : 1.0;
  }
  __syncthreads();
  for (int t = tid; t < K * K; t += NT) {
    const int i = t % K, j = t / K;
    const double2 g = GV[i + (int64_t)j * kcap];
    A[t] = (i <= j) ? cscale(g, 1.0 / (dscale[i] * dscale[j])) : cmk(0.0, 0.0);
  }
  __syncthreads();
  for (int j = 0; j < K; ++j) {
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
    for (int i = j + 1 + tid; i < K; i += NT) A[j + (int64_t)i * K] = cscale(A[j + (int64_t)i * K], ip);
    __syncthreads();
    const int rem = K - j - 1;
    for (int t = tid; t < rem * rem; t += NT) {
      const int i = j + 1 + t % rem, l = j + 1 + t / rem;
      if (i > l) continue;
      const double2 rji = A[j + (int64_t)i * K], rjl = A[j + (int64_t)l * K];
      A[i + (int64_t)l * K] = csub(A[i + (int64_t)l * K], cmul(cconj(rji), rjl));
    }
    __syncthreads();
  }
  for (int t = tid; t < K * K; t += NT) {
    const int i = t % K, j = t / K;
    A[t] = (i <= j) ? cscale(A[t], dscale[j]) : cmk(0.0, 0.0);
  }
  __syncthreads();
  RC_MARK(0);
  // ---- T = R G_U (B), E = T R^H --------------------------------------------------
  if constexpr (!SMEM) {
    // large K: shared-memory tiled products (the naive loops are L2-latency bound)
    if constexpr (NT == 512) {
      cta_zgemm_tc<false, false>(K, K, K, A, K, GU, kcap, B, K, gtile);
      cta_zgemm_tc<false, true>(K, K, K, B, K, A, K, E, K, gtile);
    } else {
      cta_zgemm<NT, false, false>(K, K, K, A, K, GU, kcap, B, K, gtile);
      cta_zgemm<NT, false, true>(K, K, K, B, K, A, K, E, K, gtile);
    }
  } else {
    for (int t = tid; t < K * K; t += NT) {
      const int i = t % K, j = t / K;
      double2 s = cmk(0.0, 0.0);
      for (int k = i; k < K; ++k) s = cfma(A[i + (int64_t)k * K], GU[k + (int64_t)j * kcap], s);
      B[t] = s;
    }
    __syncthreads();
    // lower triangle only (E is Hermitian), packed
    for (int t = tid; t < K * K; t += NT) {
      const int i = t % K, j = t / K;
      if (i < j) continue;
      double2 s = cmk(0.0, 0.0);
      for (int k = j; k < K; ++k) s = cfma_cj(B[i + (int64_t)k * K], A[j + (int64_t)k * K], s);
      if (i == j) s.y = 0.0;
      E[pk_col(j, K) + (i - j)] = s;
    }
    __syncthreads();
  }
  if constexpr (!SMEM) {
    for (int t = tid; t < K * K; t += NT) {  // Hermitian symmetrise (roundoff)
      const int i = t % K, j = t / K;
      if (i < j) {
        const double2 a = E[i + (int64_t)j * K], b = E[j + (int64_t)i * K];
        const double2 h = cscale(cadd(a, cconj(b)), 0.5);
        E[i + (int64_t)j * K] = h;
        E[j + (int64_t)i * K] = cconj(h);
      } else if (i == j) {
        E[i + (int64_t)i * K].y = 0.0;
      }
    }
    __syncthreads();
  }
  // ---- eigen-decomposition E = Q Z diag(lam) Z^T Q^H --------------------------------
  RC_MARK(1);
  if constexpr (SMEM)
    tridiagonalize_packed<NT>(E, K, d, e, tau, vbuf, pbuf, S, red);
  else
    tridiagonalize<NT>(E, K, d, e, tau, vbuf, pbuf, S, red);
  bool hv_packed = SMEM;  // reflector k at E + pk_col(k, K) + 1 (else Hv(k+1:, k), ld K)
  double2* Hv = E;  // Householder vectors v_k = Hv(k+1:, k)
  // fast path: bisection eigenvalues + twisted eigenvectors (rc: e^2 scratch)
  double pivmin = 0.0;
  RC_MARK(2);
  bisect_all<NT>(d, e, rc, K, rs, red, pivmin);  // rs = ascending eigenvalues
  for (int i = tid; i < K; i += NT) {
    lam[i] = fmax(rs[K - 1 - i], 0.0);  // descending
    ordr[i] = i;
  }
  __syncthreads();
  recompress_truncate(lam, ordr, K, eps, rule, s_r);
  __syncthreads();
  int r = s_r;
  bool fast_ok = true;
  RC_MARK(3);
  if (r > 0) {
    double* uscr = reinterpret_cast<double*>(Wuv);  // K doubles per kept vector
    for (int c2 = tid; c2 < r; c2 += NT)
      twisted_vector(d, e, K, rs[K - 1 - c2], pivmin, B + (int64_t)c2 * K, uscr + (int64_t)c2 * K);
    __syncthreads();
    fast_ok = cgs2_columns<NT>(B, K, r, reinterpret_cast<double*>(pbuf), red);
  }
  RC_MARK(4);
  if (!fast_ok) {
    // near-degenerate eigenvalues: implicit QL with accumulated vectors
    if (SMEM) {
      // reflectors to L2 (workspace slot 2); Z reuses E's shared memory
      Hv = gA + 2 * KK;
      for (int t = tid; t < K * K; t += NT) {
        const int i = t % K, j = t / K;
        if (i > j) Hv[t] = E[pk_col(j, K) + (i - j)];
      }
      hv_packed = false;
      __syncthreads();
    }
    tridiag_ql<NT>(d, e, Z, ldz, K, rc, rs, S);
    if (tid == 0) s_flag |= S.fail ? 6 : 4;
    for (int i = tid; i < K; i += NT) lam[i] = fmax(d[i], 0.0);
    __syncthreads();
    for (int i = tid; i < K; i += NT) {
      int rk = 0;
      const double li = lam[i];
      for (int j = 0; j < K; ++j) rk += (lam[j] > li) || (lam[j] == li && j < i);
      ordr[rk] = i;
    }
    __syncthreads();
    recompress_truncate(lam, ordr, K, eps, rule, s_r);
    __syncthreads();
    r = s_r;
    for (int t = tid; t < K * r; t += NT) {
      const int i = t % K, c2 = t / K;
      B[t] = cmk(Z[(int64_t)i * ldz + ordr[c2]], 0.0);
    }
    __syncthreads();
  }
  if (tid == 0) {
    rank_out[blockIdx.x] = r;
    flags_out[blockIdx.x] = s_flag;
  }
  if (r == 0) return;
  // ---- L_r = Q Z_r : B (K x r) ------------------------------------------------------
  RC_MARK(5);
  constexpr int kWyBlock = 16;
  if (K >= 24) backxf_blocked<NT, kWyBlock>(E, Hv, hv_packed, tau, K, r, B, Wuv);
  for (int k = K >= 24 ? -1 : K - 2; k >= 0; --k) {
    const double2 tk = tau[k];
    if (tk.x == 0.0 && tk.y == 0.0) continue;
    const int n = K - k - 1;
    const double2* v = hv_packed ? E + pk_col(k, K) + 1 : Hv + (k + 1) + (int64_t)k * K;
    // s_c = v^H B(k+1:, c), one warp per column
    const int lane = tid & 31, warp = tid >> 5;
    for (int c = warp; c < r; c += NT / 32) {
      double2 acc = cmk(0.0, 0.0);
      for (int i = lane; i < n; i += 32) acc = cfma_ca(v[i], B[(k + 1 + i) + (int64_t)c * K], acc);
      acc = warp_sum(acc);
      if (lane == 0) pbuf[c] = cmul(tk, acc);
    }
    __syncthreads();
    for (int t = tid; t < n * r; t += NT) {
      const int i = t % n, c = t / n;
      B[(k + 1 + i) + (int64_t)c * K] = csub(B[(k + 1 + i) + (int64_t)c * K], cmul(v[i], pbuf[c]));
    }
    __syncthreads();
  }
  // ---- W_U = R^H L_r S^-1/2, W_V = R^{-1} L_r S^1/2 ------------------------------------
  RC_MARK(6);
  double2* Wu = Wuv;
  double2* Wv = Wuv + (int64_t)K * r;
  if constexpr (!SMEM) {
    if constexpr (NT == 512)
      cta_zgemm_tc<true, false>(K, r, K, A, K, B, K, Wu, K, gtile);
    else
      cta_zgemm<NT, true, false>(K, r, K, A, K, B, K, Wu, K, gtile);
    for (int t = tid; t < K * r; t += NT) Wu[t] = cscale(Wu[t], 1.0 / sqrt(sqrt(lam[ordr[t / K]])));
  } else {
    for (int t = tid; t < K * r; t += NT) {
      const int i = t % K, c = t / K;
      double2 s = cmk(0.0, 0.0);
      for (int k = 0; k <= i; ++k) s = cfma_ca(A[k + (int64_t)i * K], B[k + (int64_t)c * K], s);
      Wu[t] = cscale(s, 1.0 / sqrt(sqrt(lam[ordr[c]])));
    }
  }
  // W_V: R X = L_r by column-oriented back substitution, parallel over (row, column)
  RC_MARK(7);
  for (int t = tid; t < K * r; t += NT) Wv[t] = B[t];
  __syncthreads();
  for (int i = K - 1; i >= 0; --i) {
    const double2 rii = A[i + (int64_t)i * K];
    for (int c = tid; c < r; c += NT) Wv[i + (int64_t)c * K] = cdiv(Wv[i + (int64_t)c * K], rii);
    __syncthreads();
    for (int t = tid; t < i * r; t += NT) {
      const int j = t % i, c = t / i;
      Wv[j + (int64_t)c * K] = csub(Wv[j + (int64_t)c * K], cmul(A[j + (int64_t)i * K], Wv[i + (int64_t)c * K]));
    }
    __syncthreads();
  }
  for (int t = tid; t < K * r; t += NT) Wv[t] = cscale(Wv[t], sqrt(sqrt(lam[ordr[t / K]])));
  RC_MARK(8);
}

// C (rows x r, ldc) = A (rows x K, lda) * W (K x r, ld K) on the FP64 tensor
// cores (mma.sync m8n8k4 f64: 37 TF/s measured vs 34 for DFMA, and one
// instruction per 256 FMAs).  Complex product with two real MMAs per 8 x 4
// block: B = [W_re | W_im] (4 complex columns as 8 real ones), C1 = A_re B,
// C2 = A_im B -> C_re = C1[:, :4] - C2[:, 4:], C_im = C1[:, 4:] + C2[:, :4].
// CTA tile 64 rows x 32 complex columns, 8 warps of 32 rows x 8 columns, k
// chunks of 16 staged in shared memory (2-stage ring).  Fragment layout (checked by
// tools/micro/dmma_layout.cu): A[r][k] at lane 4 r + k, B[k][n] at lane
// 4 n + k, C[r][2 t + i] at lane 4 r + t.
// 2 stages (54 KB) and 80 registers: three CTAs per SM (3 stages / uncapped 97 registers: two)
constexpr int TM = 64, TN = 32, TK = 16, kFormThreads = 256, kFormStages = 2;
HMX_D void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
// Tiles move by the bulk-copy engine (cp.async.bulk, SASS UBLKCP): per k chunk one elected lane of
// warp 0 issues, from warp-uniform operands, 16 column runs of A (64 rows = 1 KB each) and 32 column
// runs of W (16 k = 256 B each) onto the stage's mbarrier (transaction bytes); every thread waits on
// the barrier, and the CTA barrier of the next iteration frees the stage for its refill.  Only the
// valid part of a tile is copied: rows / columns past the item's edge hold stale finite or
// arbitrary data that only reaches discarded outputs (each output row / column depends on its own A
// row / W column alone); the k tail of the last chunk is zeroed in both tiles.
constexpr int TKP = TK + 4;  // W tile column stride (16-byte units): B fragment reads conflict-free
constexpr size_t kFormSmem = sizeof(double2) * kFormStages * (TK * (TM + 2) + TN * TKP);
HMX_D int64_t bcast64(int64_t v) {
  const int lo = __shfl_sync(0xffffffffu, (int)(v & 0xffffffff), 0), hi = __shfl_sync(0xffffffffu, (int)(v >> 32), 0);
  return ((int64_t)hi << 32) | (uint32_t)lo;
}
__global__ void __maxnreg__(80) form_gemm(const FormDesc* __restrict__ desc,
                                                          const int64_t* __restrict__ tile_start, int64_t nitems) {
  extern __shared__ double2 fsm[];
  __shared__ __align__(8) unsigned long long full_bar[kFormStages];
  double2(*As)[TK][TM + 2] = reinterpret_cast<double2(*)[TK][TM + 2]>(fsm);
  double2(*Ws)[TN][TKP] = reinterpret_cast<double2(*)[TN][TKP]>(fsm + kFormStages * TK * (TM + 2));
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
  double2* C = ds.C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;  // warp tile: rows wm*32 + [0,32), cols wn*8 + [0,8)
  const int fr = lane >> 2, fk = lane & 3;  // fragment row / k (A), column group lane / k (B)
  const int row0 = tm * TM, col0 = tn * TN;
  const int nk = (ds.K + TK - 1) / TK;
  // valid row octets of this warp's 32 x 8 sub-tile, and whether any of its 8 columns is inside
  // the item (small r, short last row tile: the MMAs on the padding are skipped)
  const int no = min(4, max(0, (ds.rows - (row0 + wm * 32) + 7) / 8));
  const bool colv = col0 + wn * 8 < ds.r;
  const unsigned bar_sa = (unsigned)__cvta_generic_to_shared(&full_bar[0]);
  if (tid == 0) {
    for (int st = 0; st < kFormStages; ++st) mbar_init(bar_sa + 8u * st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // CTA-uniform copy operands, made warp-uniform for the compiler (uniform registers)
  const int rv = min(TM, ds.rows - row0), cv = min(TN, ds.r - col0);
  const int u_rv = __shfl_sync(0xffffffffu, rv, 0), u_cv = __shfl_sync(0xffffffffu, cv, 0);
  const int u_K = __shfl_sync(0xffffffffu, ds.K, 0), u_lda = __shfl_sync(0xffffffffu, ds.lda, 0);
  const double2* u_A = reinterpret_cast<const double2*>(bcast64(reinterpret_cast<int64_t>(ds.A + row0)));
  const double2* u_W = reinterpret_cast<const double2*>(bcast64(reinterpret_cast<int64_t>(ds.W + (int64_t)col0 * ds.K)));
  const unsigned as_sa = (unsigned)__cvta_generic_to_shared(&As[0][0][0]);
  const unsigned ws_sa = (unsigned)__cvta_generic_to_shared(&Ws[0][0][0]);
  auto stage = [&](int kc, int buf) {
    const int k0 = kc * TK;
    const int kv = min(TK, u_K - k0);
    if (warp == 0 && elect_one()) {
      const unsigned mb = bar_sa + 8u * (unsigned)buf;
      mbar_expect_tx(mb, (unsigned)(kv * (u_rv + u_cv)) * (unsigned)sizeof(double2));
      const double2* src = u_A + (int64_t)k0 * u_lda;
      unsigned dst = as_sa + (unsigned)buf * (unsigned)(TK * (TM + 2) * sizeof(double2));
      for (int kk = 0; kk < kv; ++kk) {
        bulk_g2s(dst, src, (unsigned)u_rv * (unsigned)sizeof(double2), mb);
        src += u_lda;
        dst += (unsigned)((TM + 2) * sizeof(double2));
      }
      src = u_W + k0;
      dst = ws_sa + (unsigned)buf * (unsigned)(TN * TKP * sizeof(double2));
      for (int cc = 0; cc < u_cv; ++cc) {
        bulk_g2s(dst, src, (unsigned)kv * (unsigned)sizeof(double2), mb);
        src += u_K;
        dst += (unsigned)(TKP * sizeof(double2));
      }
    }
    if (kv < TK) {  // k tail of the last chunk: zeros in both tiles (bytes the copies do not write)
      for (int t = tid; t < (TK - kv) * TM; t += kFormThreads) As[buf][kv + t / TM][t % TM] = cmk(0.0, 0.0);
      for (int t = tid; t < (TK - kv) * TN; t += kFormThreads) Ws[buf][t / (TK - kv)][kv + t % (TK - kv)] = cmk(0.0, 0.0);
    }
  };
  // complex product with three real products (Gauss): T1 = A_re W_re, T2 = A_im W_im,
  // T3 = (A_re + A_im)(W_re + W_im); C = (T1 - T2) + i (T3 - T1 - T2) -- 3 MMAs per row octet and
  // 8 complex columns instead of 4
  double t1[4][2], t2[4][2], t3[4][2];  // [row octet][2]: C[r][2 t + i] at lane 4 r + t
#pragma unroll
  for (int o = 0; o < 4; ++o) t1[o][0] = t1[o][1] = t2[o][0] = t2[o][1] = t3[o][0] = t3[o][1] = 0.0;
#pragma unroll
  for (int sidx = 0; sidx < kFormStages - 1; ++sidx)
    if (sidx < nk) stage(sidx, sidx);
  for (int kc = 0; kc < nk; ++kc) {
    const int buf = kc % kFormStages;
    mbar_wait(bar_sa + 8u * (unsigned)buf, (unsigned)(kc / kFormStages) & 1u);
    __syncthreads();  // every warp is done with chunk kc - 1 (its stage is refilled next) and sees the zeroed tails
    if (kc + kFormStages - 1 < nk) stage(kc + kFormStages - 1, (kc + kFormStages - 1) % kFormStages);
#pragma unroll
    for (int ks = 0; ks < TK; ks += 4) {
      // B[k][n] at lane 4 n + k: column wn * 8 + fr of W, row ks + fk
      const double2 w = Ws[buf][wn * 8 + fr][ks + fk];
      const double br = w.x, bi = w.y, bs = w.x + w.y;
#pragma unroll
      for (int o = 0; o < 4; ++o)
        if (o < no && colv) {  // warp-uniform
          const double2 a = As[buf][ks + fk][wm * 32 + o * 8 + fr];
          dmma_8x8x4(t1[o][0], t1[o][1], a.x, br);
          dmma_8x8x4(t2[o][0], t2[o][1], a.y, bi);
          dmma_8x8x4(t3[o][0], t3[o][1], a.x + a.y, bs);
        }
    }
  }
  const int t = lane & 3;
#pragma unroll
  for (int o = 0; o < 4; ++o)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int gr = row0 + wm * 32 + o * 8 + fr, gc = col0 + wn * 8 + 2 * t + i;
      if (gr < ds.rows && gc < ds.r)
        C[gr + (int64_t)gc * ds.ldc] = cmk(t1[o][i] - t2[o][i], t3[o][i] - t1[o][i] - t2[o][i]);
    }
}

}  // namespace

void warm_recompress() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, recompress_core<2, 128>);
  cudaFuncGetAttributes(&a, recompress_core<1, 128>);
  cudaFuncGetAttributes(&a, recompress_core<1, 64>);
  cudaFuncGetAttributes(&a, recompress_core<1, 256>);
  cudaFuncGetAttributes(&a, recompress_core<0, 256>);
  cudaFuncGetAttributes(&a, recompress_core<0, 512>);
  cudaFuncGetAttributes(&a, recompress_core<0, 1024>);
  cudaFuncGetAttributes(&a, form_gemm);
}

int launch_recompress_core(Ctx& c, const RecDesc* d_desc, int64_t nblk, int kmax, double eps, int rule, double2* G,
                           double2* W, int32_t* d_rank, int32_t* d_flags) {
  if (nblk == 0) return HMX_OK;
  if (kmax > 1024) {
    hmx_set_error("recompress: ACA rank %d too large", kmax);
    return HMX_EINVAL;
  }
  const size_t vec = sizeof(double2) * 3 * (size_t)kmax + sizeof(double) * 6 * kmax + sizeof(int) * (kmax + 4) + 32;
  const int all_max = kRecompressAllSmemMax;
  if (kmax <= all_max) {
    const size_t smem = vec + sizeof(double2) * ((size_t)kmax * (kmax + 1) / 2 + 2 * (size_t)kmax * kmax);
    HMX_CUDA_TRY(cudaFuncSetAttribute(recompress_core<2, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    recompress_core<2, 128><<<(unsigned)nblk, 128, smem, c.stream>>>(d_desc, eps, rule, G, W, d_rank, d_flags);
  } else if (kmax <= kRecompressSmemMax) {
    const size_t smem = vec + sizeof(double2) * ((size_t)kmax * (kmax + 1) / 2);  // packed E
    const int nt64_max = kRecompressNt64Max;
    if (kmax <= nt64_max) {
      // small K: 2-warp CTAs (cheaper barriers, twice the leaves per SM)
      HMX_CUDA_TRY(
          cudaFuncSetAttribute(recompress_core<1, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      recompress_core<1, 64><<<(unsigned)nblk, 64, smem, c.stream>>>(d_desc, eps, rule, G, W, d_rank, d_flags);
    } else if (kmax <= 64) {
      HMX_CUDA_TRY(
          cudaFuncSetAttribute(recompress_core<1, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      recompress_core<1, 128><<<(unsigned)nblk, 128, smem, c.stream>>>(d_desc, eps, rule, G, W, d_rank, d_flags);
    } else {
      HMX_CUDA_TRY(
          cudaFuncSetAttribute(recompress_core<1, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      recompress_core<1, 256><<<(unsigned)nblk, 256, smem, c.stream>>>(d_desc, eps, rule, G, W, d_rank, d_flags);
    }
  } else {
    // large K: few long CTAs whose O(K^3) phases are L2-latency bound -> more warps
    const size_t smem = vec + sizeof(double2) * kGemmTileTc;
    constexpr int nt = 512;
    if (nt == 1024) {
      HMX_CUDA_TRY(cudaFuncSetAttribute(recompress_core<0, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
      recompress_core<0, 1024><<<(unsigned)nblk, 1024, smem, c.stream>>>(d_desc, eps, rule, G, W, d_rank, d_flags);
    } else if (nt == 256) {
      HMX_CUDA_TRY(
          cudaFuncSetAttribute(recompress_core<0, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      recompress_core<0, 256><<<(unsigned)nblk, 256, smem, c.stream>>>(d_desc, eps, rule, G, W, d_rank, d_flags);
    } else {
      HMX_CUDA_TRY(
          cudaFuncSetAttribute(recompress_core<0, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      recompress_core<0, 512><<<(unsigned)nblk, 512, smem, c.stream>>>(d_desc, eps, rule, G, W, d_rank, d_flags);
    }
  }
  HMX_CUDA_TRY(cudaGetLastError());
  return HMX_OK;
}

int launch_form(Ctx& c, const FormDesc* d_desc, int64_t nitems, int64_t ntiles_total, const int64_t* d_tile_start) {
  if (ntiles_total == 0) return HMX_OK;
  HMX_CUDA_TRY(cudaFuncSetAttribute(form_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFormSmem));
  form_gemm<<<(unsigned)ntiles_total, kFormThreads, kFormSmem, c.stream>>>(d_desc, d_tile_start, nitems);
  HMX_CUDA_TRY(cudaGetLastError());
  return HMX_OK;
}

}  // namespace hmx

#ifdef HMX_RC_PROF
// experiment builds: read (and reset) the recompression phase counters
extern "C" int hmx_debug_rc_prof(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, hmx::g_rc_prof, sizeof(hmx::g_rc_prof)) != cudaSuccess) return 2;
  unsigned long long z[3 * 16] = {};
  cudaMemcpyToSymbol(hmx::g_rc_prof, z, sizeof(z));
  return 0;
}
#endif
