// Per-pair Green's-tensor evaluation (device), complex128.
//
// Same formulas and the same formula STRUCTURE as the reference kernel core
// (/root/reference/pkg/src/hmatx/_kernelcore_np.py; math in SURVEY.md
// Appendix A): the elastodynamic coefficients are built from the differences
// f^(q) = G_ks^(q) - G_kp^(q) of the two Helmholtz radial series, exactly as
// _kernelcore_np.py:52-71 does, so the low-kappa*r cancellation behaves the
// same way and entries agree with the reference to ~1e-13 relative.
//
//   scalar  e^{i k r}/(4 pi r)                                (:37-49)
//   U_ab  = A d_ab + B z_a z_b                                (:89-102)
//   T_ab  = a1 n_a z_b + a2 z_a n_b + a3 z_a z_b + a4 d_ab     (:105-130)
//           a1 = -lam D - 2 mu B/r,  a2 = -mu (A' + B/r),
//           a3 = c mu (4 B/r - 2 B'),  a4 = -c mu (A' + B/r),
//           D = A' + B' + 2 B/r,  c = n.z   (n = column-point normal)
// which is the reference's four-term T expression with like terms collected.
// Self pairs (exact r == 0, _kernelcore_np.py:40,92,108) -> shift * I.
#pragma once
#include "hmx_common.cuh"

struct GreenParams {
  int kind;      // 0 = Helmholtz/Laplace (d=1), 1 = elasto U, 2 = elasto T (d=3)
  double kappa;  // Helmholtz
  double kp, ks, lam, mu, scale;  // elastodynamics, scale = 1/(rho omega^2)
  double shift;  // self-block value zeta
  int has_shift;
};

// Points in tree order, structure-of-arrays for coalesced loads.
struct PointsSoA {
  const double* __restrict__ x;
  const double* __restrict__ y;
  const double* __restrict__ z;
  const double* __restrict__ nx;  // normals (T only), may be null
  const double* __restrict__ ny;
  const double* __restrict__ nz;
};

#define HMX_INV_4PI 0.079577471545947667884441881686257181

// g^(q)(r), q = 0..NDER, of g = e^{ikr}/(4 pi r)  (_kernelcore_np.py:23-34)
template <int NDER>
HMX_D void radial_series(double k, double r, double ir, double2* g) {
  double s, c;
  sincos(k * r, &s, &c);
  const double scl = HMX_INV_4PI * ir;
  const double2 e = cmk(c * scl, s * scl);
  g[0] = e;
  if (NDER >= 1) g[1] = cmul(e, cmk(-ir, k));
  if (NDER >= 2) {
    const double ir2 = ir * ir;
    g[2] = cmul(e, cmk(-k * k + 2.0 * ir2, -2.0 * k * ir));
    if (NDER >= 3) g[3] = cmul(e, cmk(3.0 * k * k * ir - 6.0 * ir2 * ir, -k * k * k + 6.0 * k * ir2));
  }
}

// d = 1: out[0]; d = 3: out[3a+b] = G_ab.  Returns false for a coincident
// pair without a self rule (reference returns None -> SingularEvaluationError).
// KIND is the compile-time kernel kind (0 H, 1 U, 2 T); -1 dispatches on P.kind.
template <int KIND>
HMX_D bool green_pair_k(const GreenParams& P, double dx, double dy, double dz, double nxv, double nyv,
                        double nzv, double2* out) {
  const int kind = KIND >= 0 ? KIND : P.kind;
  const double r2 = dx * dx + dy * dy + dz * dz;
  if (r2 == 0.0) {
    if (kind == 0) {
      out[0] = cmk(P.shift, 0.0);
    } else {
#pragma unroll
      for (int t = 0; t < 9; ++t) out[t] = cmk((t % 4 == 0) ? P.shift : 0.0, 0.0);
    }
    return P.has_shift != 0;
  }
  const double r = sqrt(r2);
  const double ir = 1.0 / r;
  if (kind == 0) {
    double s, c;
    sincos(P.kappa * r, &s, &c);
    const double scl = HMX_INV_4PI * ir;
    out[0] = cmk(c * scl, s * scl);
    return true;
  }
  if (KIND == 0) return true;  // unreachable: kind 0 returned above
  const double z[3] = {dx * ir, dy * ir, dz * ir};
  if (kind == 1) {
    double2 gs[3], gp[3];
    radial_series<2>(P.ks, r, ir, gs);
    radial_series<2>(P.kp, r, ir, gp);
    const double2 f1 = csub(gs[1], gp[1]);
    const double2 f2 = csub(gs[2], gp[2]);
    const double2 f1r = cscale(f1, ir);
    const double2 A = cscale(cadd(cscale(gs[0], P.ks * P.ks), f1r), P.scale);
    const double2 B = cscale(csub(f2, f1r), P.scale);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const double zz = z[a] * z[b];
        double2 v = cscale(B, zz);
        if (a == b) v = cadd(v, A);
        out[3 * a + b] = v;
      }
    return true;
  }
  if (KIND == 1) return true;  // unreachable
  // kind == 2: traction T
  double2 gs[4], gp[4];
  radial_series<3>(P.ks, r, ir, gs);
  radial_series<3>(P.kp, r, ir, gp);
  const double2 f1 = csub(gs[1], gp[1]);
  const double2 f2 = csub(gs[2], gp[2]);
  const double2 f3 = csub(gs[3], gp[3]);
  const double2 f1r = cscale(f1, ir);
  const double2 A = cscale(cadd(cscale(gs[0], P.ks * P.ks), f1r), P.scale);
  (void)A;
  const double2 B = cscale(csub(f2, f1r), P.scale);
  const double2 h = cscale(csub(cscale(f2, r), f1), ir * ir);  // (f'' r - f')/r^2
  const double2 Ap = cscale(cadd(cscale(gs[1], P.ks * P.ks), h), P.scale);
  const double2 Bp = cscale(csub(f3, h), P.scale);
  const double2 Br = cscale(B, ir);
  const double2 D = cadd(cadd(Ap, Bp), cscale(Br, 2.0));
  const double n[3] = {nxv, nyv, nzv};
  const double c = n[0] * z[0] + n[1] * z[1] + n[2] * z[2];
  const double mu = P.mu;
  const double2 a1 = csub(cscale(D, -P.lam), cscale(Br, 2.0 * mu));
  const double2 ApBr = cadd(Ap, Br);
  const double2 a2 = cscale(ApBr, -mu);
  const double2 a3 = cscale(csub(cscale(Br, 4.0), cscale(Bp, 2.0)), c * mu);
  const double2 a4 = cscale(ApBr, -c * mu);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double2 v = cscale(a1, n[a] * z[b]);
      v = cadd(v, cscale(a2, z[a] * n[b]));
      v = cadd(v, cscale(a3, z[a] * z[b]));
      if (a == b) v = cadd(v, a4);
      out[3 * a + b] = v;
    }
  return true;
}

HMX_D bool green_pair(const GreenParams& P, double dx, double dy, double dz, double nxv, double nyv, double nzv,
                      double2* out) {
  return green_pair_k<-1>(P, dx, dy, dz, nxv, nyv, nzv, out);
}

// Entry block of row point i of X and column point j of Y (normals from Y).
template <int KIND>
HMX_D bool green_xy_k(const GreenParams& P, const PointsSoA& X, int64_t i, const PointsSoA& Y, int64_t j,
                      double2* out) {
  const double dx = X.x[i] - Y.x[j];
  const double dy = X.y[i] - Y.y[j];
  const double dz = X.z[i] - Y.z[j];
  double nx = 0, ny = 0, nz = 0;
  if ((KIND >= 0 ? KIND : P.kind) == 2) {
    nx = Y.nx[j];
    ny = Y.ny[j];
    nz = Y.nz[j];
  }
  return green_pair_k<KIND>(P, dx, dy, dz, nx, ny, nz, out);
}

HMX_D bool green_xy(const GreenParams& P, const PointsSoA& X, int64_t i, const PointsSoA& Y, int64_t j,
                    double2* out) {
  return green_xy_k<-1>(P, X, i, Y, j, out);
}
