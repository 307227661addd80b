// Affine-simplex (TRI03, TET04) geometry and closed-form element integrals,
// shared by the row-owned kernels (rows.cu) and the element-block kernels
// (blocks.cu).
#pragma once
#include "elemcore.cuh"

namespace fpb {

// ---- affine simplex geometry -------------------------------------------------
// dN is -1 on node 0 and +1 on node l+1 (elements.py:118-145), so
// J[d][l] = x[l+1][d] - x[0][d] and gN[.][0] = -(Ji[0][.] + Ji[1][.] + ...),
// bit-identical to the reference's accumulation with the tabulated dN.
template <int ET>
__device__ __forceinline__ double simplex_geometry(const double (&xe)[Elem<ET>::NN][Elem<ET>::DIM],
                                                   double (&gN)[Elem<ET>::DIM][Elem<ET>::NN]) {
  constexpr int DIM = Elem<ET>::DIM;
  double J[DIM][DIM], Ji[DIM][DIM];
#pragma unroll
  for (int d = 0; d < DIM; ++d)
#pragma unroll
    for (int l = 0; l < DIM; ++l) J[d][l] = xe[l + 1][d] - xe[0][d];
  double det;
  if constexpr (DIM == 2) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double inv = 1.0 / det;
    Ji[0][0] = J[1][1] * inv;
    Ji[0][1] = -J[0][1] * inv;
    Ji[1][0] = -J[1][0] * inv;
    Ji[1][1] = J[0][0] * inv;
  } else {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c10 = J[1][0] * J[2][2] - J[1][2] * J[2][0];
    const double c20 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    det = J[0][0] * c00 - J[0][1] * c10 + J[0][2] * c20;
    const double inv = 1.0 / det;
    Ji[0][0] = c00 * inv;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * inv;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * inv;
    Ji[1][0] = -c10 * inv;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * inv;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * inv;
    Ji[2][0] = c20 * inv;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * inv;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * inv;
  }
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    double s = -Ji[0][d];
#pragma unroll
    for (int l = 1; l < DIM; ++l) s -= Ji[l][d];
    gN[d][0] = s;
#pragma unroll
    for (int l = 0; l < DIM; ++l) gN[d][l + 1] = Ji[l][d];
  }
  return det;
}

// det * gN (the adjugate form) without the reciprocal: for integrands that
// are linear in gN and carry one factor det (MASS, CONVECTION, GRADIENT_k)
// the row kernels use dg = det gN directly, which rounds within an ulp of
// det * (adj / det) and saves the FP64 reciprocal sequence per element.
template <int ET>
__device__ __forceinline__ double simplex_adj(const double (&xe)[Elem<ET>::NN][Elem<ET>::DIM],
                                              double (&dg)[Elem<ET>::DIM][Elem<ET>::NN]) {
  constexpr int DIM = Elem<ET>::DIM;
  double J[DIM][DIM], A[DIM][DIM];  // A = det * J^-1
#pragma unroll
  for (int d = 0; d < DIM; ++d)
#pragma unroll
    for (int l = 0; l < DIM; ++l) J[d][l] = xe[l + 1][d] - xe[0][d];
  double det;
  if constexpr (DIM == 2) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    A[0][0] = J[1][1];
    A[0][1] = -J[0][1];
    A[1][0] = -J[1][0];
    A[1][1] = J[0][0];
  } else {
    A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c10 = J[1][0] * J[2][2] - J[1][2] * J[2][0];
    A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    det = J[0][0] * A[0][0] - J[0][1] * c10 + J[0][2] * A[2][0];
    A[1][0] = -c10;
    A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  }
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    double s = -A[0][d];
#pragma unroll
    for (int l = 1; l < DIM; ++l) s -= A[l][d];
    dg[d][0] = s;
#pragma unroll
    for (int l = 0; l < DIM; ++l) dg[d][l + 1] = A[l][d];
  }
  return det;
}

// v[a] for a runtime a, without dynamic register indexing (selects)
template <int NN>
__device__ __forceinline__ double pick(const double (&v)[NN], int a) {
  double r = v[0];
#pragma unroll
  for (int b = 1; b < NN; ++b) r = (a == b) ? v[b] : r;
  return r;
}

// All rows of an affine simplex's RHS in closed form (see rows.cu header):
//   MOMENTUM r[a][k] = -det (rho sum_l ubar_a[l] Mc[l][k] + 2 mu W sum_l S[k][l] gN[l][a])
//   SCALAR   r[a]    = -det (ubar_a . gphi + kappa W gphi . gN_a)
// with ubar_a = sum_c M[a][c] u_c; the reference's 4-point rule integrates
// these polynomials exactly, so the Gauss loop and this form agree to rounding.
template <int ET, int KIND>
__device__ __forceinline__ void simplex_rhs_all(
    const double (&xe)[Elem<ET>::NN][Elem<ET>::DIM], const double (&ue)[Out<ET, KIND>::NU][Elem<ET>::DIM],
    const double (&fe)[Out<ET, KIND>::NF], double rho, double mu, double kappa,
    double (&acc)[Out<ET, KIND>::NOUT]) {
  constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM;
  double gN[DIM][NN];
  const double det = simplex_geometry<ET>(xe, gN);
  const double W = refWsum<ET>();
  if constexpr (KIND == FPB_MOMENTUM_RHS) {
    double G[DIM][DIM];  // G[l][k] = d u_k / d x_l
#pragma unroll
    for (int l = 0; l < DIM; ++l)
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < NN; ++b) s += ue[b][k] * gN[l][b];
        G[l][k] = s;
      }
    double divu = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) divu += G[d][d];
    double S[DIM][DIM], Mc[DIM][DIM];
#pragma unroll
    for (int l = 0; l < DIM; ++l)
#pragma unroll
      for (int k = 0; k < DIM; ++k) S[l][k] = 0.5 * (G[l][k] + G[k][l]);
#pragma unroll
    for (int l = 0; l < DIM; ++l)
#pragma unroll
      for (int k = 0; k < DIM; ++k) Mc[l][k] = 2.0 * S[l][k] + (l == k ? divu : 0.0) - G[k][l];
    const double drho = rho * det, dvisc = 2.0 * mu * det * W;
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      double ub[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NN; ++c) s += refM<ET>(a, c) * ue[c][d];
        ub[d] = s;
      }
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        double conv = 0.0, visc = 0.0;
#pragma unroll
        for (int l = 0; l < DIM; ++l) {
          conv += ub[l] * Mc[l][k];
          visc += S[k][l] * gN[l][a];
        }
        acc[a * DIM + k] = -(drho * conv + dvisc * visc);
      }
    }
  } else if constexpr (KIND == KIND_SCALAR3) {  // three scalars, one velocity: ubar shared
    const double kap[3] = {rho, mu, kappa};
    double gphi[3][DIM];
#pragma unroll
    for (int f = 0; f < 3; ++f)
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NN; ++c) s += fe[f * NN + c] * gN[d][c];
        gphi[f][d] = s;
      }
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      double ub[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NN; ++c) s += refM<ET>(a, c) * ue[c][d];
        ub[d] = s;
      }
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        double adv = 0.0, diff = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          adv += ub[d] * gphi[f][d];
          diff += gphi[f][d] * gN[d][a];
        }
        acc[a * 3 + f] = -(det * adv + kap[f] * det * W * diff);
      }
    }
  } else {  // SCALAR_RHS
    double gphi[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < NN; ++c) s += fe[c] * gN[d][c];
      gphi[d] = s;
    }
    const double dk = kappa * det * W;
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      double adv = 0.0, diff = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NN; ++c) s += refM<ET>(a, c) * ue[c][d];
        adv += s * gphi[d];
        diff += gphi[d] * gN[d][a];
      }
      acc[a] = -(det * adv + dk * diff);
    }
  }
}

// P1 tetrahedron momentum residual in adjugate form (no J^-1 scaling, one
// reciprocal).  x[b], u[b]: positions / velocities of the local nodes b =
// 0..3 (reference order); res[b][k] -= the element residual of
// _kernels.py:320-382 (momentum_rhs_packed), closed form:
//   E_b = x_b - x_0, A = rows (E2 x E3, E3 x E1, E1 x E2) = det J^-1,
//   Ga[l][k] = sum_b (u_b - u_0)[k] A[b-1][l]  (= det du_k/dx_l),
//   convective part  rho sum_l ub_a[l] (Ga + div Ga I)[l][k]  with
//     ub_a = sum_c M[a][c] u_c = (W/20) (U + u_a),  U = sum_c u_c,
//   viscous part     (mu W / det) sum_l (Ga[k][l] + Ga[l][k]) dg[l][a],
//     dg[.][a] = A[a-1] (a >= 1), dg[.][0] = -(A[0] + A[1] + A[2]).
// r = rho W / 20 (= rho * M[0][1]); muW = mu * W.  The 4-point rule of the
// reference integrates these polynomials exactly, so this agrees with its
// Gauss loop to rounding (~190 FP64 instructions instead of ~285).
template <class Sub>
__device__ __forceinline__ void tet_mom_adj_f(const double (&x)[4][3], const double (&u)[4][3], double r, double muW,
                                              Sub&& sub) {
  double E[3][3], A[3][3], du[3][3];
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      E[b][d] = x[b + 1][d] - x[0][d];
      du[b][d] = u[b + 1][d] - u[0][d];
    }
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const double* p = E[(b + 1) % 3];
    const double* q = E[(b + 2) % 3];
    A[b][0] = p[1] * q[2] - p[2] * q[1];
    A[b][1] = p[2] * q[0] - p[0] * q[2];
    A[b][2] = p[0] * q[1] - p[1] * q[0];
  }
  const double det = E[0][0] * A[0][0] + E[0][1] * A[0][1] + E[0][2] * A[0][2];
  double G[3][3];
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int k = 0; k < 3; ++k) G[l][k] = du[0][k] * A[0][l] + du[1][k] * A[1][l] + du[2][k] * A[2][l];
  const double divu = G[0][0] + G[1][1] + G[2][2];
  const double f = muW / det;
  double Mr[3][3], Sf[3][3];
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      Mr[l][k] = r * (l == k ? G[l][k] + divu : G[l][k]);
      Sf[l][k] = l == k ? (2.0 * f) * G[l][l] : f * (G[l][k] + G[k][l]);
    }
  double vs[3][3];  // viscous part of nodes 1..3
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) vs[a][k] = Sf[k][0] * A[a][0] + Sf[k][1] * A[a][1] + Sf[k][2] * A[a][2];
  double U[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) U[d] = (u[0][d] + u[1][d]) + (u[2][d] + u[3][d]);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double w[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) w[d] = U[d] + u[a][d];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double v = a == 0 ? -((vs[0][k] + vs[1][k]) + vs[2][k]) : vs[a - 1][k];
      sub(a, k, fma(w[0], Mr[0][k], fma(w[1], Mr[1][k], fma(w[2], Mr[2][k], v))));
    }
  }
}
__device__ __forceinline__ void tet_mom_adj(const double (&x)[4][3], const double (&u)[4][3], double r, double muW,
                                            double (&res)[4][3]) {
  tet_mom_adj_f(x, u, r, muW, [&](int a, int k, double v) { res[a][k] -= v; });
}

// 1/x from the hardware approximation plus two Newton steps (~2^-100 from the
// ~2^-23 start, i.e. the FP64 result to within an ulp; no slow-path branch)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// The same residual from precomputed adjugate rows A (= rows of det J^-1),
// det, the velocity differences du[b] = u_{b+1} - u_0 and w0 = U + u_0 =
// 5 u_0 + sum_b du[b] (so that U + u_a = w0 + du[a-1]).  Used by the
// Kuhn-cell kernel (kmom.cu), where the cross products and differences
// against the cell's shared nodes are computed once per cell.
template <class Sub>
__device__ __forceinline__ void tet_mom_core(const double (&A)[3][3], double det, const double (&du)[3][3],
                                             const double (&w0)[3], double r, double muW, Sub&& sub) {
  double G[3][3];
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int k = 0; k < 3; ++k) G[l][k] = du[0][k] * A[0][l] + du[1][k] * A[1][l] + du[2][k] * A[2][l];
  const double divu = G[0][0] + G[1][1] + G[2][2];
  const double f = muW * rcp_nr(det);
  double Mr[3][3], Sf[3][3];
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      Mr[l][k] = r * (l == k ? G[l][k] + divu : G[l][k]);
      Sf[l][k] = l == k ? (2.0 * f) * G[l][l] : f * (G[l][k] + G[k][l]);
    }
  double vs[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) vs[a][k] = Sf[k][0] * A[a][0] + Sf[k][1] * A[a][1] + Sf[k][2] * A[a][2];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double w[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) w[d] = a == 0 ? w0[d] : w0[d] + du[a - 1][d];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double v = a == 0 ? -((vs[0][k] + vs[1][k]) + vs[2][k]) : vs[a - 1][k];
      sub(a, k, fma(w[0], Mr[0][k], fma(w[1], Mr[1][k], fma(w[2], Mr[2][k], v))));
    }
  }
}

__device__ __forceinline__ void cross3(const double (&p)[3], const double (&q)[3], double (&o)[3]) {
  o[0] = p[1] * q[2] - p[2] * q[1];
  o[1] = p[2] * q[0] - p[0] * q[2];
  o[2] = p[0] * q[1] - p[1] * q[0];
}
__device__ __forceinline__ double dot3(const double (&p)[3], const double (&q)[3]) {
  return p[0] * q[0] + p[1] * q[1] + p[2] * q[2];
}

// Three scalar-transport residuals of one P1 tet sharing the velocity
// (_kernels.py:420-461 for each field; enthalpy + two species), adjugate
// form: with A the adjugate rows and gp_f = sum_b (phi_f,b+1 - phi_f,0) A[b]
// (= det grad phi_f), sub(a, f, v) subtracts
//   v = r (U + u_a) . gp_f + (kW_f / det) gp_f . dg_a,   r = W / 20,
// dg_a = A[a-1] (a >= 1), -(A[0] + A[1] + A[2]) (a = 0) — the reference's
// det ubar_a . grad phi + kappa det W grad phi . gradN_a to rounding.
template <class Sub>
__device__ __forceinline__ void tet_s3_adj(const double (&x)[4][3], const double (&u)[4][3], const double (&ph)[3][4],
                                           double r, const double (&kW)[3], Sub&& sub) {
  double E[3][3], A[3][3];
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int d = 0; d < 3; ++d) E[b][d] = x[b + 1][d] - x[0][d];
  cross3(E[1], E[2], A[0]);
  cross3(E[2], E[0], A[1]);
  cross3(E[0], E[1], A[2]);
  const double det = dot3(E[0], A[0]);
  const double inv = rcp_nr(det);
  double U[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) U[d] = (u[0][d] + u[1][d]) + (u[2][d] + u[3][d]);
  double dg0[3];
#pragma unroll
  for (int l = 0; l < 3; ++l) dg0[l] = -((A[0][l] + A[1][l]) + A[2][l]);
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    double gp[3];
#pragma unroll
    for (int l = 0; l < 3; ++l)
      gp[l] = (ph[f][1] - ph[f][0]) * A[0][l] + (ph[f][2] - ph[f][0]) * A[1][l] + (ph[f][3] - ph[f][0]) * A[2][l];
    const double fk = kW[f] * inv;
    const double ug = U[0] * gp[0] + U[1] * gp[1] + U[2] * gp[2];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const double* dg = a == 0 ? dg0 : A[a - 1];
      const double adv = ug + (u[a][0] * gp[0] + u[a][1] * gp[1] + u[a][2] * gp[2]);
      const double dif = gp[0] * dg[0] + gp[1] * dg[1] + gp[2] * dg[2];
      sub(a, f, fma(r, adv, fk * dif));
    }
  }
}

// Three scalar residuals from precomputed adjugate rows A, det, the
// differences du[b] = u_{b+1} - u_0 and dp[f][b] = phi_f,b+1 - phi_f,0, and
// w0 = U + u_0 (the Kuhn-cell form of tet_s3_adj: same terms, shared
// differences and crosses).  sub(a, f, v) subtracts v from node a, field f.
template <class Sub>
__device__ __forceinline__ void tet_s3_core(const double (&A)[3][3], double det, const double (&du)[3][3],
                                            const double (&dp)[3][3], const double (&w0)[3], double r,
                                            const double (&kW)[3], Sub&& sub) {
  const double inv = rcp_nr(det);
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    double gp[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) gp[l] = dp[f][0] * A[0][l] + dp[f][1] * A[1][l] + dp[f][2] * A[2][l];
    const double fk = kW[f] * inv;
    const double wg = w0[0] * gp[0] + w0[1] * gp[1] + w0[2] * gp[2];
    double dif[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) dif[b] = gp[0] * A[b][0] + gp[1] * A[b][1] + gp[2] * A[b][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const double adv = a == 0 ? wg : wg + (du[a - 1][0] * gp[0] + du[a - 1][1] * gp[1] + du[a - 1][2] * gp[2]);
      const double df = a == 0 ? -((dif[0] + dif[1]) + dif[2]) : dif[a - 1];
      sub(a, f, fma(r, adv, fk * df));
    }
  }
}

}  // namespace fpb
