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

}  // namespace fpb
