// Per-element Gauss-point integration shared by the element kernels
// (assemble.cu: FP64-reduction scatter) and the element-block kernels
// (blocks.cu: deterministic in-block gather).  Arithmetic follows the
// reference packed kernels (_kernels.py:150-461) term by term.
#pragma once
#include "common.cuh"

#ifndef FPB_HEX_GUNROLL
#define FPB_HEX_GUNROLL 8  // Gauss-point loop unroll of hex_rhs_integrate (1 / 2 spill less in the hex-box pencils but ran 5-13 % slower at C4)
#endif
#define FPB_PRAGMA_(x) _Pragma(#x)
#define FPB_PRAGMA(x) FPB_PRAGMA_(x)

namespace fpb {

constexpr int KIND_GRADIENT_K = 100;  // CONVECTION with unit e_k, one direction k
// three SCALAR_RHS sharing one velocity (enthalpy + 2 species, timeloop.py:
// 76-79, 361-363): fields fe[s * NN + a], diffusivities (rho, mu, kappa)
// carry kappa_0..2 internally, outputs acc[a * 3 + s]
constexpr int KIND_SCALAR3 = 101;

template <int ET, int KIND>
struct Out {
  static constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM;
  static constexpr bool MAT = KIND == FPB_MASS || KIND == FPB_LAPLACIAN || KIND == FPB_CONVECTION ||
                              KIND == KIND_GRADIENT_K;
  static constexpr bool GRADXYZ = KIND == FPB_GRADIENT_XYZ;
  static constexpr bool NEED_VEL = KIND == FPB_CONVECTION || KIND == FPB_MOMENTUM_RHS || KIND == FPB_SCALAR_RHS ||
                                   KIND == KIND_SCALAR3;
  static constexpr int NU = NEED_VEL ? NN : 1;
  static constexpr int NF = KIND == FPB_SCALAR_RHS ? NN : KIND == KIND_SCALAR3 ? 3 * NN : 1;
  // values per node for RHS kinds
  static constexpr int NV = KIND == FPB_MOMENTUM_RHS ? DIM : KIND == KIND_SCALAR3 ? 3 : 1;
  static constexpr int NOUT = MAT ? NN * NN : GRADXYZ ? DIM * NN * NN : KIND == FPB_MOMENTUM_RHS ? NN * DIM
                              : KIND == KIND_SCALAR3 ? 3 * NN : NN;
};

// HEX08 momentum / scalar RHS through the Walsh forms (common.cuh): the
// same terms as element_integrate below, regrouped so that no per-node
// shape-gradient table is formed —
//   grad u_k = Ji^T du_k/dxi,  du_k/dxi from the field's Walsh coefficients;
//   sum_l S[k][l] gN_l(i) = sum_m (Ji S_k)[m] dN_i/dxi_m, and w Ji = w_g A
//   (A the adjugate, w = det w_g), so the viscous / diffusive test sums need
//   no reciprocal.  Equal to the reference's Gauss sums to rounding.
template <int KIND>
__device__ __forceinline__ void hex_rhs_integrate(const double (&xe)[8][3],
                                                  const double (&ue)[Out<FPB_HEX08, KIND>::NU][3],
                                                  const double (&fe)[Out<FPB_HEX08, KIND>::NF], double rho,
                                                  double mu, double kappa,
                                                  double (&acc)[Out<FPB_HEX08, KIND>::NOUT]) {
  constexpr int ET = FPB_HEX08;
  constexpr int NV = KIND == FPB_MOMENTUM_RHS || KIND == KIND_SCALAR3 ? 3 : 1;
  constexpr int NFLD = KIND == KIND_SCALAR3 ? 3 : 1;  // scalar fields sharing the geometry
  HexCoef hc;
  hex_coeffs(xe, hc);
  double uh[3][8];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double v[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) v[b] = ue[b][k];
    hex_walsh(v, uh[k]);
  }
  double fh[NFLD][8];
  if constexpr (KIND == FPB_SCALAR_RHS) hex_walsh(fe, fh[0]);
  if constexpr (KIND == KIND_SCALAR3) {  // fields fe[f * 8 + b], diffusivities (rho, mu, kappa)
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double v[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) v[b] = fe[f * 8 + b];
      hex_walsh(v, fh[f]);
    }
  }
  HexTest T[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) T[k].zero();

FPB_PRAGMA(unroll FPB_HEX_GUNROLL)
  for (int g = 0; g < 8; ++g) {
    double J[3][3];
    const double det = hex_jacobian(hc, g, J);
    double A[3][3];  // A[m][l] = det * Ji[m][l]
    A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double inv = 1.0 / det;
    const double w = det * refW<ET>(g);
    double ug[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) ug[k] = hex_value(uh[k], g);
    if constexpr (KIND == FPB_MOMENTUM_RHS) {  // _kernels.py:320-382
      double Gx[3][3], G[3][3], S[3][3], c[3];
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int k = 0; k < 3; ++k) Gx[m][k] = hex_dxi(uh[k], m, g);
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int k = 0; k < 3; ++k) G[l][k] = inv * (A[0][l] * Gx[0][k] + A[1][l] * Gx[1][k] + A[2][l] * Gx[2][k]);
      const double divu = G[0][0] + G[1][1] + G[2][2];
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int k = 0; k < 3; ++k) S[l][k] = 0.5 * (G[l][k] + G[k][l]);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double us = 0.0, gk = 0.0;
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          us += ug[l] * S[l][k];
          gk += ug[l] * G[k][l];
        }
        c[k] = 2.0 * us + divu * ug[k] - gk;
      }
      const double sv = -2.0 * mu * refW<ET>(g);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double V[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) V[m] = sv * (A[m][0] * S[k][0] + A[m][1] * S[k][1] + A[m][2] * S[k][2]);
        T[k].add(g, -w * (rho * c[k]), V);
      }
    } else {  // SCALAR_RHS (one field, or the three of KIND_SCALAR3 on one geometry), _kernels.py:420-461
#pragma unroll
      for (int f = 0; f < NFLD; ++f) {
        const double kap = KIND == KIND_SCALAR3 ? (f == 0 ? rho : f == 1 ? mu : kappa) : kappa;
        double px[3], gphi[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) px[m] = hex_dxi(fh[f], m, g);
#pragma unroll
        for (int l = 0; l < 3; ++l) gphi[l] = inv * (A[0][l] * px[0] + A[1][l] * px[1] + A[2][l] * px[2]);
        const double adv = ug[0] * gphi[0] + ug[1] * gphi[1] + ug[2] * gphi[2];
        const double sk = -kap * refW<ET>(g);
        double V[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) V[m] = sk * (A[m][0] * gphi[0] + A[m][1] * gphi[1] + A[m][2] * gphi[2]);
        T[f].add(g, -w * adv, V);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double o[8];
    T[k].finish(o);
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[b * NV + k] = o[b];
  }
}

// acc: matrices [i][j] (GRADIENT_XYZ: [k][i][j]); MOMENTUM [a][k]; SCALAR [a]
template <int ET, int KIND>
__device__ __forceinline__ void element_integrate(
    const double (&xe)[Elem<ET>::NN][Elem<ET>::DIM], const double (&ue)[Out<ET, KIND>::NU][Elem<ET>::DIM],
    const double (&fe)[Out<ET, KIND>::NF], double rho, double mu, double kappa, int kdir,
    double (&acc)[Out<ET, KIND>::NOUT]) {
  constexpr int NN = Elem<ET>::NN, NG = Elem<ET>::NG, DIM = Elem<ET>::DIM;
  constexpr int NOUT = Out<ET, KIND>::NOUT;
  constexpr bool NEED_GRAD = KIND != FPB_MASS;
  if constexpr (ET == FPB_HEX08 && (KIND == FPB_MOMENTUM_RHS || KIND == FPB_SCALAR_RHS)) {
    hex_rhs_integrate<KIND>(xe, ue, fe, rho, mu, kappa, acc);
    return;
  }
#pragma unroll
  for (int q = 0; q < NOUT; ++q) acc[q] = 0.0;

  double J[DIM][DIM], gN[DIM][NN], det = 0.0;
  HexCoef hc;
  if constexpr (ET == FPB_HEX08) hex_coeffs(xe, hc);
  if constexpr (Elem<ET>::AFFINE) {
    det = jacobian<ET>(xe, 0, J);
    if constexpr (NEED_GRAD) grad_shape<ET>(J, det, 0, gN);
  }

#pragma unroll
  for (int g = 0; g < NG; ++g) {
    if constexpr (!Elem<ET>::AFFINE) {
      if constexpr (ET == FPB_HEX08) det = hex_jacobian(hc, g, J);
      else det = jacobian<ET>(xe, g, J);
      if constexpr (NEED_GRAD) grad_shape<ET>(J, det, g, gN);
    }
    const double w = det * refW<ET>(g);  // detJw

    if constexpr (KIND == FPB_MASS) {  // _kernels.py:163-172
#pragma unroll
      for (int j = 0; j < NN; ++j)
#pragma unroll
        for (int i = 0; i < NN; ++i) acc[i * NN + j] += w * refN<ET>(j, g) * refN<ET>(i, g);
    } else if constexpr (KIND == FPB_LAPLACIAN) {  // _kernels.py:191-207
#pragma unroll
      for (int j = 0; j < NN; ++j)
#pragma unroll
        for (int i = 0; i < NN; ++i) {
          double s = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) s += gN[d][i] * gN[d][j];
          acc[i * NN + j] += w * s;
        }
    } else if constexpr (KIND == FPB_CONVECTION) {  // _kernels.py:238-266
      double ug[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < NN; ++a) s += ue[a][d] * refN<ET>(a, g);
        ug[d] = s;
      }
#pragma unroll
      for (int j = 0; j < NN; ++j) {
        double adv = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) adv += ug[d] * gN[d][j];
#pragma unroll
        for (int i = 0; i < NN; ++i) acc[i * NN + j] += w * adv * refN<ET>(i, g);
      }
    } else if constexpr (KIND == KIND_GRADIENT_K || KIND == FPB_GRADIENT_XYZ) {
      // CONVECTION with u = e_k at every node: u_g = (sum_a N_a) e_k
      // (timeloop.py:159-171)
      double sN = 0.0;
#pragma unroll
      for (int a = 0; a < NN; ++a) sN += refN<ET>(a, g);
      if constexpr (KIND == KIND_GRADIENT_K) {
#pragma unroll
        for (int j = 0; j < NN; ++j) {
          double gk = kdir == 0 ? gN[0][j] : (kdir == 1 ? gN[1][j] : gN[DIM - 1][j]);
          double adv = sN * gk;
#pragma unroll
          for (int i = 0; i < NN; ++i) acc[i * NN + j] += w * adv * refN<ET>(i, g);
        }
      } else {
#pragma unroll
        for (int k = 0; k < DIM; ++k)
#pragma unroll
          for (int j = 0; j < NN; ++j) {
            double adv = sN * gN[k][j];
#pragma unroll
            for (int i = 0; i < NN; ++i) acc[(k * NN + i) * NN + j] += w * adv * refN<ET>(i, g);
          }
      }
    } else if constexpr (KIND == FPB_MOMENTUM_RHS) {  // _kernels.py:320-382
      double ug[DIM], G[DIM][DIM], S[DIM][DIM], c[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < NN; ++a) s += ue[a][d] * refN<ET>(a, g);
        ug[d] = s;
      }
#pragma unroll
      for (int l = 0; l < DIM; ++l)
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < NN; ++a) s += ue[a][k] * gN[l][a];
          G[l][k] = s;
        }
      double divu = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) divu += G[d][d];
#pragma unroll
      for (int l = 0; l < DIM; ++l)
#pragma unroll
        for (int k = 0; k < DIM; ++k) S[l][k] = 0.5 * (G[l][k] + G[k][l]);
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        double us = 0.0, gk = 0.0;
#pragma unroll
        for (int l = 0; l < DIM; ++l) {
          us += ug[l] * S[l][k];
          gk += ug[l] * G[k][l];
        }
        c[k] = 2.0 * us + divu * ug[k] - gk;
      }
#pragma unroll
      for (int i = 0; i < NN; ++i)
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          double visc = 0.0;
#pragma unroll
          for (int l = 0; l < DIM; ++l) visc += S[k][l] * gN[l][i];
          acc[i * DIM + k] -= w * (rho * refN<ET>(i, g) * c[k] + 2.0 * mu * visc);
        }
    } else if constexpr (KIND == FPB_SCALAR_RHS) {  // _kernels.py:420-461
      double ug[DIM], gphi[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double au = 0.0, ap = 0.0;
#pragma unroll
        for (int a = 0; a < NN; ++a) {
          au += ue[a][d] * refN<ET>(a, g);
          ap += fe[a] * gN[d][a];
        }
        ug[d] = au;
        gphi[d] = ap;
      }
      double adv = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) adv += ug[d] * gphi[d];
#pragma unroll
      for (int i = 0; i < NN; ++i) {
        double diff = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) diff += gphi[d] * gN[d][i];
        acc[i] -= w * (refN<ET>(i, g) * adv + kappa * diff);
      }
    }
  }

}

}  // namespace fpb
