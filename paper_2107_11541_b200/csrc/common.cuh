// Shared definitions of the fempack_b200 CUDA library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/fempack_b200.h"

namespace fpb {

// ---- error plumbing (fpb_last_error) ------------------------------------
void set_error(const char* fmt, ...);

#define FPB_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      ::fpb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      return FPB_ECUDA;                                                             \
    }                                                                               \
  } while (0)

#define FPB_LAUNCH_CHECK() FPB_CUDA(cudaGetLastError())

#define FPB_REQUIRE(cond, ...)   \
  do {                           \
    if (!(cond)) {               \
      ::fpb::set_error(__VA_ARGS__); \
      return FPB_ECONFIG;        \
    }                            \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;  // B200; grids are sized in multiples of this

// ---- element traits -------------------------------------------------------
// NN nodes, NG Gauss points, DIM; AFFINE: dN is constant over Gauss points
// (TRI03/TET04, elements.py:118-145), so J, det and gradN are identical at
// every point and are computed once — bit-identical to recomputing them.
template <int ET> struct Elem;
template <> struct Elem<FPB_TRI03> { static constexpr int NN = 3, NG = 3, DIM = 2; static constexpr bool AFFINE = true; };
template <> struct Elem<FPB_QUAD04> { static constexpr int NN = 4, NG = 4, DIM = 2; static constexpr bool AFFINE = false; };
template <> struct Elem<FPB_TET04> { static constexpr int NN = 4, NG = 4, DIM = 3; static constexpr bool AFFINE = true; };
template <> struct Elem<FPB_PYR05> { static constexpr int NN = 5, NG = 8, DIM = 3; static constexpr bool AFFINE = false; };
template <> struct Elem<FPB_HEX08> { static constexpr int NN = 8, NG = 8, DIM = 3; static constexpr bool AFFINE = false; };

inline int etype_nn(int et) { const int t[5] = {3, 4, 4, 5, 8}; return (et >= 0 && et < 5) ? t[et] : 0; }
inline int etype_ng(int et) { const int t[5] = {3, 4, 4, 8, 8}; return (et >= 0 && et < 5) ? t[et] : 0; }
inline int etype_dim(int et) { const int t[5] = {2, 2, 3, 3, 3}; return (et >= 0 && et < 5) ? t[et] : 0; }

// Reference tables in constant memory, uploaded once by
// fpb_set_reference_element.  Layouts follow elements.py: N[a][g],
// dN[l][a][g], w[g]; with every loop fully unrolled the indices are
// compile-time constants and the values become constant-bank operands.
struct RefTables {
  double N[8 * 8];
  double dN[3 * 8 * 8];
  double w[8];
  // derived once on the host from N and w (fpb_set_reference_element), used
  // by the closed-form affine-simplex kernels (rows.cu):
  double M[8 * 8];  // M[a][b] = sum_g w_g N_b(g) N_a(g)        (mass integrand / det)
  double mN[8];     // mN[a]   = sum_g w_g (sum_c N_c(g)) N_a(g) (unit-velocity convection)
  double W;         // sum_g w_g
};
extern __constant__ RefTables c_ref[5];
extern bool g_ref_loaded[5];

template <int ET> __device__ __forceinline__ double refN(int a, int g) {
  return c_ref[ET].N[a * Elem<ET>::NG + g];
}
template <int ET> __device__ __forceinline__ double refdN(int l, int a, int g) {
  return c_ref[ET].dN[(l * Elem<ET>::NN + a) * Elem<ET>::NG + g];
}
template <int ET> __device__ __forceinline__ double refW(int g) { return c_ref[ET].w[g]; }
template <int ET> __device__ __forceinline__ double refM(int a, int b) {
  return c_ref[ET].M[a * Elem<ET>::NN + b];
}
template <int ET> __device__ __forceinline__ double refmN(int a) { return c_ref[ET].mN[a]; }
template <int ET> __device__ __forceinline__ double refWsum() { return c_ref[ET].W; }

// ---- geometry -------------------------------------------------------------
// J[d][l] = sum_a x[a][d] dN[l][a][g]; det; gradN[d][a] = sum_l Ji[l][d] dN[l][a][g]
// (_kernels.py:88-146).  Returns det.
template <int ET>
__device__ __forceinline__ double jacobian(const double (&xe)[Elem<ET>::NN][Elem<ET>::DIM], int g,
                                           double (&J)[Elem<ET>::DIM][Elem<ET>::DIM]) {
  constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM;
#pragma unroll
  for (int d = 0; d < DIM; ++d)
#pragma unroll
    for (int l = 0; l < DIM; ++l) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < NN; ++a) acc += xe[a][d] * refdN<ET>(l, a, g);
      J[d][l] = acc;
    }
  if constexpr (DIM == 2) {
    return J[0][0] * J[1][1] - J[0][1] * J[1][0];
  } else {
    return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  }
}

// Q1 hexahedron, sum-factorised Jacobian.  With the reference's corner order
// (elements.py: a = (-,-,-), (+,-,-), (+,+,-), (-,+,-), then z = +1) and Gauss
// points g = 4 iz + 2 iy + ix at -+1/sqrt(3), dx/dxi is bilinear in the two
// transverse coordinates:
//   J[d][0] = A_x + A_xy eta + A_xz zeta + A_xyz eta zeta,
//   J[d][1] = A_y + A_xy xi  + A_yz zeta + A_xyz xi zeta,
//   J[d][2] = A_z + A_xz xi  + A_yz eta  + A_xyz xi eta,
// with A_m = (1/8) sum_a m(corner a) x_a[d] (a 20-add butterfly per d), so
// J costs 3 FMA per entry instead of 8 — equal to sum_a x_a dN_a to rounding.
struct HexCoef {
  double A[7][3];  // x, y, z, xy, xz, yz, xyz
};

__device__ __forceinline__ void hex_coeffs(const double (&x)[8][3], HexCoef& h) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    // pairs along x for (y, z) = (-,-), (+,-), (-,+), (+,+): corners (0,1), (3,2), (4,5), (7,6)
    const double t1 = x[1][d] - x[0][d], t2 = x[2][d] - x[3][d], t3 = x[5][d] - x[4][d], t4 = x[6][d] - x[7][d];
    const double s1 = x[1][d] + x[0][d], s2 = x[2][d] + x[3][d], s3 = x[5][d] + x[4][d], s4 = x[6][d] + x[7][d];
    h.A[0][d] = 0.125 * ((t1 + t2) + (t3 + t4));
    h.A[3][d] = 0.125 * ((t2 - t1) + (t4 - t3));
    h.A[4][d] = 0.125 * ((t3 + t4) - (t1 + t2));
    h.A[6][d] = 0.125 * ((t1 - t2) + (t4 - t3));
    h.A[1][d] = 0.125 * ((s2 - s1) + (s4 - s3));
    h.A[2][d] = 0.125 * ((s3 + s4) - (s1 + s2));
    h.A[5][d] = 0.125 * ((s1 - s2) + (s4 - s3));
  }
}

// J at Gauss point g (compile-time after unrolling); returns det
__device__ __forceinline__ double hex_jacobian(const HexCoef& h, int g, double (&J)[3][3]) {
  constexpr double q = 0.5773502691896258;  // 1 / sqrt(3), as elements.py
  const double xi = (g & 1) ? q : -q, eta = (g & 2) ? q : -q, zeta = (g & 4) ? q : -q;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    J[d][0] = h.A[0][d] + h.A[3][d] * eta + h.A[4][d] * zeta + h.A[6][d] * (eta * zeta);
    J[d][1] = h.A[1][d] + h.A[3][d] * xi + h.A[5][d] * zeta + h.A[6][d] * (xi * zeta);
    J[d][2] = h.A[2][d] + h.A[4][d] * xi + h.A[5][d] * eta + h.A[6][d] * (xi * eta);
  }
  return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

// Q1 hexahedron, Walsh (sign-product) forms on the 2x2x2 Gauss rule
// (elements.py:148-166 corners, :226-229 points).  U is a bitmask of
// directions (1 = xi, 2 = eta, 4 = zeta); corner b has signs s_d(b),
// Gauss point g has x_d(g) = (bit d of g) ? q : -q.  With
// mono(U, g) = prod_{d in U} x_d(g) and s_U(b) = prod_{d in U} s_d(b):
//   nodal field  v(xi) = 1/8 sum_U h8[U] mono(U, xi),  h8 = hex_walsh(v)
//   N_b(g)          = 1/8 sum_U s_U(b) mono(U, g)
//   dN_b/dxi_m (g)  = 1/8 sum_{U ∋ m} s_U(b) mono(U \ m, g)
// so point values, reference-space derivatives and the test-function sums
// sum_g (W_g N_b + sum_m V_g[m] dN_b/dxi_m) all go through 8 coefficients:
// 8 FMA per value or point instead of 8 per (node, point) and direction.
// corner b -> p with bit d of p = (s_d(b) > 0): 0 1 3 2 4 5 7 6
__host__ __device__ constexpr int hex_corner_p(int b) { return b ^ ((b >> 1) & 1); }

__host__ __device__ constexpr double hex_mono(int U, int g) {
  constexpr double q = 0.5773502691896258;
  double r = 1.0;
  for (int d = 0; d < 3; ++d)
    if ((U >> d) & 1) r *= ((g >> d) & 1) ? q : -q;
  return r;
}

// h8[U] = sum_b s_U(b) v_b (8x the Walsh coefficient): 24 adds
__device__ __forceinline__ void hex_walsh(const double (&v)[8], double (&h8)[8]) {
#pragma unroll
  for (int b = 0; b < 8; ++b) h8[hex_corner_p(b)] = v[b];
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int p = 0; p < 8; ++p)
      if (!((p >> d) & 1)) {
        const double lo = h8[p], hi = h8[p | (1 << d)];
        h8[p] = lo + hi;
        h8[p | (1 << d)] = hi - lo;
      }
}

// v(g) and dv/dxi_m(g) from h8 (g compile-time after unrolling)
__device__ __forceinline__ double hex_value(const double (&h8)[8], int g) {
  double r = 0.0;
#pragma unroll
  for (int U = 0; U < 8; ++U) r = fma(0.125 * hex_mono(U, g), h8[U], r);
  return r;
}
__device__ __forceinline__ double hex_dxi(const double (&h8)[8], int m, int g) {
  double r = 0.0;
#pragma unroll
  for (int U = 0; U < 8; ++U)
    if ((U >> m) & 1) r = fma(0.125 * hex_mono(U & ~(1 << m), g), h8[U], r);
  return r;
}

// test-function sums R_b = sum_g (W_g N_b(g) + sum_m V_g[m] dN_b/dxi_m(g))
struct HexTest {
  double R[8];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int U = 0; U < 8; ++U) R[U] = 0.0;
  }
  __device__ __forceinline__ void add(int g, double W, const double (&V)[3]) {
#pragma unroll
    for (int U = 0; U < 8; ++U) {
      double r = fma(0.125 * hex_mono(U, g), W, R[U]);
#pragma unroll
      for (int m = 0; m < 3; ++m)
        if ((U >> m) & 1) r = fma(0.125 * hex_mono(U & ~(1 << m), g), V[m], r);
      R[U] = r;
    }
  }
  // out[b] = sum_U s_U(b) R[U]: 24 adds
  __device__ __forceinline__ void finish(double (&out)[8]) {
    double t[8];
#pragma unroll
    for (int U = 0; U < 8; ++U) t[U] = R[U];
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (!((p >> d) & 1)) {
          const double lo = t[p], hi = t[p | (1 << d)];
          t[p] = lo - hi;
          t[p | (1 << d)] = lo + hi;
        }
#pragma unroll
    for (int b = 0; b < 8; ++b) out[b] = t[hex_corner_p(b)];
  }
};

template <int ET>
__device__ __forceinline__ void grad_shape(const double (&J)[Elem<ET>::DIM][Elem<ET>::DIM], double det,
                                           int g, double (&gN)[Elem<ET>::DIM][Elem<ET>::NN]) {
  constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM;
  double Ji[DIM][DIM];
  const double inv = 1.0 / det;
  if constexpr (DIM == 2) {
    Ji[0][0] = J[1][1] * inv;
    Ji[0][1] = -J[0][1] * inv;
    Ji[1][0] = -J[1][0] * inv;
    Ji[1][1] = J[0][0] * inv;
  } else {
    Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * inv;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * inv;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * inv;
    Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * inv;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * inv;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * inv;
    Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * inv;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * inv;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * inv;
  }
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < DIM; ++l) acc += Ji[l][d] * refdN<ET>(l, a, g);
      gN[d][a] = acc;
    }
}

// ---- misc -------------------------------------------------------------------
// one 256-bit read-only load (sm_100a: LDG.E.ENL2.256) of a 32-byte record
__device__ __forceinline__ void ld256(const double* p, double (&r)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
               : "l"(p));
}

__device__ __forceinline__ void red_add(double* p, double v) { atomicAdd(p, v); }

inline int grid_for(int64_t work, int block, int per_sm = 16) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = (int64_t)kNumSMs * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace fpb
