// Element assembly kernels: gather -> Gauss-point integration in registers ->
// FP64 scatter-add.  One warp per 32-lane pack, one thread per element, so a
// pack's connectivity row lane_conn[p][a][0:32] is one coalesced 128-byte
// load.  Per-element arithmetic follows the reference packed kernels
// (_kernels.py:150-461) term by term; nvcc contracts mul+add into DFMA, which
// changes results only at the rounding level (parity bar: 1e-12 max-normalised).
#include "elemcore.cuh"

namespace fpb {

template <int ET, int KIND>
__global__ void __launch_bounds__(128)
k_assemble(int64_t nelem, const int32_t* __restrict__ lane_conn, const double* __restrict__ coords,
           const double* __restrict__ vel, const double* __restrict__ phi, double rho, double mu,
           double kappa, const int32_t* __restrict__ pos, int64_t nnz, int kdir,
           double* __restrict__ out) {
  constexpr int NN = Elem<ET>::NN, NG = Elem<ET>::NG, DIM = Elem<ET>::DIM;
  constexpr bool MAT = KIND == FPB_MASS || KIND == FPB_LAPLACIAN || KIND == FPB_CONVECTION ||
                       KIND == KIND_GRADIENT_K;
  constexpr bool GRADXYZ = KIND == FPB_GRADIENT_XYZ;
  constexpr bool NEED_VEL = KIND == FPB_CONVECTION || KIND == FPB_MOMENTUM_RHS || KIND == FPB_SCALAR_RHS;

  const int lane = threadIdx.x & 31;
  const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t e = p * 32 + lane;
  if (e >= nelem) return;  // padded lanes contribute exact zeros: skip them

  int node[NN];
#pragma unroll
  for (int a = 0; a < NN; ++a) node[a] = __ldg(lane_conn + (p * NN + a) * 32 + lane);
  double xe[NN][DIM];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int d = 0; d < DIM; ++d) xe[a][d] = __ldg(coords + (int64_t)node[a] * DIM + d);
  double ue[Out<ET, KIND>::NU][DIM];
  if constexpr (NEED_VEL) {
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int d = 0; d < DIM; ++d) ue[a][d] = __ldg(vel + (int64_t)node[a] * DIM + d);
  }
  double fe[Out<ET, KIND>::NF];
  if constexpr (KIND == FPB_SCALAR_RHS) {
#pragma unroll
    for (int a = 0; a < NN; ++a) fe[a] = __ldg(phi + node[a]);
  }

  constexpr int NOUT = Out<ET, KIND>::NOUT;
  double acc[NOUT];
  element_integrate<ET, KIND>(xe, ue, fe, rho, mu, kappa, kdir, acc);

  // scatter-add (_kernels.py:473-519): FP64 reductions at L2
  if constexpr (MAT) {
#pragma unroll
    for (int i = 0; i < NN; ++i)
#pragma unroll
      for (int j = 0; j < NN; ++j)
        red_add(out + __ldg(pos + ((p * NN + i) * NN + j) * 32 + lane), acc[i * NN + j]);
  } else if constexpr (GRADXYZ) {
#pragma unroll
    for (int i = 0; i < NN; ++i)
#pragma unroll
      for (int j = 0; j < NN; ++j) {
        const int64_t k0 = __ldg(pos + ((p * NN + i) * NN + j) * 32 + lane);
#pragma unroll
        for (int k = 0; k < DIM; ++k) red_add(out + k * nnz + k0, acc[(k * NN + i) * NN + j]);
      }
  } else if constexpr (KIND == FPB_MOMENTUM_RHS) {
#pragma unroll
    for (int i = 0; i < NN; ++i)
#pragma unroll
      for (int k = 0; k < DIM; ++k) red_add(out + (int64_t)node[i] * DIM + k, acc[i * DIM + k]);
  } else {
#pragma unroll
    for (int i = 0; i < NN; ++i) red_add(out + node[i], acc[i]);
  }
}

template <int ET, int KIND>
static int launch(int64_t nelem, const int32_t* lane_conn, const double* coords, const double* vel,
                  const double* phi, double rho, double mu, double kappa, const int32_t* pos,
                  int64_t nnz, int kdir, double* out, cudaStream_t s) {
  int64_t npacks = (nelem + 31) / 32;
  int64_t blocks = (npacks + 3) / 4;
  k_assemble<ET, KIND><<<(unsigned)blocks, 128, 0, s>>>(nelem, lane_conn, coords, vel, phi, rho,
                                                         mu, kappa, pos, nnz, kdir, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

template <int ET>
static int dispatch_kind(int kind, int64_t nelem, const int32_t* lane_conn, const double* coords,
                         const double* vel, const double* phi, double rho, double mu, double kappa,
                         const int32_t* pos, int64_t nnz, double* out, cudaStream_t s) {
  switch (kind) {
    case FPB_MASS: return launch<ET, FPB_MASS>(nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, 0, out, s);
    case FPB_LAPLACIAN: return launch<ET, FPB_LAPLACIAN>(nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, 0, out, s);
    case FPB_CONVECTION: return launch<ET, FPB_CONVECTION>(nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, 0, out, s);
    case FPB_MOMENTUM_RHS: return launch<ET, FPB_MOMENTUM_RHS>(nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, 0, out, s);
    case FPB_SCALAR_RHS: return launch<ET, FPB_SCALAR_RHS>(nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, 0, out, s);
    case FPB_GRADIENT_XYZ:
      if constexpr (Elem<ET>::AFFINE) {
        return launch<ET, FPB_GRADIENT_XYZ>(nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, 0, out, s);
      } else {
        // three register-resident outputs would spill for 8-node elements:
        // one direction per pass
        for (int k = 0; k < Elem<ET>::DIM; ++k) {
          int rc = launch<ET, KIND_GRADIENT_K>(nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos,
                                               nnz, k, out + k * nnz, s);
          if (rc) return rc;
        }
        return FPB_OK;
      }
  }
  set_error("unknown kernel kind %d", kind);
  return FPB_ECONFIG;
}


// Element-local contributions, no scatter (assembly.py:296-380,
// assemble_element_scalar / assemble_element_packed): thread per (pack,
// lane); out[(p * NOUT + o) * vs + v] — the reference's scalar layout at
// vs = 1 ([e][i][j], [e][a][k], [e][a]) and its lane-last packed layout
// otherwise ([p][i][j][v] ...).  Padded lanes are left untouched (the caller
// zero-fills, as the reference's aligned_zeros does), matching its detJw = 0.
template <int ET, int KIND>
__global__ void __launch_bounds__(128)
k_element_local(int64_t nelem, int vs, const int32_t* __restrict__ lane_conn, const double* __restrict__ coords,
                const double* __restrict__ vel, const double* __restrict__ phi, double rho, double mu, double kappa,
                double* __restrict__ out) {
  constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM;
  constexpr bool NEED_VEL = Out<ET, KIND>::NEED_VEL;
  constexpr int NOUT = Out<ET, KIND>::NOUT;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t p = t / vs, v = t % vs;
  if (t >= nelem) return;
  int node[NN];
#pragma unroll
  for (int a = 0; a < NN; ++a) node[a] = __ldg(lane_conn + (p * NN + a) * vs + v);
  double xe[NN][DIM];
#pragma unroll
  for (int a = 0; a < NN; ++a)
#pragma unroll
    for (int d = 0; d < DIM; ++d) xe[a][d] = __ldg(coords + (int64_t)node[a] * DIM + d);
  double ue[Out<ET, KIND>::NU][DIM];
  if constexpr (NEED_VEL) {
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int d = 0; d < DIM; ++d) ue[a][d] = __ldg(vel + (int64_t)node[a] * DIM + d);
  }
  double fe[Out<ET, KIND>::NF];
  if constexpr (KIND == FPB_SCALAR_RHS) {
#pragma unroll
    for (int a = 0; a < NN; ++a) fe[a] = __ldg(phi + node[a]);
  }
  double acc[NOUT];
  element_integrate<ET, KIND>(xe, ue, fe, rho, mu, kappa, 0, acc);
#pragma unroll
  for (int o = 0; o < NOUT; ++o) out[(p * NOUT + o) * vs + v] = acc[o];
}

template <int ET>
static int element_local_kind(int kind, int64_t nelem, int vs, const int32_t* lane_conn, const double* coords,
                              const double* vel, const double* phi, double rho, double mu, double kappa, double* out,
                              cudaStream_t s) {
  const unsigned grid = (unsigned)((nelem + 127) / 128);
#define FPB_EL(K)                                                                                          \
  k_element_local<ET, K><<<grid, 128, 0, s>>>(nelem, vs, lane_conn, coords, vel, phi, rho, mu, kappa, out); \
  break
  switch (kind) {
    case FPB_MASS: FPB_EL(FPB_MASS);
    case FPB_LAPLACIAN: FPB_EL(FPB_LAPLACIAN);
    case FPB_CONVECTION: FPB_EL(FPB_CONVECTION);
    case FPB_MOMENTUM_RHS: FPB_EL(FPB_MOMENTUM_RHS);
    case FPB_SCALAR_RHS: FPB_EL(FPB_SCALAR_RHS);
    default:
      set_error("element-local assembly covers the reference's five kinds (got %d)", kind);
      return FPB_ECONFIG;
  }
#undef FPB_EL
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

}  // namespace fpb

using namespace fpb;

extern "C" int fpb_assemble(int kind, int etype, int64_t nelem, const int32_t* lane_conn,
                            const double* coords, const double* vel, const double* phi,
                            double rho, double mu, double kappa, const int32_t* pos, int64_t nnz,
                            double* out, void* stream) {
  FPB_REQUIRE(etype >= 0 && etype < 5 && g_ref_loaded[etype],
              "reference tables for element type %d not uploaded", etype);
  FPB_REQUIRE(kind >= 0 && kind <= FPB_GRADIENT_XYZ, "unknown kernel kind %d", kind);
  bool mat = kind == FPB_MASS || kind == FPB_LAPLACIAN || kind == FPB_CONVECTION || kind == FPB_GRADIENT_XYZ;
  FPB_REQUIRE(!mat || pos != nullptr, "matrix kinds need the element->CSR map");
  FPB_REQUIRE(!(kind == FPB_CONVECTION || kind == FPB_MOMENTUM_RHS || kind == FPB_SCALAR_RHS) || vel,
              "kind %d needs a velocity field", kind);
  FPB_REQUIRE(kind != FPB_SCALAR_RHS || phi, "SCALAR_RHS needs a scalar field");
  if (nelem == 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  switch (etype) {
    case FPB_TRI03: return dispatch_kind<FPB_TRI03>(kind, nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, out, s);
    case FPB_QUAD04: return dispatch_kind<FPB_QUAD04>(kind, nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, out, s);
    case FPB_TET04: return dispatch_kind<FPB_TET04>(kind, nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, out, s);
    case FPB_PYR05: return dispatch_kind<FPB_PYR05>(kind, nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, out, s);
    case FPB_HEX08: return dispatch_kind<FPB_HEX08>(kind, nelem, lane_conn, coords, vel, phi, rho, mu, kappa, pos, nnz, out, s);
  }
  return FPB_ECONFIG;
}

extern "C" int fpb_assemble_elements(int kind, int etype, int64_t nelem, int vs, const int32_t* lane_conn,
                                     const double* coords, const double* vel, const double* phi, double rho,
                                     double mu, double kappa, double* out, void* stream) {
  FPB_REQUIRE(etype >= 0 && etype < 5 && g_ref_loaded[etype],
              "reference tables for element type %d not uploaded", etype);
  FPB_REQUIRE(vs >= 1 && vs <= 32, "vector size %d out of range", vs);
  FPB_REQUIRE(!(kind == FPB_CONVECTION || kind == FPB_MOMENTUM_RHS || kind == FPB_SCALAR_RHS) || vel,
              "kind %d needs a velocity field", kind);
  FPB_REQUIRE(kind != FPB_SCALAR_RHS || phi, "SCALAR_RHS needs a scalar field");
  if (nelem == 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  switch (etype) {
    case FPB_TRI03: return element_local_kind<FPB_TRI03>(kind, nelem, vs, lane_conn, coords, vel, phi, rho, mu, kappa, out, s);
    case FPB_QUAD04: return element_local_kind<FPB_QUAD04>(kind, nelem, vs, lane_conn, coords, vel, phi, rho, mu, kappa, out, s);
    case FPB_TET04: return element_local_kind<FPB_TET04>(kind, nelem, vs, lane_conn, coords, vel, phi, rho, mu, kappa, out, s);
    case FPB_PYR05: return element_local_kind<FPB_PYR05>(kind, nelem, vs, lane_conn, coords, vel, phi, rho, mu, kappa, out, s);
    default: return element_local_kind<FPB_HEX08>(kind, nelem, vs, lane_conn, coords, vel, phi, rho, mu, kappa, out, s);
  }
}
