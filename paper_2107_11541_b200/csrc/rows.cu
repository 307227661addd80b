// Row-owned ("node-gather") assembly for affine simplices (TRI03, TET04).
//
// The element-scatter formulation (assemble.cu) issues one FP64 reduction
// per (element, i, j) — 16 per tet per matrix — and is bound by L2 atomic
// throughput.  Here every CSR row / mesh node is owned by one thread, which
// walks the elements incident to its node in ascending element order,
// recomputes each element's geometry in registers (affine: one Jacobian per
// element, ~60 flops) and adds the element's row contribution in closed
// form.  Outputs are written once — no atomics, no zero-fill pass, and the
// summation order is fixed, so results are bitwise reproducible run to run.
//
// Incidence lists are stored SELL-32 ("sliced ELLPACK", the paper's SIMD
// packing applied to the node side): rows are grouped in slices of 32
// consecutive rows, slice s holds width_s columns of 32 element ids, entry
// (s, m, lane) = m-th incident element of row 32 s + lane, so every load of
// the hot loop is one coalesced 128-byte row.  For matrices a parallel
// SELL-32 array holds, per incidence, the 8-bit offsets of the element's
// nodes within the row's column list (the row-local form of the reference's
// element->CSR map, assembly.py:44-52).
//
// Closed forms (affine: gradN and detJ constant per element; the reference
// quadrature is exact for these integrands, so they agree to rounding with
// _kernels.py's Gauss loops — parity bar 1e-12):
//   MASS        A[a][b] = det M[a][b],             M[a][b] = sum_g w_g N_b N_a
//   LAPLACIAN   A[a][b] = det W gN_a . gN_b,       W = sum_g w_g
//   CONVECTION  A[a][b] = det (sum_c M[a][c] u_c) . gN_b
//   GRADIENT_k  A[a][b] = det mN[a] gN_b[k],       mN[a] = sum_g w_g (sum_c N_c) N_a
//   MOMENTUM    r_a = -det (rho ubar_a . Mc + 2 mu W S gN_a),
//               ubar_a = sum_c M[a][c] u_c, Mc = 2S + div(u) I - G^T
//   SCALAR      r_a = -det (ubar_a . gphi + kappa W gphi . gN_a)
#include <cub/device/device_scan.cuh>

#include <cstring>

#include "simplex.cuh"

namespace fpb {

constexpr int kRowsBlock = 128;
#ifndef FPB_ROWS_MINB
#define FPB_ROWS_MINB 4  // matrix kinds: CTAs per SM the register budget is sized for
#endif
constexpr int kOwnerSpan = 256;  // write-out chunk of a warp's CSR range (bytes of owner map)
int g_tuning_rows_nb = 1;         // fpb_set_tuning("rows_nb", 0|1): neighbour-staged matrix kernel
extern int g_tuning_hex_canon_rows;  // hexblock.cu
extern int g_tuning_blk_pipe;
extern int g_tuning_kmom_smem_kb;    // kmom.cu
extern int g_tuning_kgrad_march;     // pairs.cu
extern int g_tuning_kgrad_kchunk;    // pairs.cu
extern int g_tuning_kgrad_bthreads;  // pairs.cu


template <int ET, int KIND>
__global__ void __launch_bounds__(kRowsBlock, (KIND == FPB_MOMENTUM_RHS || KIND == FPB_SCALAR_RHS) ? 1 : (KIND == FPB_CONVECTION ? 4 : FPB_ROWS_MINB))
k_rows(int32_t n, int32_t row0, const int32_t* __restrict__ slice_ptr, const int4* __restrict__ incn,
       const uint32_t* __restrict__ slots, const double* __restrict__ xyz4,
       const double* __restrict__ uvw4, double rho, double mu, double kappa,
       const int32_t* __restrict__ rowptr, int64_t nnz, int rowcap, int accumulate,
       double* __restrict__ out) {
  constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM;
  constexpr bool MAT = KIND == FPB_MASS || KIND == FPB_LAPLACIAN || KIND == FPB_CONVECTION ||
                       KIND == FPB_GRADIENT_XYZ;
  constexpr int NMAT = KIND == FPB_GRADIENT_XYZ ? DIM : 1;
  constexpr bool NEED_VEL = KIND == FPB_CONVECTION || KIND == FPB_MOMENTUM_RHS || KIND == FPB_SCALAR_RHS;
  constexpr int NACC = KIND == FPB_MOMENTUM_RHS ? DIM : (MAT ? NMAT : 1);
  // MASS / CONVECTION / GRADIENT are linear in det*gN: adjugate form, no
  // reciprocal (gN then holds det*gN and det_s is 1)
  constexpr bool ADJ = KIND == FPB_MASS || KIND == FPB_CONVECTION || KIND == FPB_GRADIENT_XYZ;
  // off-diagonal accumulators [NMAT][rowcap-1][kRowsBlock]; the diagonal
  // entry (local node 0 of every record) lives in registers
  extern __shared__ double sacc[];

  const int tid = threadIdx.x;
  const int row = row0 + blockIdx.x * kRowsBlock + tid;  // rows [row0, n), row0 % 32 == 0
  // matrix kinds keep every lane alive for the warp-cooperative write-out;
  // rows past n get an empty incidence range
  if (!MAT && row >= n) return;
  const bool live = row < n;
  const int lane = row & 31;
  const int m0 = live ? __ldg(slice_ptr + (row >> 5)) : 0;
  const int m1 = live ? __ldg(slice_ptr + (row >> 5) + 1) : 0;

  int rlo = 0, rlen = 0;
  if constexpr (MAT) {
    if (live) {
      rlo = __ldg(rowptr + row);
      rlen = __ldg(rowptr + row + 1) - rlo;
    }
    for (int r = 0; r + 1 < rlen; ++r)
#pragma unroll
      for (int k = 0; k < NMAT; ++k) sacc[(r * NMAT + k) * kRowsBlock + tid] = 0.0;
  }
  double acc[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q] = 0.0;
  const double W = refWsum<ET>();

  // Records are rotated at setup (fpb_incidence_nodes) so the row's own node
  // is local node 0 (even permutation: orientation and det unchanged); its
  // data are loaded once per row.  Node data are 32-byte records read with
  // one 256-bit load each: xyz4[n] = (x, y, z|0, 0), uvw4[n] = (u, v, w|0, phi).
  //
  // Software pipeline without register rotation: two buffer sets alternate
  // roles (the loop body is unrolled by two), so a load's destination is not
  // read until its consumer step.  Step m integrates set m&1 while the
  // nodes of m+1 (other set) and the ids / slot bytes of m+2 (this set,
  // after use) are in flight.
  constexpr int NU = NEED_VEL ? NN : 1;
  constexpr int NF = KIND == FPB_SCALAR_RHS ? NN : 1;
  struct Stage {
    int c[4];
    uint32_t sl;
    double x[NN][DIM], u[NU][DIM], f[NF];
  };
  auto ld_c = [&](int mm, Stage& S) {
    if (mm < m1) {
      if constexpr (MAT) S.sl = __ldg(slots + (int64_t)mm * 32 + lane);
      const int4 c4 = __ldg(incn + (int64_t)mm * 32 + lane);
      S.c[0] = c4.x; S.c[1] = c4.y; S.c[2] = c4.z; S.c[3] = c4.w;
    } else {
      S.c[0] = -1;
    }
  };
  auto ld_node = [&](int node, double (&x)[DIM], double (&u)[DIM], double& f) {
    double r[4];
    ld256(xyz4 + 4 * (int64_t)node, r);
#pragma unroll
    for (int d = 0; d < DIM; ++d) x[d] = r[d];
    if constexpr (NEED_VEL) {
      ld256(uvw4 + 4 * (int64_t)node, r);
#pragma unroll
      for (int d = 0; d < DIM; ++d) u[d] = r[d];
      f = r[3];
    }
  };
  auto ld_x = [&](Stage& S) {
    if (S.c[0] < 0) return;
#pragma unroll
    for (int b = 1; b < NN; ++b) {
      double fu = 0.0;
      ld_node(S.c[b], S.x[b], S.u[NEED_VEL ? b : 0], fu);
      if constexpr (KIND == FPB_SCALAR_RHS) S.f[b] = fu;
    }
  };
  // row node (local node 0 of every record)
  double x0[DIM] = {}, u0[DIM] = {}, f0 = 0.0;
  if (live) ld_node(row, x0, u0, f0);

  // row 0 of the reference tables (local node 0 is the row node)
  double M0[NN];
#pragma unroll
  for (int b = 0; b < NN; ++b) M0[b] = refM<ET>(0, b);
  const double mN0 = refmN<ET>(0);

  auto step = [&](Stage& S) {
    const uint32_t sl = S.sl;
    double xe[NN][DIM], ue[NU][DIM], fe[NF];
#pragma unroll
    for (int d = 0; d < DIM; ++d) xe[0][d] = x0[d];
#pragma unroll
    for (int b = 1; b < NN; ++b)
#pragma unroll
      for (int d = 0; d < DIM; ++d) xe[b][d] = S.x[b][d];
    if constexpr (NEED_VEL) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) ue[0][d] = u0[d];
#pragma unroll
      for (int b = 1; b < NN; ++b)
#pragma unroll
        for (int d = 0; d < DIM; ++d) ue[b][d] = S.u[b][d];
    }
    if constexpr (KIND == FPB_SCALAR_RHS) {
      fe[0] = f0;
#pragma unroll
      for (int b = 1; b < NN; ++b) fe[b] = S.f[b];
    }
    (void)fe;
    (void)ue;
    double gN[DIM][NN];
    const double det = ADJ ? simplex_adj<ET>(xe, gN) : simplex_geometry<ET>(xe, gN);
    const double det_s = ADJ ? 1.0 : det;

    double ubar[DIM];
    if constexpr (NEED_VEL) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < NN; ++b) s += M0[b] * ue[b][d];
        ubar[d] = s;
      }
    }

    if constexpr (MAT) {
      double val[NMAT][NN];
      if constexpr (KIND == FPB_MASS) {
#pragma unroll
        for (int b = 0; b < NN; ++b) val[0][b] = det * M0[b];
      } else if constexpr (KIND == FPB_LAPLACIAN) {
        const double dw = det * W;
#pragma unroll
        for (int b = 0; b < NN; ++b) {
          double s = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) s += gN[d][0] * gN[d][b];
          val[0][b] = dw * s;
        }
      } else if constexpr (KIND == FPB_CONVECTION) {
#pragma unroll
        for (int b = 0; b < NN; ++b) {
          double s = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) s += ubar[d] * gN[d][b];
          val[0][b] = det_s * s;
        }
      } else {  // GRADIENT_XYZ
        const double f = det_s * mN0;
#pragma unroll
        for (int k = 0; k < NMAT; ++k)
#pragma unroll
          for (int b = 0; b < NN; ++b) val[k][b] = f * gN[k][b];
      }
#pragma unroll
      for (int k = 0; k < NMAT; ++k) acc[k] += val[k][0];
      // off-diagonal columns are distinct, so all loads are issued before the
      // stores (the compiler cannot prove the slots differ and would
      // otherwise serialise the read-modify-writes)
      double* p[NN];
      double old[NN][NMAT];
#pragma unroll
      for (int b = 1; b < NN; ++b) {
        const int s = (sl >> (8 * b)) & 0xff;  // off-diagonal index (diagonal skipped)
        p[b] = sacc + s * (NMAT * kRowsBlock) + tid;
#pragma unroll
        for (int k = 0; k < NMAT; ++k) old[b][k] = p[b][k * kRowsBlock];
      }
#pragma unroll
      for (int b = 1; b < NN; ++b)
#pragma unroll
        for (int k = 0; k < NMAT; ++k) p[b][k * kRowsBlock] = old[b][k] + val[k][b];
    } else if constexpr (KIND == FPB_MOMENTUM_RHS) {
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
      const double dw2mu = 2.0 * mu * det * W, drho = rho * det;
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        double conv = 0.0, visc = 0.0;
#pragma unroll
        for (int l = 0; l < DIM; ++l) {
          const double S_lk = 0.5 * (G[l][k] + G[k][l]);
          const double Mc = 2.0 * S_lk + (l == k ? divu : 0.0) - G[k][l];
          conv += ubar[l] * Mc;
          visc += S_lk * gN[l][0];
        }
        acc[k] -= drho * conv + dw2mu * visc;
      }
    } else {  // SCALAR_RHS
      double gphi[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < NN; ++b) s += fe[b] * gN[d][b];
        gphi[d] = s;
      }
      double adv = 0.0, diff = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        adv += ubar[d] * gphi[d];
        diff += gphi[d] * gN[d][0];
      }
      acc[0] -= det * adv + kappa * det * W * diff;
    }
  };

  Stage SA, SB;
  SA.sl = SB.sl = 0;
  ld_c(m0, SA);
  ld_c(m0 + 1, SB);
  ld_x(SA);
  int dslot = rlen - 1;  // diagonal position in the row (slot byte 0)
  if constexpr (MAT) {
    if (m0 < m1 && SA.c[0] >= 0) dslot = SA.sl & 0xff;
  }
  for (int m = m0; m < m1; m += 2) {
    if (SA.c[0] < 0) break;  // row lists are padded at the end
    ld_x(SB);
    step(SA);
    ld_c(m + 2, SA);
    if (SB.c[0] < 0) break;
    ld_x(SA);
    step(SB);
    ld_c(m + 3, SB);
  }

  if constexpr (MAT) {
    // Warp-cooperative, coalesced write-out: the warp's 32 consecutive rows
    // are one contiguous CSR range [base, base + span).  Each lane marks its
    // row's positions with its lane id in a per-warp byte map, then lane l
    // writes positions base + l, base + l + 32, ... taking the value from
    // the owner's accumulators (shared memory) or diagonal (shuffle).
    __shared__ uint8_t owner_map[kRowsBlock / 32][kOwnerSpan];
    uint8_t* om = owner_map[tid >> 5];
    const int wlane = tid & 31;
    const int base = __shfl_sync(0xffffffffu, rlo, 0);
    int wend = live ? rlo + rlen : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wend = max(wend, __shfl_xor_sync(0xffffffffu, wend, o));
    const int span = wend - base;
    const int dpos = rlo + dslot;
    for (int c0 = 0; c0 < span; c0 += kOwnerSpan) {
      const int c1 = min(span, c0 + kOwnerSpan);
      for (int q = max(rlo - base, c0); q < min(rlo - base + rlen, c1); ++q) om[q - c0] = (uint8_t)wlane;
      __syncwarp();
      for (int q = c0 + wlane; q < c0 + ((c1 - c0 + 31) & ~31); q += 32) {
        const bool ok = q < c1;
        const int own = ok ? om[q - c0] : wlane;
        const int own_rlo = __shfl_sync(0xffffffffu, rlo, own);
        const int own_d = __shfl_sync(0xffffffffu, dpos, own);
        const int pos = base + q;
        const int r = pos - own_rlo;
        const int sidx = max(0, min(r - (pos > own_d), rowcap - 2));
        const double* src = sacc + sidx * (NMAT * kRowsBlock) + (tid & ~31) + own;
#pragma unroll
        for (int k = 0; k < NMAT; ++k) {
          const double dg = __shfl_sync(0xffffffffu, acc[k], own);
          if (ok) {
            const double v = pos == own_d ? dg : src[k * kRowsBlock];
            double* o = out + k * nnz + pos;
            *o = accumulate ? *o + v : v;
          }
        }
      }
      __syncwarp();
    }
  } else {
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      double* o = out + (int64_t)row * NACC + q;
      *o = accumulate ? *o + acc[q] : acc[q];
    }
  }
}

// ---- neighbour-staged row kernel (matrix kinds) --------------------------------
// The row's column list IS the set of nodes its incident elements touch, so
// each thread first stages its neighbours' records in shared memory (one
// gather per distinct neighbour instead of one per (element, node)), then
// walks its incidences reading nothing from global memory but the 32-bit
// slot word: byte b (b = 1..NN-1) is the off-diagonal index s of rotated
// record node b, which addresses both the staged neighbour record and the
// accumulator of column s.  Shared memory per thread, per off-diagonal
// slot: DIM coordinates (+ DIM velocities for CONVECTION) + NMAT sums, laid
// out [s][field][thread] so every access is conflict-free.
#ifndef FPB_NB_BLOCK
#define FPB_NB_BLOCK 32  // one warp per CTA: finest occupancy granularity (measured best)
#endif
#ifndef FPB_NB_W
#define FPB_NB_W 8
#endif
#ifndef FPB_NB_MINB
#define FPB_NB_MINB 1
#endif
constexpr int kNbBlock = FPB_NB_BLOCK;

template <int ET, int KIND>
struct NbLayout {
  static constexpr int DIM = Elem<ET>::DIM;
  static constexpr int NMAT = KIND == FPB_GRADIENT_XYZ ? DIM : 1;
  static constexpr int NV = KIND == FPB_CONVECTION ? DIM : 0;
  static constexpr int FIELDS = DIM + NV + NMAT;  // doubles per (slot, thread)
  static constexpr int OX = 0, OU = DIM, OA = DIM + NV;
};

template <int ET, int KIND>
__global__ void __launch_bounds__(kNbBlock, FPB_NB_MINB)
k_rows_nb(int32_t n, int32_t row0, const int32_t* __restrict__ slice_ptr, const uint32_t* __restrict__ slots,
          const double* __restrict__ xyz4, const double* __restrict__ uvw4,
          const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind, int64_t nnz, int rowcap,
          int accumulate, double* __restrict__ out) {
  using L = NbLayout<ET, KIND>;
  constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM, NMAT = L::NMAT, F = L::FIELDS;
  constexpr bool VEL = L::NV > 0;
  constexpr int SS = F * kNbBlock;  // doubles per off-diagonal slot
  extern __shared__ double sm[];

  const int tid = threadIdx.x;
  const int row = row0 + blockIdx.x * kNbBlock + tid;  // rows [row0, n), row0 % 32 == 0
  const bool live = row < n;
  const int lane = row & 31;
  const int m0 = live ? __ldg(slice_ptr + (row >> 5)) : 0;
  const int m1 = live ? __ldg(slice_ptr + (row >> 5) + 1) : 0;
  int rlo = 0, rlen = 0;
  if (live) {
    rlo = __ldg(rowptr + row);
    rlen = __ldg(rowptr + row + 1) - rlo;
  }
  double* const my = sm + tid;

  // ---- stage the neighbours (and find the diagonal) ----
  // batches of kStage columns: all gathers of a batch are in flight before
  // the first shared-memory store
  constexpr int kStage = 8;
  double x0[DIM] = {}, u0[DIM] = {};
  int dslot = rlen - 1;
  {
    int s = 0;
    for (int r0 = 0; r0 < rlen; r0 += kStage) {
      int col[kStage];
      double rx[kStage][4], ru[kStage][4];
#pragma unroll
      for (int j = 0; j < kStage; ++j) col[j] = r0 + j < rlen ? __ldg(colind + rlo + r0 + j) : -1;
#pragma unroll
      for (int j = 0; j < kStage; ++j) {
        if (col[j] >= 0) {
          ld256(xyz4 + 4 * (int64_t)col[j], rx[j]);
          if constexpr (VEL) ld256(uvw4 + 4 * (int64_t)col[j], ru[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < kStage; ++j) {
        if (col[j] < 0) continue;
        if (col[j] == row) {
          dslot = r0 + j;
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            x0[d] = rx[j][d];
            if constexpr (VEL) u0[d] = ru[j][d];
          }
          continue;
        }
        double* q = my + s * SS;
#pragma unroll
        for (int d = 0; d < DIM; ++d) q[(L::OX + d) * kNbBlock] = rx[j][d];
        if constexpr (VEL) {
#pragma unroll
          for (int d = 0; d < DIM; ++d) q[(L::OU + d) * kNbBlock] = ru[j][d];
        }
#pragma unroll
        for (int k = 0; k < NMAT; ++k) q[(L::OA + k) * kNbBlock] = 0.0;
        ++s;
      }
    }
  }
  (void)u0;

  double M0[NN];
#pragma unroll
  for (int b = 0; b < NN; ++b) M0[b] = refM<ET>(0, b);
  const double mN0 = refmN<ET>(0);
  const double W = refWsum<ET>();
  double dacc[NMAT];
#pragma unroll
  for (int k = 0; k < NMAT; ++k) dacc[k] = 0.0;

  // ---- walk the incidences: slot words only (prefetched two ahead) ----
  struct Nodes {
    double x[NN][DIM];
    double u[NN][DIM];
    int s[NN];
  };
  auto ld_nodes = [&](uint32_t w, Nodes& Q) {
#pragma unroll
    for (int b = 1; b < NN; ++b) {
      const int s = (w >> (8 * b)) & 0xff;
      Q.s[b] = s;
      const double* q = my + s * SS;
#pragma unroll
      for (int d = 0; d < DIM; ++d) Q.x[b][d] = q[(L::OX + d) * kNbBlock];
      if constexpr (VEL) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) Q.u[b][d] = q[(L::OU + d) * kNbBlock];
      }
    }
  };
  auto step = [&](Nodes& Q) {
    double xe[NN][DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) xe[0][d] = x0[d];
#pragma unroll
    for (int b = 1; b < NN; ++b)
#pragma unroll
      for (int d = 0; d < DIM; ++d) xe[b][d] = Q.x[b][d];
    constexpr bool ADJ = KIND != FPB_LAPLACIAN;
    double gN[DIM][NN];
    const double det = ADJ ? simplex_adj<ET>(xe, gN) : simplex_geometry<ET>(xe, gN);
    double val[NMAT][NN];
    if constexpr (KIND == FPB_MASS) {
#pragma unroll
      for (int b = 0; b < NN; ++b) val[0][b] = det * M0[b];
    } else if constexpr (KIND == FPB_LAPLACIAN) {
      const double dw = det * W;
#pragma unroll
      for (int b = 0; b < NN; ++b) {
        double t = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) t += gN[d][0] * gN[d][b];
        val[0][b] = dw * t;
      }
    } else if constexpr (KIND == FPB_CONVECTION) {
      double ubar[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double t = M0[0] * u0[d];
#pragma unroll
        for (int b = 1; b < NN; ++b) t += M0[b] * Q.u[b][d];
        ubar[d] = t;
      }
#pragma unroll
      for (int b = 0; b < NN; ++b) {
        double t = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) t += ubar[d] * gN[d][b];
        val[0][b] = t;
      }
    } else {  // GRADIENT_XYZ: det gN scaled by mN[0]
#pragma unroll
      for (int k = 0; k < NMAT; ++k)
#pragma unroll
        for (int b = 0; b < NN; ++b) val[k][b] = mN0 * gN[k][b];
    }
#pragma unroll
    for (int k = 0; k < NMAT; ++k) dacc[k] += val[k][0];
    double old[NN][NMAT];
#pragma unroll
    for (int b = 1; b < NN; ++b)
#pragma unroll
      for (int k = 0; k < NMAT; ++k) old[b][k] = my[Q.s[b] * SS + (L::OA + k) * kNbBlock];
#pragma unroll
    for (int b = 1; b < NN; ++b)
#pragma unroll
      for (int k = 0; k < NMAT; ++k) my[Q.s[b] * SS + (L::OA + k) * kNbBlock] = old[b][k] + val[k][b];
  };

  // slot words in groups of kW, double-buffered: group g+1 is in flight
  // while group g is integrated (one register copy per step)
  constexpr int kW = FPB_NB_W;
  uint32_t wc[kW], wn[kW];
  auto ld_w = [&](int mm, uint32_t (&w)[kW]) {
#pragma unroll
    for (int j = 0; j < kW; ++j) w[j] = mm + j < m1 ? __ldg(slots + (int64_t)(mm + j) * 32 + lane) : 0xffffffffu;
  };
  ld_w(m0, wc);
  ld_w(m0 + kW, wn);
  Nodes QA, QB;
  bool done = m0 >= m1 || wc[0] == 0xffffffffu;
  if (!done) ld_nodes(wc[0], QA);
  for (int m = m0; !done && m < m1; m += kW) {
#pragma unroll
    for (int j = 0; j < kW; j += 2) {
      // QA holds entry j; stage j+1 into QB, integrate j, stage j+2 into QA
      const bool h1 = wc[j + 1] != 0xffffffffu;
      if (h1) ld_nodes(wc[j + 1], QB);
      step(QA);
      if (!h1) {
        done = true;
        break;
      }
      const uint32_t w2 = j + 2 < kW ? wc[j + 2] : wn[0];
      const bool h2 = w2 != 0xffffffffu;
      if (h2) ld_nodes(w2, QA);
      step(QB);
      if (!h2) {
        done = true;
        break;
      }
    }
#pragma unroll
    for (int j = 0; j < kW; ++j) wc[j] = wn[j];
    ld_w(m + 2 * kW, wn);
  }

  // ---- warp-cooperative coalesced write-out ----
  // The warp's 32 consecutive rows are one contiguous CSR range
  // [base, base + span).  Per matrix, every lane copies its row (diagonal
  // from registers) into a per-warp linear buffer laid over the warp's
  // now-dead coordinate fields (chunks of 32 doubles: slot s, field d), then
  // the warp streams the buffer out with fully coalesced stores.
  const int wbase = tid & ~31;
  const int wlane = tid & 31;
  const int base = __shfl_sync(0xffffffffu, rlo, 0);
  int wend = live ? rlo + rlen : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wend = max(wend, __shfl_xor_sync(0xffffffffu, wend, o));
  const int span = wend - base;  // <= 32 rowcap <= 32 DIM (rowcap - 1): fits
  auto buf = [&](int i) -> double& {
    const int c = i >> 5;  // chunk -> (slot, coordinate field)
    return sm[(c / DIM) * SS + (L::OX + c % DIM) * kNbBlock + wbase + (i & 31)];
  };
#pragma unroll
  for (int k = 0; k < NMAT; ++k) {
    __syncwarp();
    for (int r = 0; r < rlen; ++r) {
      const double v = r == dslot ? dacc[k] : my[(r - (r > dslot)) * SS + (L::OA + k) * kNbBlock];
      buf(rlo - base + r) = v;
    }
    __syncwarp();
    double* o = out + k * nnz + base;
    for (int q = wlane; q < span; q += 32) {
      const double v = buf(q);
      o[q] = accumulate ? o[q] + v : v;
    }
  }
}

// ---- SELL-32 incidence setup ---------------------------------------------------
__global__ void k_inc_count(int64_t total, const int32_t* conn, int32_t* cnt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[conn[t]], 1);
}

__global__ void k_slice_width(int32_t n, const int32_t* cnt, int32_t* width) {
  int64_t nsl = ((int64_t)n + 31) / 32;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nsl * 32;
       t += (int64_t)gridDim.x * blockDim.x) {
    int v = t < n ? cnt[t] : 0;
    v = __reduce_max_sync(0xffffffffu, v);
    if ((t & 31) == 0) width[t >> 5] = v;
  }
}

__global__ void k_inc_fill(int64_t nelem, int nn, const int32_t* conn, const int32_t* slice_ptr,
                           int32_t* cursor, int32_t* inc) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nelem * nn;
       t += (int64_t)gridDim.x * blockDim.x) {
    int row = conn[t];
    int slot = atomicAdd(&cursor[row], 1);
    inc[((int64_t)slice_ptr[row >> 5] + slot) * 32 + (row & 31)] = (int32_t)(t / nn);
  }
}

// ascending element order per row (insertion sort; lists are short) — makes
// the summation order, and therefore every output bit, deterministic
__global__ void k_inc_sort(int32_t n, const int32_t* cnt, const int32_t* slice_ptr, int32_t* inc) {
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    int32_t* base = inc + (int64_t)slice_ptr[row >> 5] * 32 + (row & 31);
    int len = cnt[row];
    for (int i = 1; i < len; ++i) {
      int v = base[(int64_t)i * 32];
      int j = i - 1;
      while (j >= 0 && base[(int64_t)j * 32] > v) {
        base[(int64_t)(j + 1) * 32] = base[(int64_t)j * 32];
        --j;
      }
      base[(int64_t)(j + 1) * 32] = v;
    }
  }
}

// Even permutation that brings local node a to position 0: XOR with a for
// 4-node simplices (identity or a double transposition), rotation for 3.
__device__ __forceinline__ int rot_node(int nn, int a, int b) { return nn == 4 ? (b ^ a) : (a + b) % 3; }

// row of SELL entry (column m, lane): largest s with slice_ptr[s] <= m
__device__ __forceinline__ int sell_row(int64_t nsl, const int32_t* slice_ptr, int64_t m, int lane) {
  int64_t lo = 0, hi = nsl;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (slice_ptr[mid] <= m) lo = mid; else hi = mid;
  }
  return (int)(lo * 32 + lane);
}

// Slot bytes in record order (node b of the rotated record): byte 0 = the
// diagonal's offset in the row, bytes 1.. = off-diagonal index (row offset
// with the diagonal skipped, so the row kernel keeps rowcap-1 accumulators).
__global__ void k_inc_slots(int32_t n, int nn, int64_t total, const int32_t* slice_ptr,
                            const int32_t* inc, const int32_t* conn, const int32_t* rowptr,
                            const int32_t* colind, uint32_t* slots, int* err) {
  const int64_t nsl = ((int64_t)n + 31) / 32;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int e = inc[t];
    uint32_t packed = 0xffffffffu;  // padding entry
    if (e >= 0) {
      const int row = sell_row(nsl, slice_ptr, t >> 5, (int)(t & 31));
      const int r0 = rowptr[row], r1 = rowptr[row + 1];
      int a = 0;
      for (int b = 0; b < nn; ++b) a = conn[(int64_t)e * nn + b] == row ? b : a;
      int off[4] = {0, 0, 0, 0};
      for (int b = 0; b < nn; ++b) {
        const int col = conn[(int64_t)e * nn + rot_node(nn, a, b)];
        int l = r0, h = r1;
        while (l < h) {
          int mid = (l + h) >> 1;
          if (colind[mid] < col) l = mid + 1; else h = mid;
        }
        off[b] = l - r0;
        if (l >= r1 || colind[l] != col || off[b] > 255) atomicExch(err, 1);
      }
      packed = (uint32_t)(off[0] & 0xff);
      for (int b = 1; b < nn; ++b) {
        const int o = off[b] - (off[b] > off[0]);
        packed |= (uint32_t)(o & 0xff) << (8 * b);
      }
    }
    slots[t] = packed;
  }
}

// inline node ids of every SELL entry, rotated so the row's node comes
// first (padding: -1)
__global__ void k_inc_nodes(int32_t n, int64_t total, int nn, const int32_t* slice_ptr, const int32_t* inc,
                            const int32_t* conn, int4* incn) {
  const int64_t nsl = ((int64_t)n + 31) / 32;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int e = inc[t];
    int4 v = make_int4(-1, -1, -1, -1);
    if (e >= 0) {
      const int row = sell_row(nsl, slice_ptr, t >> 5, (int)(t & 31));
      const int32_t* c = conn + (int64_t)e * nn;
      int a = 0;
      for (int b = 0; b < nn; ++b) a = c[b] == row ? b : a;
      v.x = c[rot_node(nn, a, 0)];
      v.y = c[rot_node(nn, a, 1)];
      v.z = c[rot_node(nn, a, 2)];
      v.w = nn > 3 ? c[rot_node(nn, a, 3)] : -1;
    }
    incn[t] = v;
  }
}

// 32-byte node records: rec[i] = (a[i][0..dim), 0..., extra[i] | 0)
__global__ void k_pack4(int64_t n, int dim, const double* a, const double* extra, double* rec) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double r[4] = {0.0, 0.0, 0.0, 0.0};
    for (int d = 0; d < dim; ++d) r[d] = a[i * dim + d];
    if (extra) r[3] = extra[i];
    reinterpret_cast<double4*>(rec)[i] = make_double4(r[0], r[1], r[2], r[3]);
  }
}

__global__ void k_max_rowlen(int32_t n, const int32_t* rowptr, int* out) {
  int best = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    best = max(best, rowptr[i + 1] - rowptr[i]);
  best = __reduce_max_sync(0xffffffffu, best);
  if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

template <int ET, int KIND>
static int launch_rows(int32_t n, int32_t row0, const int32_t* slice_ptr, const int32_t* incn,
                       const uint32_t* slots, const double* xyz4, const double* uvw4, double rho, double mu,
                       double kappa, const int32_t* rowptr, int64_t nnz, int rowcap, int accumulate,
                       double* out, cudaStream_t s) {
  constexpr bool MAT = KIND == FPB_MASS || KIND == FPB_LAPLACIAN || KIND == FPB_CONVECTION ||
                       KIND == FPB_GRADIENT_XYZ;
  constexpr int NMAT = KIND == FPB_GRADIENT_XYZ ? Elem<ET>::DIM : 1;
  size_t smem = MAT ? (size_t)NMAT * (rowcap > 1 ? rowcap - 1 : 1) * kRowsBlock * sizeof(double) : 0;
  if (smem > 48 * 1024)
    FPB_CUDA(cudaFuncSetAttribute(k_rows<ET, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks = (n - row0 + kRowsBlock - 1) / kRowsBlock;
  k_rows<ET, KIND><<<blocks, kRowsBlock, smem, s>>>(n, row0, slice_ptr, reinterpret_cast<const int4*>(incn), slots,
                                                    xyz4, uvw4, rho, mu, kappa, rowptr, nnz, rowcap,
                                                    accumulate, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

template <int ET, int KIND>
static int launch_rows_nb(int32_t n, int32_t row0, const int32_t* slice_ptr, const uint32_t* slots, const double* xyz4,
                          const double* uvw4, const int32_t* rowptr, const int32_t* colind, int64_t nnz,
                          int rowcap, int accumulate, double* out, cudaStream_t s) {
  using L = NbLayout<ET, KIND>;
  const size_t smem = (size_t)L::FIELDS * (rowcap > 1 ? rowcap - 1 : 1) * kNbBlock * sizeof(double);
  if (smem > 48 * 1024)
    FPB_CUDA(cudaFuncSetAttribute(k_rows_nb<ET, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int blocks = (n - row0 + kNbBlock - 1) / kNbBlock;
  k_rows_nb<ET, KIND><<<blocks, kNbBlock, smem, s>>>(n, row0, slice_ptr, slots, xyz4, uvw4, rowptr, colind, nnz,
                                                     rowcap, accumulate, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

template <int ET>
static int rows_kind(int kind, int32_t n, int32_t row0, const int32_t* slice_ptr, const int32_t* incn,
                     const uint32_t* slots, const double* xyz4, const double* uvw4, double rho, double mu,
                     double kappa, const int32_t* rowptr, const int32_t* colind, int64_t nnz, int rowcap,
                     int accumulate, double* out, cudaStream_t s) {
  const bool nb = g_tuning_rows_nb && colind && rowcap >= 2 && rowcap <= 256;
#define FPB_ROWS_CASE(K)                                                                                 \
  case K:                                                                                                \
    return launch_rows<ET, K>(n, row0, slice_ptr, incn, slots, xyz4, uvw4, rho, mu, kappa, rowptr, nnz, rowcap, \
                              accumulate, out, s);
#define FPB_ROWS_NB_CASE(K)                                                                                  \
  case K:                                                                                                    \
    if (nb)                                                                                                  \
      return launch_rows_nb<ET, K>(n, row0, slice_ptr, slots, xyz4, uvw4, rowptr, colind, nnz, rowcap, accumulate, \
                                   out, s);                                                                  \
    return launch_rows<ET, K>(n, row0, slice_ptr, incn, slots, xyz4, uvw4, rho, mu, kappa, rowptr, nnz, rowcap,     \
                              accumulate, out, s);
  switch (kind) {
    FPB_ROWS_NB_CASE(FPB_MASS)
    FPB_ROWS_NB_CASE(FPB_LAPLACIAN)
    FPB_ROWS_NB_CASE(FPB_CONVECTION)
    FPB_ROWS_CASE(FPB_MOMENTUM_RHS)
    FPB_ROWS_CASE(FPB_SCALAR_RHS)
    case FPB_GRADIENT_XYZ:
      if (nb)
        return launch_rows_nb<ET, FPB_GRADIENT_XYZ>(n, row0, slice_ptr, slots, xyz4, uvw4, rowptr, colind, nnz, rowcap,
                                                    accumulate, out, s);
      return launch_rows<ET, FPB_GRADIENT_XYZ>(n, row0, slice_ptr, incn, slots, xyz4, uvw4, rho, mu, kappa, rowptr,
                                               nnz, rowcap, accumulate, out, s);
  }
#undef FPB_ROWS_CASE
#undef FPB_ROWS_NB_CASE
  set_error("unknown kernel kind %d", kind);
  return FPB_ECONFIG;
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_set_tuning(const char* name, int value) {
  if (name && strcmp(name, "rows_nb") == 0) {
    g_tuning_rows_nb = value;
    return FPB_OK;
  }
  if (name && strcmp(name, "blk_pipe") == 0) {
    g_tuning_blk_pipe = value;
    return FPB_OK;
  }
  if (name && strcmp(name, "kgrad_march") == 0) {
    g_tuning_kgrad_march = value;
    return FPB_OK;
  }
  if (name && strcmp(name, "kgrad_kchunk") == 0) {
    FPB_REQUIRE(value >= 0, "kgrad_kchunk must be >= 0 (0: automatic)");
    g_tuning_kgrad_kchunk = value;
    return FPB_OK;
  }
  if (name && strcmp(name, "kgrad_bthreads") == 0) {
    FPB_REQUIRE(value == 32 || value == 64 || value == 128, "kgrad_bthreads must be 32, 64 or 128");
    g_tuning_kgrad_bthreads = value;
    return FPB_OK;
  }
  if (name && strcmp(name, "kmom_smem_kb") == 0) {
    FPB_REQUIRE(value >= 0 && value <= 227, "kmom_smem_kb must be 0..227");
    g_tuning_kmom_smem_kb = value;
    return FPB_OK;
  }
  if (name && strcmp(name, "hex_canon_rows") == 0) {
    FPB_REQUIRE(value == 32 || value == 64, "hex_canon_rows must be 32 or 64");
    g_tuning_hex_canon_rows = value;
    return FPB_OK;
  }
  set_error("unknown tuning knob %s", name ? name : "(null)");
  return FPB_ECONFIG;
}

int fpb_incidence_build(int32_t n, int64_t nelem, int nn, const int32_t* conn, int32_t* slice_ptr,
                        int32_t* inc, int64_t* ncols_h, void* stream) {
  FPB_REQUIRE(n >= 0 && nelem >= 0 && nn > 0 && nn <= 8, "bad incidence arguments");
  cudaStream_t s = as_stream(stream);
  const int64_t nsl = ((int64_t)n + 31) / 32;
  int32_t *cnt = nullptr, *width = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  FPB_CUDA(cudaMallocAsync(&cnt, sizeof(int32_t) * (n + 1), s));
  FPB_CUDA(cudaMallocAsync(&width, sizeof(int32_t) * (nsl + 1), s));
  FPB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), s));
  FPB_CUDA(cudaMemsetAsync(width, 0, sizeof(int32_t) * (nsl + 1), s));
  if (nelem > 0) k_inc_count<<<grid_for(nelem * nn, 256), 256, 0, s>>>(nelem * nn, conn, cnt);
  if (nsl > 0) k_slice_width<<<grid_for(nsl * 32, 256), 256, 0, s>>>(n, cnt, width);
  FPB_LAUNCH_CHECK();
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, width, slice_ptr, nsl + 1, s);
  FPB_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
  FPB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, width, slice_ptr, nsl + 1, s));
  int32_t ncols = 0;
  FPB_CUDA(cudaMemcpyAsync(&ncols, slice_ptr + nsl, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FPB_CUDA(cudaStreamSynchronize(s));
  *ncols_h = ncols;
  if (inc) {
    FPB_CUDA(cudaMemsetAsync(inc, 0xff, sizeof(int32_t) * (size_t)ncols * 32, s));
    FPB_CUDA(cudaMemsetAsync(width, 0, sizeof(int32_t) * (nsl + 1), s));
    int32_t* cursor = nullptr;
    FPB_CUDA(cudaMallocAsync(&cursor, sizeof(int32_t) * (n + 1), s));
    FPB_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (n + 1), s));
    if (nelem > 0) k_inc_fill<<<grid_for(nelem * nn, 256), 256, 0, s>>>(nelem, nn, conn, slice_ptr, cursor, inc);
    if (n > 0) k_inc_sort<<<grid_for(n, 128), 128, 0, s>>>(n, cnt, slice_ptr, inc);
    FPB_LAUNCH_CHECK();
    FPB_CUDA(cudaFreeAsync(cursor, s));
  }
  FPB_CUDA(cudaFreeAsync(tmp, s));
  FPB_CUDA(cudaFreeAsync(cnt, s));
  FPB_CUDA(cudaFreeAsync(width, s));
  return FPB_OK;
}

int fpb_incidence_slots(int32_t n, int nn, int64_t ncols, const int32_t* slice_ptr,
                        const int32_t* inc, const int32_t* conn, const int32_t* rowptr,
                        const int32_t* colind, uint32_t* slots, int* rowcap_h, void* stream) {
  FPB_REQUIRE(nn <= 4, "row-owned assembly supports elements with at most 4 nodes");
  cudaStream_t s = as_stream(stream);
  int* dev = nullptr;
  FPB_CUDA(cudaMallocAsync(&dev, 2 * sizeof(int), s));
  FPB_CUDA(cudaMemsetAsync(dev, 0, 2 * sizeof(int), s));
  int64_t total = ncols * 32;
  if (total > 0)
    k_inc_slots<<<grid_for(total, 256), 256, 0, s>>>(n, nn, total, slice_ptr, inc, conn, rowptr, colind,
                                                     slots, dev);
  if (n > 0) k_max_rowlen<<<grid_for(n, 256), 256, 0, s>>>(n, rowptr, dev + 1);
  FPB_LAUNCH_CHECK();
  int h[2] = {0, 0};
  FPB_CUDA(cudaMemcpyAsync(h, dev, sizeof(h), cudaMemcpyDeviceToHost, s));
  FPB_CUDA(cudaFreeAsync(dev, s));
  FPB_CUDA(cudaStreamSynchronize(s));
  *rowcap_h = h[1];
  if (h[0]) {
    set_error("element node pair missing from CSR pattern (or a row longer than 256 entries)");
    return FPB_EPATTERN;
  }
  return FPB_OK;
}

int fpb_incidence_nodes(int32_t n, int64_t ncols, int nn, const int32_t* slice_ptr, const int32_t* inc,
                        const int32_t* conn, int32_t* incn, void* stream) {
  FPB_REQUIRE(nn == 3 || nn == 4, "inline incidence records hold at most 4 nodes");
  if (ncols <= 0) return FPB_OK;
  k_inc_nodes<<<grid_for(ncols * 32, 256), 256, 0, as_stream(stream)>>>(n, ncols * 32, nn, slice_ptr, inc, conn,
                                                                        reinterpret_cast<int4*>(incn));
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_pack4(int64_t n, int dim, const double* a, const double* extra, double* rec, void* stream) {
  FPB_REQUIRE(dim >= 1 && dim <= 3, "pack4 holds at most 3 components plus one extra");
  FPB_REQUIRE(((uintptr_t)rec & 31) == 0, "node records must be 32-byte aligned");
  if (n <= 0) return FPB_OK;
  k_pack4<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, dim, a, extra, rec);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_assemble_rows(int kind, int etype, int32_t n, int32_t row0, int32_t row1, const int32_t* slice_ptr,
                      const int32_t* inc,
                      const int32_t* conn, const int32_t* incn, const uint32_t* slots, const double* xyz4,
                      const double* uvw4, double rho, double mu, double kappa, const int32_t* rowptr,
                      const int32_t* colind, int64_t nnz, int rowcap, int accumulate, double* out, void* stream) {
  (void)inc;
  (void)conn;
  FPB_REQUIRE(etype == FPB_TRI03 || etype == FPB_TET04,
              "row-owned assembly is for affine simplices (TRI03, TET04)");
  FPB_REQUIRE(g_ref_loaded[etype], "reference tables for element type %d not uploaded", etype);
  bool mat = kind == FPB_MASS || kind == FPB_LAPLACIAN || kind == FPB_CONVECTION || kind == FPB_GRADIENT_XYZ;
  FPB_REQUIRE(!mat || (slots && rowptr && colind && rowcap > 0), "matrix kinds need slots, rowptr, colind and rowcap");
  FPB_REQUIRE(!(kind == FPB_CONVECTION || kind == FPB_MOMENTUM_RHS || kind == FPB_SCALAR_RHS) || uvw4,
              "kind %d needs a velocity field", kind);
  FPB_REQUIRE(rowcap <= 256, "row too long for row-owned assembly");
  FPB_REQUIRE(incn, "row-owned assembly needs the rotated inline node records (fpb_incidence_nodes)");
  FPB_REQUIRE(row0 >= 0 && row0 % 32 == 0 && row1 <= n && row0 <= row1, "row window [%d, %d) must start on a 32-row slice",
              row0, row1);
  if (row1 <= row0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  if (etype == FPB_TET04)
    return rows_kind<FPB_TET04>(kind, row1, row0, slice_ptr, incn, slots, xyz4, uvw4, rho, mu, kappa, rowptr, colind, nnz,
                                rowcap, accumulate, out, s);
  return rows_kind<FPB_TRI03>(kind, row1, row0, slice_ptr, incn, slots, xyz4, uvw4, rho, mu, kappa, rowptr, colind, nnz,
                              rowcap, accumulate, out, s);
}

}  // extern "C"
