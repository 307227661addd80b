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
int g_tuning_gradient_split = 0;  // fpb_set_tuning("gradient_split", 0|1)
#ifndef FPB_ROWS_LD256
#define FPB_ROWS_LD256 1
#endif

constexpr int KIND_GRAD1 = 101;  // one gradient direction (kdir) per launch

template <int ET, int KIND>
__global__ void __launch_bounds__(kRowsBlock)
k_rows(int32_t n, const int32_t* __restrict__ slice_ptr, const int32_t* __restrict__ incn,
       const int32_t* __restrict__ inc, const int32_t* __restrict__ conn,
       const uint32_t* __restrict__ slots, const double* __restrict__ xyz4,
       const double* __restrict__ uvw4, double rho, double mu, double kappa,
       const int32_t* __restrict__ rowptr, int64_t nnz, int rowcap, int accumulate, int kdir,
       double* __restrict__ out) {
  constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM;
  constexpr bool MAT = KIND == FPB_MASS || KIND == FPB_LAPLACIAN || KIND == FPB_CONVECTION ||
                       KIND == FPB_GRADIENT_XYZ || KIND == KIND_GRAD1;
  constexpr int NMAT = KIND == FPB_GRADIENT_XYZ ? DIM : 1;
  constexpr bool NEED_VEL = KIND == FPB_CONVECTION || KIND == FPB_MOMENTUM_RHS || KIND == FPB_SCALAR_RHS;
  constexpr int NACC = KIND == FPB_MOMENTUM_RHS ? DIM : 1;
  extern __shared__ double sacc[];  // [NMAT][rowcap][kRowsBlock] (matrix kinds)

  const int tid = threadIdx.x;
  const int row = blockIdx.x * kRowsBlock + tid;
  if (row >= n) return;  // no block-wide synchronisation below
  const int lane = row & 31;
  const int m0 = __ldg(slice_ptr + (row >> 5)), m1 = __ldg(slice_ptr + (row >> 5) + 1);

  int rlo = 0, rlen = 0;
  if constexpr (MAT) {
    rlo = __ldg(rowptr + row);
    rlen = __ldg(rowptr + row + 1) - rlo;
    for (int k = 0; k < NMAT; ++k)
      for (int r = 0; r < rlen; ++r) sacc[(k * rowcap + r) * kRowsBlock + tid] = 0.0;
  }
  double acc[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q] = 0.0;
  const double W = refWsum<ET>();

  // Software pipeline over the incidence list: while element m is
  // integrated, the node records of m+1 and the node ids of m+2 are in
  // flight.  Incidences carry the element's node ids inline (int4 SELL
  // entries), and node data are 32-byte records read with one 256-bit load
  // (LDG.E.ENL2.256) each: xyz4[n] = (x, y, z|0, 0), uvw4[n] = (u, v, w|0, phi).
  auto ld_c = [&](int mm, int (&c)[4]) {
    if (mm < m1) {
      if (incn) {  // inline node ids (one dependent load level less)
        const int4 c4 = __ldg(reinterpret_cast<const int4*>(incn) + (int64_t)mm * 32 + lane);
        c[0] = c4.x; c[1] = c4.y; c[2] = c4.z; c[3] = c4.w;
        return;
      }
      const int e = __ldg(inc + (int64_t)mm * 32 + lane);
      if (e < 0) {
        c[0] = -1;
      } else if constexpr (NN == 4) {
        const int4 c4 = __ldg(reinterpret_cast<const int4*>(conn) + e);
        c[0] = c4.x; c[1] = c4.y; c[2] = c4.z; c[3] = c4.w;
      } else {
#pragma unroll
        for (int b = 0; b < NN; ++b) c[b] = __ldg(conn + (int64_t)e * NN + b);
      }
    } else {
      c[0] = -1;
    }
  };
  constexpr int NU = NEED_VEL ? NN : 1;
  constexpr int NF = KIND == FPB_SCALAR_RHS ? NN : 1;
  auto ld_x = [&](const int (&c)[4], double (&x)[NN][DIM], double (&u)[NU][DIM], double (&f)[NF]) {
    if (c[0] < 0) return;
#pragma unroll
    for (int b = 0; b < NN; ++b) {
#if FPB_ROWS_LD256
      double r[4];
      ld256(xyz4 + 4 * (int64_t)c[b], r);
#pragma unroll
      for (int d = 0; d < DIM; ++d) x[b][d] = r[d];
#else
#pragma unroll
      for (int d = 0; d < DIM; ++d) x[b][d] = __ldg(xyz4 + 4 * (int64_t)c[b] + d);
#endif
    }
    if constexpr (NEED_VEL) {
#pragma unroll
      for (int b = 0; b < NN; ++b) {
        double r[4];
        ld256(uvw4 + 4 * (int64_t)c[b], r);
#pragma unroll
        for (int d = 0; d < DIM; ++d) u[b][d] = r[d];
        if constexpr (KIND == FPB_SCALAR_RHS) f[b] = r[3];
      }
    }
  };
  int cA[4], cB[4], cC[4];
  double xA[NN][DIM] = {}, xB[NN][DIM] = {}, uA[NU][DIM] = {}, uB[NU][DIM] = {}, fA[NF] = {}, fB[NF] = {};
  ld_c(m0, cA);
  ld_c(m0 + 1, cB);
  ld_x(cA, xA, uA, fA);

  for (int m = m0; m < m1; ++m) {
    if (cA[0] < 0) break;  // row lists are padded at the end
    ld_x(cB, xB, uB, fB);
    ld_c(m + 2, cC);
    int c[NN];
    double xe[NN][DIM], ue[NU][DIM], fe[NF];
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      c[b] = cA[b];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        xe[b][d] = xA[b][d];
        xA[b][d] = xB[b][d];
      }
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      cA[b] = cB[b];
      cB[b] = cC[b];
    }
#pragma unroll
    for (int b = 0; b < NU; ++b)
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        ue[b][d] = uA[b][d];
        uA[b][d] = uB[b][d];
      }
#pragma unroll
    for (int b = 0; b < NF; ++b) {
      fe[b] = fA[b];
      fA[b] = fB[b];
    }
    int a = 0;
#pragma unroll
    for (int b = 1; b < NN; ++b) a = (c[b] == row) ? b : a;
    double gN[DIM][NN];
    const double det = simplex_geometry<ET>(xe, gN);

    // row a of the element mass table, M[a][0..NN)
    double Ma[NN];
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      double t[NN];
#pragma unroll
      for (int q = 0; q < NN; ++q) t[q] = refM<ET>(q, b);
      Ma[b] = pick<NN>(t, a);
    }
    double ubar[DIM];
    if constexpr (NEED_VEL) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < NN; ++b) s += Ma[b] * ue[b][d];
        ubar[d] = s;
      }
    }
    double gNa[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      double t[NN];
#pragma unroll
      for (int b = 0; b < NN; ++b) t[b] = gN[d][b];
      gNa[d] = pick<NN>(t, a);
    }

    if constexpr (MAT) {
      double val[NMAT][NN];
      if constexpr (KIND == FPB_MASS) {
#pragma unroll
        for (int b = 0; b < NN; ++b) val[0][b] = det * Ma[b];
      } else if constexpr (KIND == FPB_LAPLACIAN) {
        const double dw = det * W;
#pragma unroll
        for (int b = 0; b < NN; ++b) {
          double s = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) s += gNa[d] * gN[d][b];
          val[0][b] = dw * s;
        }
      } else if constexpr (KIND == FPB_CONVECTION) {
#pragma unroll
        for (int b = 0; b < NN; ++b) {
          double s = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) s += ubar[d] * gN[d][b];
          val[0][b] = det * s;
        }
      } else {  // GRADIENT_XYZ / GRAD1
        double t[NN];
#pragma unroll
        for (int b = 0; b < NN; ++b) t[b] = refmN<ET>(b);
        const double f = det * pick<NN>(t, a);
        if constexpr (KIND == KIND_GRAD1) {
#pragma unroll
          for (int b = 0; b < NN; ++b) val[0][b] = f * (kdir == 0 ? gN[0][b] : (kdir == 1 ? gN[1][b] : gN[DIM - 1][b]));
        } else {
#pragma unroll
          for (int k = 0; k < NMAT; ++k)
#pragma unroll
            for (int b = 0; b < NN; ++b) val[k][b] = f * gN[k][b];
        }
      }
      const uint32_t sl = __ldg(slots + (int64_t)m * 32 + lane);
#pragma unroll
      for (int b = 0; b < NN; ++b) {
        const int s = (sl >> (8 * b)) & 0xff;
#pragma unroll
        for (int k = 0; k < NMAT; ++k) sacc[(k * rowcap + s) * kRowsBlock + tid] += val[k][b];
      }
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
          visc += S_lk * gNa[l];
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
        diff += gphi[d] * gNa[d];
      }
      acc[0] -= det * adv + kappa * det * W * diff;
    }
  }

  if constexpr (MAT) {
#pragma unroll
    for (int k = 0; k < NMAT; ++k) {
      double* o = out + k * nnz + rlo;
      for (int r = 0; r < rlen; ++r) {
        const double v = sacc[(k * rowcap + r) * kRowsBlock + tid];
        o[r] = accumulate ? o[r] + v : v;
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      double* o = out + (int64_t)row * NACC + q;
      *o = accumulate ? *o + acc[q] : acc[q];
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

__global__ void k_inc_slots(int32_t n, int nn, int64_t total, const int32_t* slice_ptr,
                            const int32_t* inc, const int32_t* conn, const int32_t* rowptr,
                            const int32_t* colind, uint32_t* slots, int* err) {
  // entry t = (column m, lane); row = 32 * slice(m) + lane is recovered by
  // binary search of m over slice_ptr
  int64_t nsl = ((int64_t)n + 31) / 32;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = t >> 5;
    int lane = (int)(t & 31);
    int e = inc[t];
    uint32_t packed = 0;
    if (e >= 0) {
      int64_t lo = 0, hi = nsl;  // largest s with slice_ptr[s] <= m
      while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (slice_ptr[mid] <= m) lo = mid; else hi = mid;
      }
      int row = (int)(lo * 32 + lane);
      int r0 = rowptr[row], r1 = rowptr[row + 1];
      for (int b = 0; b < nn; ++b) {
        int col = conn[(int64_t)e * nn + b];
        int l = r0, h = r1;
        while (l < h) {
          int mid = (l + h) >> 1;
          if (colind[mid] < col) l = mid + 1; else h = mid;
        }
        int off = l - r0;
        if (l >= r1 || colind[l] != col || off > 255) atomicExch(err, 1);
        packed |= (uint32_t)(off & 0xff) << (8 * b);
      }
    }
    slots[t] = packed;
  }
}

// inline node ids of every SELL entry (padding: -1)
__global__ void k_inc_nodes(int64_t total, int nn, const int32_t* inc, const int32_t* conn, int4* incn) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int e = inc[t];
    int4 v = make_int4(-1, -1, -1, -1);
    if (e >= 0) {
      const int32_t* c = conn + (int64_t)e * nn;
      v.x = c[0]; v.y = c[1]; v.z = c[2];
      v.w = nn > 3 ? c[3] : -1;
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
static int launch_rows(int32_t n, const int32_t* slice_ptr, const int32_t* incn, const int32_t* inc,
                       const int32_t* conn, const uint32_t* slots,
                       const double* xyz4, const double* uvw4, double rho, double mu, double kappa, const int32_t* rowptr, int64_t nnz,
                       int rowcap, int accumulate, double* out, cudaStream_t s, int kdir = 0) {
  constexpr bool MAT = KIND == FPB_MASS || KIND == FPB_LAPLACIAN || KIND == FPB_CONVECTION ||
                       KIND == FPB_GRADIENT_XYZ || KIND == KIND_GRAD1;
  constexpr int NMAT = KIND == FPB_GRADIENT_XYZ ? Elem<ET>::DIM : 1;
  size_t smem = MAT ? (size_t)NMAT * rowcap * kRowsBlock * sizeof(double) : 0;
  if (smem > 48 * 1024)
    FPB_CUDA(cudaFuncSetAttribute(k_rows<ET, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks = (n + kRowsBlock - 1) / kRowsBlock;
  k_rows<ET, KIND><<<blocks, kRowsBlock, smem, s>>>(n, slice_ptr, incn, inc, conn, slots, xyz4,
                                                    uvw4, rho, mu, kappa,
                                                    rowptr, nnz, rowcap, accumulate, kdir, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

template <int ET>
static int rows_kind(int kind, int32_t n, const int32_t* slice_ptr, const int32_t* incn,
                     const int32_t* inc, const int32_t* conn, const uint32_t* slots, const double* xyz4, const double* uvw4, double rho, double mu,
                     double kappa,
                     const int32_t* rowptr, int64_t nnz, int rowcap, int accumulate, double* out,
                     cudaStream_t s) {
#define FPB_ROWS_CASE(K)                                                                       \
  case K:                                                                                      \
    return launch_rows<ET, K>(n, slice_ptr, incn, inc, conn, slots, xyz4, uvw4, rho, mu, kappa, \
                              rowptr, nnz, rowcap, accumulate, out, s);
  switch (kind) {
    FPB_ROWS_CASE(FPB_MASS)
    FPB_ROWS_CASE(FPB_LAPLACIAN)
    FPB_ROWS_CASE(FPB_CONVECTION)
    FPB_ROWS_CASE(FPB_MOMENTUM_RHS)
    FPB_ROWS_CASE(FPB_SCALAR_RHS)
    case FPB_GRADIENT_XYZ:
      if (g_tuning_gradient_split) {
        for (int k = 0; k < Elem<ET>::DIM; ++k) {
          int rc = launch_rows<ET, KIND_GRAD1>(n, slice_ptr, incn, inc, conn, slots, xyz4, uvw4, rho, mu, kappa,
                                               rowptr, nnz, rowcap, accumulate, out + k * nnz, s, k);
          if (rc) return rc;
        }
        return FPB_OK;
      }
      return launch_rows<ET, FPB_GRADIENT_XYZ>(n, slice_ptr, incn, inc, conn, slots, xyz4, uvw4, rho, mu, kappa,
                                               rowptr, nnz, rowcap, accumulate, out, s);
  }
#undef FPB_ROWS_CASE
  set_error("unknown kernel kind %d", kind);
  return FPB_ECONFIG;
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_set_tuning(const char* name, int value) {
  if (name && strcmp(name, "gradient_split") == 0) {
    g_tuning_gradient_split = value;
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

int fpb_incidence_nodes(int64_t ncols, int nn, const int32_t* inc, const int32_t* conn, int32_t* incn,
                        void* stream) {
  FPB_REQUIRE(nn == 3 || nn == 4, "inline incidence records hold at most 4 nodes");
  if (ncols <= 0) return FPB_OK;
  k_inc_nodes<<<grid_for(ncols * 32, 256), 256, 0, as_stream(stream)>>>(ncols * 32, nn, inc, conn,
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

int fpb_assemble_rows(int kind, int etype, int32_t n, const int32_t* slice_ptr, const int32_t* inc,
                      const int32_t* conn, const int32_t* incn, const uint32_t* slots, const double* xyz4, const double* uvw4, double rho, double mu,
                      double kappa, const int32_t* rowptr, int64_t nnz, int rowcap, int accumulate,
                      double* out, void* stream) {
  FPB_REQUIRE(etype == FPB_TRI03 || etype == FPB_TET04,
              "row-owned assembly is for affine simplices (TRI03, TET04)");
  FPB_REQUIRE(g_ref_loaded[etype], "reference tables for element type %d not uploaded", etype);
  bool mat = kind == FPB_MASS || kind == FPB_LAPLACIAN || kind == FPB_CONVECTION || kind == FPB_GRADIENT_XYZ;
  FPB_REQUIRE(!mat || (slots && rowptr && rowcap > 0), "matrix kinds need slots, rowptr and rowcap");
  FPB_REQUIRE(!(kind == FPB_CONVECTION || kind == FPB_MOMENTUM_RHS || kind == FPB_SCALAR_RHS) || uvw4,
              "kind %d needs a velocity field", kind);
  FPB_REQUIRE(rowcap <= 256, "row too long for row-owned assembly");
  FPB_REQUIRE(incn || (inc && conn), "need inline node records or incidence + connectivity");
  if (n <= 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  if (etype == FPB_TET04)
    return rows_kind<FPB_TET04>(kind, n, slice_ptr, incn, inc, conn, slots, xyz4, uvw4, rho, mu, kappa, rowptr, nnz,
                                rowcap, accumulate, out, s);
  return rows_kind<FPB_TRI03>(kind, n, slice_ptr, incn, inc, conn, slots, xyz4, uvw4, rho, mu, kappa, rowptr, nnz, rowcap,
                              accumulate, out, s);
}

}  // extern "C"
