// Row-owned matrix assembly for Gauss-loop (non-affine) elements: QUAD04,
// PYR05, HEX08 (_kernels.py:150-266 via the reference's Gauss loops).
//
// The element-scatter path (assemble.cu) issues one FP64 reduction per
// (element, i, j, matrix) — 192 per hex for B_x, B_y, B_z — and is bound by
// L2 atomic throughput (~117 G/s on B200, 33 ms for config 4's 20 M hexes).
// Here, as for the simplices (rows.cu), every CSR row is owned by one thread
// that walks its incident elements in ascending element order and writes its
// row once: no atomics, no zero fill, fixed summation order (bitwise
// reproducible).  The price is that each element's Gauss-point geometry is
// evaluated once per node (8x for a hex) — the work is FP64-bound, not
// atomic-bound.  Per Gauss point g the thread forms J_g, its adjugate
// A_g = det J_g^-1 (no reciprocal for MASS, CONVECTION, GRADIENT), and
// G_g[d][b] = sum_l A_g[l][d] dN[l][b](g) = det * dN_b/dx_d, then adds
//   MASS        w_g det N_a N_b
//   LAPLACIAN   (w_g / det) G_a . G_b = sum_l q_l dN_b,l, q = (w_g / det) A G_a
//   CONVECTION  w_g N_a (u_g . G_b),        u_g = sum_c N_c u_c
//   GRADIENT_k  w_g N_a (sum_c N_c) G_b[k]  (CONVECTION with u = e_k)
// which equal the reference's detJw-weighted Gauss sums to rounding (parity
// bar 1e-12).
//
// Incidences are SELL-32 (rows.cu): inc[32 m + lane] = element id (-1 pad);
// slots8[32 m + lane] packs one byte per element node b: 0xff for the row's
// own node (its local index a), else the node's off-diagonal index in the
// row (CSR offset with the diagonal skipped).  Off-diagonal sums live in
// shared memory [s][k][thread], the diagonal in registers.
#include "elemcore.cuh"

namespace fpb {

#ifndef FPB_GL_BLOCK
#define FPB_GL_BLOCK 64
#endif
#ifndef FPB_GL_MINB
#define FPB_GL_MINB 4
#endif
#ifndef FPB_GL_MINB_MASS
#define FPB_GL_MINB_MASS 5  // hex MASS: 5 CTAs / SM measured faster (profiles/r01m_hexmom)
#endif
constexpr int kGlBlock = FPB_GL_BLOCK;

// Gauss-point sign moments for the 8-node hex (elements.py:148-166 corners
// (+-1, +-1, +-1), :226-229 the 2x2x2 rule, x fastest, unit weights):
//   dN_l(b, g) = s_l(b)/8 * prod_{m != l} (1 + s_m(b) x_m(g)),  x_m(g) = +-q,
// so for any Gauss-point vector V_g
//   sum_g V_g[l] dN_l(b, g) = s_l(b)/8 * (M0 + s_m1(b) q M1 + s_m2(b) q M2 + s_m1 s_m2 q^2 M3)[l]
// with M_t the moments of V[l] against 1, sgn x_m1, sgn x_m2, their product
// (m1 < m2 the two directions other than l).  12 FMA per point and matrix
// replace 24 (8 columns x 3 directions), plus 8 + 16 adds per matrix at the
// end; the 1/8 and q powers ride in the point coefficients c, c1, c2.
template <int NM>
struct HexMoments {
  double M[NM][3][4];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < NM; ++k)
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int t = 0; t < 4; ++t) M[k][l][t] = 0.0;
  }
  // c = 1/8 * point weight, c1 = c q, c2 = c q^2; g compile-time after unrolling
  __device__ __forceinline__ void add(int g, int k, const double (&V)[3], double c, double c1, double c2) {
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const int m1 = l == 0 ? 1 : 0, m2 = l == 2 ? 1 : 2;
      const double s1 = ((g >> m1) & 1) ? 1.0 : -1.0, s2 = ((g >> m2) & 1) ? 1.0 : -1.0;
      M[k][l][0] = fma(c, V[l], M[k][l][0]);
      M[k][l][1] = fma(s1 * c1, V[l], M[k][l][1]);
      M[k][l][2] = fma(s2 * c1, V[l], M[k][l][2]);
      M[k][l][3] = fma((s1 * s2) * c2, V[l], M[k][l][3]);
    }
  }
  // acc[k][b] = sum_l sum_g V_g[l] dN_l(b, g) (overwrites)
  __device__ __forceinline__ void finish(double (&acc)[NM][8]) {
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      double T[3][4];  // T[l][2 * (s_m2 > 0) + (s_m1 > 0)]
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const double p = M[k][l][0] + M[k][l][3], m = M[k][l][0] - M[k][l][3];
        const double u = M[k][l][1] + M[k][l][2], v = M[k][l][1] - M[k][l][2];
        T[l][3] = p + u;
        T[l][0] = p - u;
        T[l][1] = m + v;
        T[l][2] = m - v;
      }
      constexpr int sg[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};  // corner b: s_d > 0
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        double r = 0.0;
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          const int m1 = l == 0 ? 1 : 0, m2 = l == 2 ? 1 : 2;
          const double t = T[l][2 * sg[b][m2] + sg[b][m1]];
          r = l == 0 ? (sg[b][0] ? t : -t) : (sg[b][l] ? r + t : r - t);
        }
        acc[k][b] = r;
      }
    }
  }
};

// slot bytes of every SELL entry (nn <= 8), see header comment; also
// reports the longest row (rowcap) and missing node pairs
__global__ void k_inc_slots8(int32_t n, int nn, int64_t total, const int32_t* slice_ptr, const int32_t* inc,
                             const int32_t* conn, const int32_t* rowptr, const int32_t* colind, uint2* slots,
                             int* err) {
  const int64_t nsl = ((int64_t)n + 31) / 32;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int e = inc[t];
    uint32_t w[2] = {0xffffffffu, 0xffffffffu};
    if (e >= 0) {
      const int64_t m = t >> 5;
      int64_t lo = 0, hi = nsl;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (slice_ptr[mid] <= m) lo = mid; else hi = mid;
      }
      const int row = (int)(lo * 32 + (t & 31));
      const int r0 = rowptr[row], r1 = rowptr[row + 1];
      int d = -1;  // diagonal offset
      {
        int l = r0, h = r1;
        while (l < h) {
          const int mid = (l + h) >> 1;
          if (colind[mid] < row) l = mid + 1; else h = mid;
        }
        if (l < r1 && colind[l] == row) d = l - r0;
      }
      if (d < 0) atomicExch(err, 1);
      for (int b = 0; b < nn; ++b) {
        const int col = conn[(int64_t)e * nn + b];
        uint32_t byte = 0xffu;
        if (col != row) {
          int l = r0, h = r1;
          while (l < h) {
            const int mid = (l + h) >> 1;
            if (colind[mid] < col) l = mid + 1; else h = mid;
          }
          const int off = l - r0;
          if (l >= r1 || colind[l] != col || off > 255) atomicExch(err, 1);
          byte = (uint32_t)((off - (off > d)) & 0xff);
        }
        w[b >> 2] = (w[b >> 2] & ~(0xffu << (8 * (b & 3)))) | (byte << (8 * (b & 3)));
      }
    }
    slots[t] = make_uint2(w[0], w[1]);
  }
}

__global__ void k_rowlen_max(int32_t n, const int32_t* rowptr, int* out) {
  int best = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    best = max(best, rowptr[i + 1] - rowptr[i]);
  best = __reduce_max_sync(0xffffffffu, best);
  if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

template <int ET, int KIND>
__global__ void __launch_bounds__(kGlBlock, (KIND == FPB_MASS && ET == FPB_HEX08) ? FPB_GL_MINB_MASS : FPB_GL_MINB)
k_rows_gl(int32_t n, int32_t row0, const int32_t* __restrict__ slice_ptr, const int32_t* __restrict__ inc,
          const int32_t* __restrict__ conn, const uint2* __restrict__ slots, const double* __restrict__ xyz4,
          const double* __restrict__ uvw4, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
          int64_t nnz, int rowcap, int accumulate, double* __restrict__ out) {
  constexpr int NN = Elem<ET>::NN, NG = Elem<ET>::NG, DIM = Elem<ET>::DIM;
  constexpr int NMAT = KIND == FPB_GRADIENT_XYZ ? DIM : 1;
  constexpr bool VEL = KIND == FPB_CONVECTION;
  constexpr int SS = NMAT * kGlBlock;  // doubles per off-diagonal slot
  extern __shared__ double sm[];
  __shared__ double sN[NN * NG];           // N[a][g], runtime a
  __shared__ double sdN[DIM * NN * NG];    // dN[l][a][g], runtime a (LAPLACIAN)
  // hexes except MASS: Gauss-point sign moments (HexMoments); for GRADIENT
  // sN holds the point coefficient 1/8 w_g N_a(g) sum_c N_c(g) instead of N
  constexpr bool HMOM = ET == FPB_HEX08 && KIND != FPB_MASS;
  constexpr double kQ = 0.5773502691896258, kQ2 = kQ * kQ;
  const int tid = threadIdx.x;
  for (int i = tid; i < NN * NG; i += kGlBlock) {
    if constexpr (HMOM && KIND == FPB_GRADIENT_XYZ) {
      const int g = i % NG;
      double sNg = 0.0;
      for (int c = 0; c < NN; ++c) sNg += c_ref[ET].N[c * NG + g];
      sN[i] = 0.125 * (c_ref[ET].w[g] * c_ref[ET].N[i] * sNg);
    } else {
      sN[i] = c_ref[ET].N[i];
    }
  }
  if constexpr (KIND == FPB_LAPLACIAN)
    for (int i = tid; i < DIM * NN * NG; i += kGlBlock) sdN[i] = c_ref[ET].dN[i];
  __syncthreads();

  const int row = row0 + blockIdx.x * kGlBlock + tid;  // rows [row0, n)
  if (row >= n) return;
  const int lane = row & 31;
  const int m0 = __ldg(slice_ptr + (row >> 5)), m1 = __ldg(slice_ptr + (row >> 5) + 1);
  const int rlo = __ldg(rowptr + row), rlen = __ldg(rowptr + row + 1) - rlo;
  double* const my = sm + tid;
  for (int r = 0; r + 1 < rlen; ++r)
#pragma unroll
    for (int k = 0; k < NMAT; ++k) my[r * SS + k * kGlBlock] = 0.0;
  double dacc[NMAT];
#pragma unroll
  for (int k = 0; k < NMAT; ++k) dacc[k] = 0.0;

  struct Stage {
    int e;
    uint2 w;
    double x[NN][DIM];
    double u[VEL ? NN : 1][DIM];
  };
  auto load = [&](int mm, Stage& S) {
    S.e = mm < m1 ? __ldg(inc + (int64_t)mm * 32 + lane) : -1;
    if (S.e < 0) return;
    S.w = __ldg(slots + (int64_t)mm * 32 + lane);
    int c[NN];
#pragma unroll
    for (int b = 0; b < NN; ++b) c[b] = __ldg(conn + (int64_t)S.e * NN + b);
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      double r4[4];
      ld256(xyz4 + 4 * (int64_t)c[b], r4);
#pragma unroll
      for (int d = 0; d < DIM; ++d) S.x[b][d] = r4[d];
      if constexpr (VEL) {
        ld256(uvw4 + 4 * (int64_t)c[b], r4);
#pragma unroll
        for (int d = 0; d < DIM; ++d) S.u[b][d] = r4[d];
      }
    }
  };

  // keep the next element's node records in flight while integrating the
  // current one (two register stages; profiles/r01i/gl_variants.txt,
  // profiles/r01m_hexmom: with the Gauss-point moments the 3-matrix hex
  // gradient gains too)
  Stage cur, nxt;
  load(m0, cur);
  for (int m = m0; m < m1 && cur.e >= 0; ++m) {
    load(m + 1, nxt);
    // the row's local node a (slot byte 0xff)
    int a = 0;
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      const uint32_t byte = ((b < 4 ? cur.w.x : cur.w.y) >> (8 * (b & 3))) & 0xffu;
      a = byte == 0xffu ? b : a;
    }
    double acc[NMAT][NN];
#pragma unroll
    for (int k = 0; k < NMAT; ++k)
#pragma unroll
      for (int b = 0; b < NN; ++b) acc[k][b] = 0.0;
    HexMoments<HMOM ? NMAT : 1> hm;
    if constexpr (HMOM) hm.zero();

    HexCoef hc;
    if constexpr (ET == FPB_HEX08) hex_coeffs(cur.x, hc);
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      double J[DIM][DIM];
      if constexpr (ET == FPB_HEX08) {
        hex_jacobian(hc, g, J);  // sum-factorised (common.cuh)
      } else {
#pragma unroll
        for (int d = 0; d < DIM; ++d)
#pragma unroll
          for (int l = 0; l < DIM; ++l) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < NN; ++b) s += cur.x[b][d] * refdN<ET>(l, b, g);
            J[d][l] = s;
          }
      }
      double A[DIM][DIM], det;  // A[l][d] = det * Ji[l][d]
      if constexpr (DIM == 2) {
        det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        A[0][0] = J[1][1];
        A[0][1] = -J[0][1];
        A[1][0] = -J[1][0];
        A[1][1] = J[0][0];
      } else {
        A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        det = J[0][0] * A[0][0] + J[0][1] * A[1][0] + J[0][2] * A[2][0];
        A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
        A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
        A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
        A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
        A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
        A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      }
      const double Na = sN[a * NG + g];
      if constexpr (KIND == FPB_MASS) {
        const double wa = refW<ET>(g) * det * Na;
#pragma unroll
        for (int b = 0; b < NN; ++b) acc[0][b] += wa * refN<ET>(b, g);
      } else if constexpr (KIND == FPB_LAPLACIAN) {
        double Ga[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          double s = 0.0;
#pragma unroll
          for (int l = 0; l < DIM; ++l) s += A[l][d] * sdN[(l * NN + a) * NG + g];
          Ga[d] = s;
        }
        // G_a . G_b = sum_l q[l] dN[l][b] with q = A Ga: 3 FMA per column
        const double wd = refW<ET>(g) / det;
        double q[DIM];
#pragma unroll
        for (int l = 0; l < DIM; ++l) {
          double t = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) t += A[l][d] * Ga[d];
          q[l] = wd * t;
        }
        if constexpr (HMOM) {
          const double V[3] = {q[0], q[1], q[2]};
          hm.add(g, 0, V, 0.125, 0.125 * kQ, 0.125 * kQ2);
        } else {
#pragma unroll
          for (int b = 0; b < NN; ++b) {
            double t = 0.0;
#pragma unroll
            for (int l = 0; l < DIM; ++l) t += q[l] * refdN<ET>(l, b, g);
            acc[0][b] += t;
          }
        }
      } else if constexpr (KIND == FPB_CONVECTION) {
        double ug[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < NN; ++c) s += cur.u[c][d] * refN<ET>(c, g);
          ug[d] = s;
        }
        double Au[DIM];  // A u_g: adv_b = sum_l dN[l][b] (A u)[l]
#pragma unroll
        for (int l = 0; l < DIM; ++l) {
          double s = 0.0;
#pragma unroll
          for (int d = 0; d < DIM; ++d) s += A[l][d] * ug[d];
          Au[l] = s;
        }
        const double wa = refW<ET>(g) * Na;
        if constexpr (HMOM) {
          const double c = 0.125 * wa;
          const double V[3] = {Au[0], Au[1], Au[2]};
          hm.add(g, 0, V, c, c * kQ, c * kQ2);
        } else {
#pragma unroll
          for (int b = 0; b < NN; ++b) {
            double adv = 0.0;
#pragma unroll
            for (int l = 0; l < DIM; ++l) adv += Au[l] * refdN<ET>(l, b, g);
            acc[0][b] += wa * adv;
          }
        }
      } else if constexpr (HMOM) {  // GRADIENT_XYZ, hex: Na is the point coefficient
        const double c1 = Na * kQ, c2 = Na * kQ2;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          const double V[3] = {A[0][k], A[1][k], A[2][k]};
          hm.add(g, k, V, Na, c1, c2);
        }
      } else {  // GRADIENT_XYZ
        double sNg = 0.0;
#pragma unroll
        for (int c = 0; c < NN; ++c) sNg += refN<ET>(c, g);
        const double wa = refW<ET>(g) * Na * sNg;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          double Ak[DIM];
#pragma unroll
          for (int l = 0; l < DIM; ++l) Ak[l] = wa * A[l][k];
#pragma unroll
          for (int b = 0; b < NN; ++b) {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < DIM; ++l) s += Ak[l] * refdN<ET>(l, b, g);
            acc[k][b] += s;
          }
        }
      }
    }
    if constexpr (HMOM) hm.finish(acc);
    // scatter the row's NN x NMAT values: own node to registers, others to
    // the off-diagonal sums (distinct slots: loads before stores)
    double old[NN][NMAT];
    int so[NN];
#pragma unroll
    for (int b = 0; b < NN; ++b) {
      const uint32_t byte = ((b < 4 ? cur.w.x : cur.w.y) >> (8 * (b & 3))) & 0xffu;
      so[b] = byte == 0xffu ? -1 : (int)byte;
#pragma unroll
      for (int k = 0; k < NMAT; ++k) old[b][k] = so[b] >= 0 ? my[so[b] * SS + k * kGlBlock] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < NN; ++b)
#pragma unroll
      for (int k = 0; k < NMAT; ++k) {
        if (so[b] >= 0) my[so[b] * SS + k * kGlBlock] = old[b][k] + acc[k][b];
        else dacc[k] += acc[k][b];
      }
    cur = nxt;
  }

  // write the row (diagonal from registers)
  int dslot = rlen - 1;
  {
    int l = 0, h = rlen;
    while (l < h) {
      const int mid = (l + h) >> 1;
      if (__ldg(colind + rlo + mid) < row) l = mid + 1; else h = mid;
    }
    if (l < rlen) dslot = l;
  }
#pragma unroll
  for (int k = 0; k < NMAT; ++k) {
    double* o = out + k * nnz + rlo;
    for (int r = 0; r < rlen; ++r) {
      const double v = r == dslot ? dacc[k] : my[(r - (r > dslot)) * SS + k * kGlBlock];
      o[r] = accumulate ? o[r] + v : v;
    }
  }
}

template <int ET, int KIND>
static int launch_gl(int32_t n, int32_t row0, const int32_t* slice_ptr, const int32_t* inc, const int32_t* conn,
                     const uint2* slots, const double* xyz4, const double* uvw4, const int32_t* rowptr,
                     const int32_t* colind, int64_t nnz, int rowcap, int accumulate, double* out, cudaStream_t s) {
  constexpr int NMAT = KIND == FPB_GRADIENT_XYZ ? Elem<ET>::DIM : 1;
  const size_t smem = (size_t)NMAT * (rowcap > 1 ? rowcap - 1 : 1) * kGlBlock * sizeof(double);
  FPB_REQUIRE(smem <= 200 * 1024, "row too long for row-owned assembly (%d entries)", rowcap);
  if (smem > 48 * 1024)
    FPB_CUDA(cudaFuncSetAttribute(k_rows_gl<ET, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_rows_gl<ET, KIND><<<(n - row0 + kGlBlock - 1) / kGlBlock, kGlBlock, smem, s>>>(
      n, row0, slice_ptr, inc, conn, slots, xyz4, uvw4, rowptr, colind, nnz, rowcap, accumulate, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

template <int ET>
static int gl_kind(int kind, int32_t n, int32_t row0, const int32_t* slice_ptr, const int32_t* inc, const int32_t* conn,
                   const uint2* slots, const double* xyz4, const double* uvw4, const int32_t* rowptr,
                   const int32_t* colind, int64_t nnz, int rowcap, int accumulate, double* out, cudaStream_t s) {
  switch (kind) {
    case FPB_MASS:
      return launch_gl<ET, FPB_MASS>(n, row0, slice_ptr, inc, conn, slots, xyz4, uvw4, rowptr, colind, nnz, rowcap, accumulate, out, s);
    case FPB_LAPLACIAN:
      return launch_gl<ET, FPB_LAPLACIAN>(n, row0, slice_ptr, inc, conn, slots, xyz4, uvw4, rowptr, colind, nnz, rowcap, accumulate, out, s);
    case FPB_CONVECTION:
      return launch_gl<ET, FPB_CONVECTION>(n, row0, slice_ptr, inc, conn, slots, xyz4, uvw4, rowptr, colind, nnz, rowcap, accumulate, out, s);
    case FPB_GRADIENT_XYZ:
      return launch_gl<ET, FPB_GRADIENT_XYZ>(n, row0, slice_ptr, inc, conn, slots, xyz4, uvw4, rowptr, colind, nnz, rowcap, accumulate, out, s);
  }
  set_error("row-owned Gauss-loop assembly covers the matrix kinds (got %d)", kind);
  return FPB_ECONFIG;
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_incidence_slots8(int32_t n, int nn, int64_t ncols, const int32_t* slice_ptr, const int32_t* inc,
                         const int32_t* conn, const int32_t* rowptr, const int32_t* colind, uint32_t* slots,
                         int* rowcap_h, void* stream) {
  FPB_REQUIRE(nn >= 1 && nn <= 8, "slot records hold at most 8 nodes");
  cudaStream_t s = as_stream(stream);
  int* dev = nullptr;
  FPB_CUDA(cudaMallocAsync(&dev, 2 * sizeof(int), s));
  FPB_CUDA(cudaMemsetAsync(dev, 0, 2 * sizeof(int), s));
  const int64_t total = ncols * 32;
  if (total > 0)
    k_inc_slots8<<<grid_for(total, 256), 256, 0, s>>>(n, nn, total, slice_ptr, inc, conn, rowptr, colind,
                                                      reinterpret_cast<uint2*>(slots), dev);
  if (n > 0) k_rowlen_max<<<grid_for(n, 256), 256, 0, s>>>(n, rowptr, dev + 1);
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

int fpb_assemble_rows_gl(int kind, int etype, int32_t n, int32_t row0, int32_t row1, const int32_t* slice_ptr,
                         const int32_t* inc,
                         const int32_t* conn, const uint32_t* slots, const double* xyz4, const double* uvw4,
                         const int32_t* rowptr, const int32_t* colind, int64_t nnz, int rowcap, int accumulate,
                         double* out, void* stream) {
  FPB_REQUIRE(etype == FPB_QUAD04 || etype == FPB_PYR05 || etype == FPB_HEX08,
              "row-owned Gauss-loop assembly is for QUAD04, PYR05, HEX08 (got %d)", etype);
  FPB_REQUIRE(g_ref_loaded[etype], "reference tables for element type %d not uploaded", etype);
  FPB_REQUIRE(slots && rowptr && colind && inc && conn && rowcap > 0, "missing incidence / pattern arrays");
  FPB_REQUIRE(kind != FPB_CONVECTION || uvw4, "CONVECTION needs a velocity field");
  FPB_REQUIRE(rowcap <= 256, "row too long for row-owned assembly");
  FPB_REQUIRE(row0 >= 0 && row0 % 32 == 0 && row1 <= n && row0 <= row1, "row window [%d, %d) must start on a 32-row slice",
              row0, row1);
  if (row1 <= row0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  const uint2* sl = reinterpret_cast<const uint2*>(slots);
  switch (etype) {
    case FPB_QUAD04: return gl_kind<FPB_QUAD04>(kind, row1, row0, slice_ptr, inc, conn, sl, xyz4, uvw4, rowptr, colind, nnz, rowcap, accumulate, out, s);
    case FPB_PYR05: return gl_kind<FPB_PYR05>(kind, row1, row0, slice_ptr, inc, conn, sl, xyz4, uvw4, rowptr, colind, nnz, rowcap, accumulate, out, s);
    default: return gl_kind<FPB_HEX08>(kind, row1, row0, slice_ptr, inc, conn, sl, xyz4, uvw4, rowptr, colind, nnz, rowcap, accumulate, out, s);
  }
}

}  // extern "C"
