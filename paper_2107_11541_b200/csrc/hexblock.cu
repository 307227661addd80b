// HEX08 continuity matrices B_x, B_y, B_z (GRADIENT_XYZ = 3 x CONVECTION(e_k),
// timeloop.py:159-171, _kernels.py:238-266) by node bricks: every element's
// Gauss-point geometry is evaluated ONCE per block instead of once per
// incident row (8x for an interior hex, rowsq.cu).
//
// Rows are grouped into blocks of R rows that are compact in space (Morton
// order of the per-axis coordinate ranks; any mesh, no structure assumed).
// One CTA per block, three threads per row (one per matrix k):
//   phase 1  (element, Gauss point) items: J_g from the 8 node records, its
//            adjugate A_g[l][k] (det J * Ji, no reciprocal) into shared memory;
//   phase 2  (element, l, k) items: 8-point Walsh-Hadamard transform over the
//            Gauss points, F[U] = sum_g sigma^U(g) A_g[l][k], contracted with
//            the row-side factor of direction l (2 signs) into
//            H[s][U'] = (F[U'] + s q F[U' + l]) / 64, U' in {0, m1, m2, m1m2};
//   phase 3  (row, k) threads: for each incident element (local index and
//            the row's column slot bytes from the build), the row's 8 entries
//            from 4 H values per l —
//              B_k[a][b] = sum_l s_bl/64 sum_g N8_a(g) D8_bl(g) A_g[l][k]
//            with N8_a = prod_m (1 + q s_am sigma_m), D8_bl = prod_{m!=l}(...):
//            per direction m != l the factor pair (1 + q s_am sigma)(1 + q s_bm
//            sigma) is (4/3) + 2q s_am sigma when s_bm = s_am, else 2/3, so
//            the 8 columns take 4 distinct values per l (classes "same/diff"
//            in m1, m2), indexed by the relative corner d = p(a) ^ p(b) —
//            compile-time after unrolling.  Off-diagonal sums accumulate in
//            shared memory [k][slot][row], the diagonal in a register; no
//            atomics, fixed order (bitwise reproducible);
//   phase 4  warp-per-row coalesced write-out of the block's CSR rows.
// Equal to the reference's Gauss sums to rounding (w_g = 1, sum_c N_c = 1).
#include "elemcore.cuh"

namespace fpb {

constexpr int kHbP = 74;  // doubles per element record (72 + pad; 16-byte aligned, spreads banks)

// one (element, l, k) column: v[g] = A_g[l][k] -> H[s][U'] (see header)
template <int L>
__device__ __forceinline__ void hb_walsh_col(double* h) {
  constexpr double q = 0.5773502691896258;
  constexpr int m1 = L == 0 ? 1 : 0, m2 = L == 2 ? 1 : 2;
  double v[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) v[g] = h[g];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int g = 0; g < 8; ++g)
      if (!((g >> m) & 1)) {
        const double lo = v[g], hi = v[g | (1 << m)];
        v[g] = lo + hi;
        v[g | (1 << m)] = hi - lo;
      }
  double o[8];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int U = ((u & 1) ? (1 << m1) : 0) | ((u & 2) ? (1 << m2) : 0);
    const double f0 = v[U] * (1.0 / 64.0), f1 = v[U | (1 << L)] * (q / 64.0);
    o[u] = f0 - f1;      // s = -1
    o[4 + u] = f0 + f1;  // s = +1
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) h[t] = o[t];
}

template <int R>
__global__ void __launch_bounds__(3 * R, 1)
k_hex_grad_blocks(int maxinc, int rowcap, const int32_t* __restrict__ blk_rows,
                  const uint16_t* __restrict__ bloc, const uint2* __restrict__ bslot,
                  const int32_t* __restrict__ blk_eptr, const int32_t* __restrict__ blk_elems,
                  const int32_t* __restrict__ conn, const double* __restrict__ xyz4,
                  const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind, int64_t nnz,
                  int accumulate, double* __restrict__ out) {
  constexpr int NT = 3 * R;
  constexpr int RS = R + 1;  // padded row stride of the accumulators
  constexpr double q = 0.5773502691896258;
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x, tid = threadIdx.x;
  const int e0 = __ldg(blk_eptr + b), E = __ldg(blk_eptr + b + 1) - e0;
  double* const H = sm;                                  // [E][kHbP]
  double* const acc = sm + (((size_t)E * kHbP + 1) & ~(size_t)1);  // [3][rowcap][RS]
  int* const dslot = reinterpret_cast<int*>(acc + 3 * rowcap * RS);  // [R]

  for (int i = tid; i < 3 * rowcap * RS; i += NT) acc[i] = 0.0;

  // ---- phase 1: adjugates at the Gauss points --------------------------------
  for (int i = tid; i < E * 8; i += NT) {
    const int el = i >> 3, g = i & 7;
    const int e = __ldg(blk_elems + e0 + el);
    double x[8][3];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double r4[4];
      ld256(xyz4 + 4 * (int64_t)__ldg(conn + (int64_t)e * 8 + c), r4);
      x[c][0] = r4[0];
      x[c][1] = r4[1];
      x[c][2] = r4[2];
    }
    HexCoef hc;
    hex_coeffs(x, hc);
    double J[3][3];
    hex_jacobian(hc, g, J);
    double A[3][3];
    A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    double* h = H + el * kHbP + g;
#pragma unroll
    for (int l = 0; l < 3; ++l)
#pragma unroll
      for (int k = 0; k < 3; ++k) h[(l * 3 + k) * 8] = A[l][k];
  }
  __syncthreads();

  // ---- phase 2: Walsh transform + row-side contraction, in place -------------
  for (int i = tid; i < E * 9; i += NT) {
    const int lk = i / E, el = i - lk * E;  // consecutive lanes: consecutive elements
    double* h = H + el * kHbP + lk * 8;
    const int l = lk / 3;
    if (l == 0) hb_walsh_col<0>(h); else if (l == 1) hb_walsh_col<1>(h); else hb_walsh_col<2>(h);
  }
  __syncthreads();

  // ---- phase 3: rows --------------------------------------------------------
  const int k = tid / R, r = tid - k * R;
  const int row = __ldg(blk_rows + (int64_t)b * R + r);
  double diag = 0.0;
  if (row >= 0) {
    if (k == 0) {
      const int rlo = __ldg(rowptr + row), rhi = __ldg(rowptr + row + 1);
      int lo = rlo, hi = rhi;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(colind + mid) < row) lo = mid + 1; else hi = mid;
      }
      dslot[r] = lo - rlo;
    }
    double* const myacc = acc + k * rowcap * RS + r;
    const int64_t base = (int64_t)b * maxinc * R + r;
    for (int m = 0; m < maxinc; ++m) {
      const int u = __ldg(bloc + base + (int64_t)m * R);
      if (u == 0xffff) break;
      const uint2 w = __ldg(bslot + base + (int64_t)m * R);
      const uint64_t w64 = ((uint64_t)w.y << 32) | w.x;
      int a = 0;
#pragma unroll
      for (int c = 0; c < 8; ++c) a = ((w64 >> (8 * c)) & 0xff) == 0xff ? c : a;
      const int pa = hex_corner_p(a);
      const double sg0 = (pa & 1) ? 1.0 : -1.0, sg1 = (pa & 2) ? 1.0 : -1.0, sg2 = (pa & 4) ? 1.0 : -1.0;
      const double sg[3] = {sg0, sg1, sg2};
      const double* hu = H + u * kHbP + k * 8;
      // V[l][cls]: cls bit0 = m1 differs, bit1 = m2 differs (relative corner bits)
      double V[3][4];
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const int m1 = l == 0 ? 1 : 0, m2 = l == 2 ? 1 : 2;
        const double* hp = hu + l * 24 + (((pa >> l) & 1) ? 4 : 0);
        const double2 h01 = *reinterpret_cast<const double2*>(hp);
        const double2 h23 = *reinterpret_cast<const double2*>(hp + 2);
        const double s = sg[l];
        const double t1 = (2.0 * q) * sg[m1] * h01.y, t2 = (2.0 * q) * sg[m2] * h23.x;
        const double t3 = (4.0 * q * q) * (sg[m1] * sg[m2]) * h23.y;
        const double h0 = h01.x;
        V[l][3] = s * ((4.0 / 9.0) * h0);                                   // m1 diff, m2 diff
        V[l][2] = s * fma(2.0 / 3.0, t1, (8.0 / 9.0) * h0);                 // m1 same, m2 diff
        V[l][1] = s * fma(2.0 / 3.0, t2, (8.0 / 9.0) * h0);                 // m1 diff, m2 same
        V[l][0] = s * (fma(4.0 / 3.0, t1 + t2, (16.0 / 9.0) * h0) + t3);   // both same
      }
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        double val = 0.0;
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          const int m1 = l == 0 ? 1 : 0, m2 = l == 2 ? 1 : 2;
          const int cls = ((d >> m1) & 1) | (((d >> m2) & 1) << 1);
          const double t = V[l][cls];
          val = ((d >> l) & 1) ? val - t : val + t;  // s_bl = s_al * (-1)^{bit l of d}
        }
        if (d == 0) {
          diag += val;
        } else {
          const int bnode = hex_corner_p(pa ^ d);
          const int slot = (int)((w64 >> (8 * bnode)) & 0xff);
          myacc[slot * RS] += val;
        }
      }
    }
    acc[(k * rowcap + rowcap - 1) * RS + r] = diag;  // diagonal in the spare slot
  }
  __syncthreads();

  // ---- phase 4: coalesced write-out, one warp per (row, k) segment -----------
  const int warp = tid >> 5, lane = tid & 31;
  for (int seg = warp; seg < 3 * R; seg += NT / 32) {
    const int kk = seg / R, rr = seg - kk * R;
    const int rw = __ldg(blk_rows + (int64_t)b * R + rr);
    if (rw < 0) continue;
    const int rlo = __ldg(rowptr + rw), rlen = __ldg(rowptr + rw + 1) - rlo;
    const int ds = dslot[rr];
    const double* a = acc + kk * rowcap * RS + rr;
    double* o = out + kk * nnz + rlo;
    for (int j = lane; j < rlen; j += 32) {
      const double v = j == ds ? a[(rowcap - 1) * RS] : a[(j - (j > ds)) * RS];
      o[j] = accumulate ? o[j] + v : v;
    }
  }
}

template <int R>
static size_t hb_smem(int emax, int rowcap) {
  return ((((size_t)emax * kHbP + 1) & ~(size_t)1) + 3 * (size_t)rowcap * (R + 1)) * sizeof(double) +
         R * sizeof(int);
}

template <int R>
static int hb_launch(int nblocks, int maxinc, int rowcap, int emax, const int32_t* blk_rows, const uint16_t* bloc,
                     const uint2* bslot, const int32_t* blk_eptr, const int32_t* blk_elems, const int32_t* conn,
                     const double* xyz4, const int32_t* rowptr, const int32_t* colind, int64_t nnz, int accumulate,
                     double* out, cudaStream_t s) {
  const size_t smem = hb_smem<R>(emax, rowcap);
  FPB_REQUIRE(smem <= 227 * 1024, "hex brick block needs %zu bytes of shared memory", smem);
  FPB_CUDA(cudaFuncSetAttribute(k_hex_grad_blocks<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_hex_grad_blocks<R><<<nblocks, 3 * R, smem, s>>>(maxinc, rowcap, blk_rows, bloc, bslot, blk_eptr, blk_elems,
                                                    conn, xyz4, rowptr, colind, nnz, accumulate, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int64_t fpb_hex_blocks_smem(int rows_per_block, int emax, int rowcap) {
  if (rows_per_block == 128) return (int64_t)hb_smem<128>(emax, rowcap);
  if (rows_per_block == 64) return (int64_t)hb_smem<64>(emax, rowcap);
  return -1;
}

int fpb_assemble_hex_gradient_blocks(int nblocks, int rows_per_block, int maxinc, int rowcap, int emax,
                                     const int32_t* blk_rows, const uint16_t* bloc, const uint32_t* bslot,
                                     const int32_t* blk_eptr, const int32_t* blk_elems, const int32_t* conn,
                                     const double* xyz4, const int32_t* rowptr, const int32_t* colind, int64_t nnz,
                                     int accumulate, double* out, void* stream) {
  FPB_REQUIRE(rowcap >= 2 && rowcap <= 256, "row length %d out of range", rowcap);
  FPB_REQUIRE(emax >= 0 && emax < 0xffff, "block element count %d out of range", emax);
  if (nblocks <= 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  const uint2* bs = reinterpret_cast<const uint2*>(bslot);
  if (rows_per_block == 128)
    return hb_launch<128>(nblocks, maxinc, rowcap, emax, blk_rows, bloc, bs, blk_eptr, blk_elems, conn, xyz4,
                          rowptr, colind, nnz, accumulate, out, s);
  if (rows_per_block == 64)
    return hb_launch<64>(nblocks, maxinc, rowcap, emax, blk_rows, bloc, bs, blk_eptr, blk_elems, conn, xyz4,
                         rowptr, colind, nnz, accumulate, out, s);
  set_error("rows per block must be 64 or 128 (got %d)", rows_per_block);
  return FPB_ECONFIG;
}

}  // extern "C"
