// HEX08 continuity matrices B_x, B_y, B_z (GRADIENT_XYZ = 3 x CONVECTION(e_k),
// timeloop.py:159-171, _kernels.py:238-266) with every element's Gauss-point
// geometry evaluated ONCE (the per-row kernel, rowsq.cu, re-evaluates it for
// each of the element's 8 rows).  Two passes:
//
//   k_hex_h      thread per element: J_g at the 8 Gauss points from the
//                sum-factorised coefficients (common.cuh), adjugate columns
//                A_g[l][k] = (det J Ji)[l][k], an 8-point Walsh-Hadamard
//                transform over the Gauss points F[U] = sum_g sigma^U(g) A_g,
//                contracted with the row-side factor of direction l:
//                  H[e][k][l][s][U'] = (F[U'] + s q F[U' + l]) / 64,
//                  s = -/+, U' in {0, m1, m2, m1m2} (m1 < m2 the other axes)
//                — 72 doubles per element, written once to an HBM scratch laid
//                out [72][nelem] (plane q = 24 k + 8 l + 4 s + U'), so that a
//                warp's lanes (consecutive elements / rows) read and write
//                contiguous 256-byte runs.
//   rows         thread per (row, k): for each incident element, the row's 8
//                entries from 4 H values per l —
//                  B_k[a][b] = sum_l s_bl/64 sum_g N8_a(g) D8_bl(g) A_g[l][k]
//                with N8_a = prod_m (1 + q s_am sigma_m), D8_bl = prod_{m!=l}
//                (1 + q s_bm sigma_m); per axis m != l the factor pair is
//                (4/3) + 2q s_am sigma when s_bm = s_am, else 2/3, so the 8
//                columns take 4 distinct values per l, indexed by the relative
//                corner d = p(a) ^ p(b) (p = corner sign bits).
//     canonical  rows whose 8 incidences and 27 columns follow the interior
//                pattern of the generator's Q1 box (mesh.py:265-267 corner
//                order, k-major cells, node ids i + (nx+1)(j + (ny+1)k)),
//                verified row by row at build time against the actual slot
//                bytes: the (incidence, corner) -> column map is a compile-time
//                table and the 27 sums live in registers;
//     generic    any other row (boundary, unstructured): blocks of 32 rows,
//                the column slot of each relative corner from the build
//                (slot bytes), off-diagonal sums in shared memory
//                [k][slot][row], the diagonal in a register, warp-per-row
//                coalesced write-out.
// Deterministic (fixed order, no atomics); equal to the reference's Gauss
// sums to rounding (w_g = 1, sum_c N_c = 1).
#include "elemcore.cuh"

namespace fpb {

constexpr double kHbQ = 0.5773502691896258;
constexpr int kHbRec = 72;  // H planes per element: q = [k][l][s][4]

// ---- element pass ----------------------------------------------------------
#ifndef FPB_HEXH_MINB
#define FPB_HEXH_MINB 4
#endif
#ifndef FPB_HEXR_PFM
#define FPB_HEXR_PFM 4  // cell lines L2-prefetched by the box row pass (bit my + 2 mz; 0 = off): C4 B_xyz 8.50 -> 7.93 ms (3, 12, 15: 8.51, 8.37, 9.70)
#endif
#ifndef FPB_HEXR_MINB
#define FPB_HEXR_MINB 4  // 8 CTAs of 96 threads at 80 registers: C4 B_xyz 8.78 -> 8.53 ms (5: 64 registers, 11.4 ms)
#endif
__global__ void __launch_bounds__(128, FPB_HEXH_MINB)
k_hex_h(int64_t nelem, const int32_t* __restrict__ conn, const double* __restrict__ xyz4, double* __restrict__ H) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nelem) return;
  HexCoef hc;
  {
    const int4 ca = __ldg(reinterpret_cast<const int4*>(conn + e * 8));
    const int4 cb = __ldg(reinterpret_cast<const int4*>(conn + e * 8 + 4));
    const int c8[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
    double x[8][3];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double r4[4];
      ld256(xyz4 + 4 * (int64_t)c8[c], r4);
      x[c][0] = r4[0];
      x[c][1] = r4[1];
      x[c][2] = r4[2];
    }
    hex_coeffs(x, hc);
  }
  double* const h = H + e;  // plane q at h[q * nelem]
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int m1 = l == 0 ? 1 : 0, m2 = l == 2 ? 1 : 2;
    const int l1 = (l + 1) % 3, l2 = (l + 2) % 3;
    double v[3][8];  // v[k][g] = A_g[l][k]
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      double J[3][3];
      hex_jacobian(hc, g, J);
      // adjugate row l: A[l][k] = J[k1][l1] J[k2][l2] - J[k1][l2] J[k2][l1] (cyclic)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int k1 = (k + 1) % 3, k2 = (k + 2) % 3;
        v[k][g] = J[k1][l1] * J[k2][l2] - J[k1][l2] * J[k2][l1];
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int g = 0; g < 8; ++g)
          if (!((g >> m) & 1)) {
            const double lo = v[k][g], hi = v[k][g | (1 << m)];
            v[k][g] = lo + hi;
            v[k][g | (1 << m)] = hi - lo;
          }
      double o[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int U = ((u & 1) ? (1 << m1) : 0) | ((u & 2) ? (1 << m2) : 0);
        const double f0 = v[k][U] * (1.0 / 64.0), f1 = v[k][U | (1 << l)] * (kHbQ / 64.0);
        o[u] = f0 - f1;      // s = -1
        o[4 + u] = f0 + f1;  // s = +1
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) h[(int64_t)(k * 24 + l * 8 + t) * nelem] = o[t];
    }
  }
}

// V[l][cls] of one (element, row corner pa, matrix k) from its H planes
// (hk = H + e + 24 k nelem): cls bit0 = the relative corner differs from a
// in m1, bit1 = differs in m2; the row-side sign s_al is folded in
__device__ __forceinline__ void hb_classes(const double* __restrict__ hk, int64_t nelem, int pa,
                                           double (&V)[3][4]) {
  constexpr double q = kHbQ;
  const double sg[3] = {(pa & 1) ? 1.0 : -1.0, (pa & 2) ? 1.0 : -1.0, (pa & 4) ? 1.0 : -1.0};
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int m1 = l == 0 ? 1 : 0, m2 = l == 2 ? 1 : 2;
    const double* hp = hk + (int64_t)(l * 8 + (((pa >> l) & 1) ? 4 : 0)) * nelem;
    const double h0 = __ldg(hp), h1 = __ldg(hp + nelem), h2 = __ldg(hp + 2 * nelem), h3 = __ldg(hp + 3 * nelem);
    const double s = sg[l];
    const double t1 = (2.0 * q) * sg[m1] * h1, t2 = (2.0 * q) * sg[m2] * h2;
    const double t3 = (4.0 * q * q) * (sg[m1] * sg[m2]) * h3;
    V[l][3] = s * ((4.0 / 9.0) * h0);                                  // m1 diff, m2 diff
    V[l][2] = s * fma(2.0 / 3.0, t1, (8.0 / 9.0) * h0);                // m1 same, m2 diff
    V[l][1] = s * fma(2.0 / 3.0, t2, (8.0 / 9.0) * h0);                // m1 diff, m2 same
    V[l][0] = s * (fma(4.0 / 3.0, t1 + t2, (16.0 / 9.0) * h0) + t3);  // both same
  }
}

// contribution of one element to the row's column at relative corner d
__device__ __forceinline__ double hb_value(const double (&V)[3][4], int d) {
  double val = 0.0;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int m1 = l == 0 ? 1 : 0, m2 = l == 2 ? 1 : 2;
    const int cls = ((d >> m1) & 1) | (((d >> m2) & 1) << 1);
    const double t = V[l][cls];
    val = ((d >> l) & 1) ? val - t : val + t;  // s_bl = s_al * (-1)^{bit l of d}
  }
  return val;
}

// canonical interior pattern: incidence m = the cell (i-1+mx, j-1+my, k-1+mz)
// (bits of m), where the row node is corner p(a) = m ^ 7; relative corner d
// moves by delta_dir = bit_dir(d) * (1 - 2 bit_dir(p(a))); CSR offset in the
// 27-entry row = 9 (dz+1) + 3 (dy+1) + (dx+1)
__host__ __device__ constexpr int hb_canon_slot(int m, int d) {
  const int pa = m ^ 7;
  int off = 0, mul = 1;
  for (int dir = 0; dir < 3; ++dir) {
    const int delta = ((d >> dir) & 1) ? (((pa >> dir) & 1) ? -1 : 1) : 0;
    off += mul * (delta + 1);
    mul *= 3;
  }
  return off;
}

// ---- canonical rows: thread per (row, k), R rows per CTA ---------------------
int g_tuning_hex_canon_rows = 32;  // fpb_set_tuning("hex_canon_rows", 32 | 64)

// FPB_HEXR_TMA: CTAs loop over row blocks (grid = resident CTAs); a block
// of consecutive rows leaves by one TMA bulk store per matrix
// (cp.async.bulk.global.shared::cta) from the staging buffer, shifted to the
// destination's 16-byte phase, instead of ld.shared + st.global per value;
// the buffer's next writes wait for the bulk read after the next block's
// H loads and arithmetic.  Measured (profiles/r02y_hextma): 11.9 ms for C4
// B_xyz against 7.84 with plain stores — the looping CTAs and their block
// barriers cost this latency-bound kernel far more than the LSU work the
// bulk stores save; off.
#ifndef FPB_HEXR_TMA
#define FPB_HEXR_TMA 0
#endif
template <int R, bool ACC, bool BOX>
__global__ void __launch_bounds__(3 * R, R == 32 ? 2 * FPB_HEXR_MINB : FPB_HEXR_MINB)
k_hex_rows_canon(int32_t nrows, const int32_t* __restrict__ rows, const int32_t* __restrict__ inc8,
                 const double* __restrict__ H, int64_t nelem, const int32_t* __restrict__ rowptr, int64_t nnz,
                 double* __restrict__ out, int bnx = 0, int bny = 0) {
  constexpr int NT = 3 * R;
  constexpr bool TMA = FPB_HEXR_TMA && !ACC;
  constexpr int KS = R * 27 + 2;  // per-matrix stage stride (+2: phase shift room, 16-byte multiple)
  __shared__ __align__(16) double stage[3 * KS];  // the CTA's output rows, for coalesced / bulk stores
  __shared__ int rlo_s[R];
  const int k = threadIdx.x / R, r = threadIdx.x - k * R;
  bool pending = false;  // a bulk store still reads the stage (thread 0)
  for (int32_t i0 = (TMA ? blockIdx.x : blockIdx.x) * R; i0 < nrows; i0 += (TMA ? gridDim.x * R : nrows)) {
  const int32_t i = i0 + r;
  const int nr = min(R, nrows - i0);
  const bool cons = __ldg(rows + i0 + nr - 1) - __ldg(rows + i0) == nr - 1;
  double a27[27];
  int row = 0;
  if (r < nr) {
    int el[8];
    row = __ldg(rows + i);
    if constexpr (BOX) {  // element ids of the generator's hex box (verified by the caller)
      const int ii = row % (bnx + 1), rj = row / (bnx + 1), jj = rj % (bny + 1), kk = rj / (bny + 1);
      const int e0 = (ii - 1) + bnx * ((jj - 1) + bny * (kk - 1));
#pragma unroll
      for (int m = 0; m < 8; ++m) el[m] = e0 + (m & 1) + bnx * (((m >> 1) & 1) + bny * (m >> 2));
#if FPB_HEXR_PFM
      // L2 prefetch of the H planes (this thread's matrix k) of the row's
      // own cell lines before the loads: bit (my + 2 mz) of FPB_HEXR_PFM
      // selects cell line (j-1+my, k-1+mz).  Fire-and-forget, no registers:
      // the whole batch of 128-byte runs is in flight at once instead of
      // one cell's twelve loads at a time.  Lanes 0 / 16 cover the warp's
      // two runs per plane.
      if ((r & 15) == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if ((FPB_HEXR_PFM >> c) & 1) {
            const double* hp = H + e0 + (int64_t)bnx * ((c & 1) + (int64_t)bny * (c >> 1)) + (int64_t)k * 24 * nelem;
#pragma unroll
            for (int q = 0; q < 24; ++q) asm volatile("prefetch.global.L2 [%0];" ::"l"(hp + (int64_t)q * nelem));
          }
      }
#endif
    } else {
#pragma unroll
      for (int m = 0; m < 8; ++m) el[m] = __ldg(inc8 + (int64_t)m * nrows + i);
    }
#pragma unroll
    for (int j = 0; j < 27; ++j) a27[j] = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      double V[3][4];
      hb_classes(H + el[m] + (int64_t)k * 24 * nelem, nelem, m ^ 7, V);
#pragma unroll
      for (int d = 0; d < 8; ++d) a27[hb_canon_slot(m, d)] += hb_value(V, d);
    }
  }
  if constexpr (TMA) {  // the previous block's stage readers (bulk or plain) are done
    if (threadIdx.x == 0 && pending) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
  }
  const int base0 = __ldg(rowptr + __ldg(rows + i0));
  int sh = 0;  // this thread's matrix: stage shift matching the destination's 16-byte phase
  if (TMA && cons) sh = (int)((reinterpret_cast<uintptr_t>(out + k * nnz + base0) >> 3) & 1);
  if (r < nr) {
    if (k == 0) rlo_s[r] = __ldg(rowptr + row);
#pragma unroll
    for (int j = 0; j < 27; ++j) stage[k * KS + sh + r * 27 + j] = a27[j];
  }
  if constexpr (TMA) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (cons) {
    // consecutive rows: each matrix's block is one contiguous CSR range of
    // 27 nr values (the stage's [r][27] order)
    if constexpr (TMA) {
      if (threadIdx.x == 0) {
        const int span = 27 * nr;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          double* o = out + kk * nnz + base0;
          const int h = (int)((reinterpret_cast<uintptr_t>(o) >> 3) & 1);
          const double* b = stage + kk * KS + h;
          const int nb = ((span - h) >> 1) << 1;
          if (h) o[0] = b[0];
          if (h + nb < span) o[span - 1] = b[span - 1];
          if (nb > 0) {
            const unsigned src = (unsigned)__cvta_generic_to_shared(b + h);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o + h), "r"(src),
                         "r"(nb * 8)
                         : "memory");
          }
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        pending = true;
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) {
        double* o = out + kk * nnz + base0;
        const double* sk = stage + kk * KS;
        for (int j = threadIdx.x; j < 27 * nr; j += NT) o[j] = ACC ? o[j] + sk[j] : sk[j];
      }
    }
  } else {
    // brick (Morton) order or boundary gaps: one 27-lane store per (row, k)
    // segment, two segments per warp instruction
    const int half = lane >= 16 ? 1 : 0, j = lane - 16 * half;  // lanes 0-15 / 16-31, 2 stores each
#pragma unroll
    for (int kk = 0; kk < 3; ++kk)
      for (int rr = 2 * warp + half; rr < nr; rr += NT / 16) {
        double* o = out + kk * nnz + rlo_s[rr];
        const double v0 = stage[kk * KS + rr * 27 + j];
        o[j] = ACC ? o[j] + v0 : v0;
        if (j < 11) {
          const double v1 = stage[kk * KS + rr * 27 + 16 + j];
          o[16 + j] = ACC ? o[16 + j] + v1 : v1;
        }
      }
  }
  if constexpr (!TMA) break;
  }
  if constexpr (TMA) {
    if (threadIdx.x == 0 && pending) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// ---- generic rows: blocks of 32 rows ----------------------------------------
constexpr int kHbGenRows = 32;

template <bool ACC>
__global__ void __launch_bounds__(3 * kHbGenRows)
k_hex_rows_generic(int maxinc, int rowcap, const int32_t* __restrict__ blk_rows, const int32_t* __restrict__ binc,
                   const uint2* __restrict__ bslot, const double* __restrict__ H, int64_t nelem,
                   const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind, int64_t nnz,
                   double* __restrict__ out) {
  constexpr int R = kHbGenRows, NT = 3 * R, RS = R + 1;
  extern __shared__ __align__(16) double acc[];                          // [3][rowcap][RS]
  int* const rmeta = reinterpret_cast<int*>(acc + 3 * rowcap * RS);  // [R][diag slot, rowptr, length]
  const int b = blockIdx.x, tid = threadIdx.x;
  for (int i = tid; i < 3 * rowcap * RS; i += NT) acc[i] = 0.0;
  __syncthreads();
  const int k = tid / R, r = tid - k * R;
  const int row = __ldg(blk_rows + (int64_t)b * R + r);
  if (row >= 0) {
    if (k == 0) {
      const int rlo = __ldg(rowptr + row), rhi = __ldg(rowptr + row + 1);
      int lo = rlo, hi = rhi;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(colind + mid) < row) lo = mid + 1; else hi = mid;
      }
      rmeta[3 * r] = lo - rlo;
      rmeta[3 * r + 1] = rlo;
      rmeta[3 * r + 2] = rhi - rlo;
    }
    double* const myacc = acc + k * rowcap * RS + r;
    double diag = 0.0;
    const int64_t base = (int64_t)b * maxinc * R + r;
    for (int m = 0; m < maxinc; ++m) {
      const int e = __ldg(binc + base + (int64_t)m * R);
      if (e < 0) break;
      // byte 0: sign bits p(a) of the row's own corner; byte d: the row's
      // off-diagonal slot of the corner p(a) ^ d (HexRowPlan)
      const uint2 w = __ldg(bslot + base + (int64_t)m * R);
      double V[3][4];
      hb_classes(H + e + (int64_t)k * 24 * nelem, nelem, (int)(w.x & 7u), V);
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        const double val = hb_value(V, d);
        if (d == 0) {
          diag += val;
        } else {
          const int slot = (int)(((d < 4 ? w.x : w.y) >> (8 * (d & 3))) & 0xffu);
          myacc[slot * RS] += val;
        }
      }
    }
    acc[(k * rowcap + rowcap - 1) * RS + r] = diag;  // diagonal in the spare slot
  } else if (k == 0) {
    rmeta[3 * r + 2] = 0;  // padding row: nothing to write
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  for (int rr = warp; rr < R; rr += NT / 32) {
    const int ds = rmeta[3 * rr], rlo = rmeta[3 * rr + 1], rlen = rmeta[3 * rr + 2];
    for (int j = lane; j < rlen; j += 32) {
      const int sl = j == ds ? rowcap - 1 : j - (j > ds);
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) {
        const double v = acc[(kk * rowcap + sl) * RS + rr];
        double* o = out + kk * nnz + rlo + j;
        *o = ACC ? *o + v : v;
      }
    }
  }
}

static size_t hb_generic_smem(int rowcap) {
  return 3 * (size_t)rowcap * (kHbGenRows + 1) * sizeof(double) + 3 * kHbGenRows * sizeof(int);
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_hex_canon_slots(int32_t* slots_h) {
  for (int m = 0; m < 8; ++m)
    for (int d = 0; d < 8; ++d) slots_h[m * 8 + d] = hb_canon_slot(m, d);
  return FPB_OK;
}

int fpb_hex_gradient_h(int64_t nelem, const int32_t* conn, const double* xyz4, double* H, void* stream) {
  FPB_REQUIRE(((uintptr_t)conn & 15) == 0, "conn must be 16-byte aligned");
  if (nelem <= 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  k_hex_h<<<(unsigned)((nelem + 127) / 128), 128, 0, s>>>(nelem, conn, xyz4, H);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_hex_gradient_rows(int32_t ncanon, const int32_t* canon_rows, const int32_t* canon_inc8, int32_t ngblocks,
                          int maxinc, int rowcap, const int32_t* gblk_rows, const int32_t* ginc,
                          const uint32_t* gslot, const double* H, int64_t nelem, const int32_t* rowptr,
                          const int32_t* colind, int64_t nnz, int accumulate, double* out, int box_nx, int box_ny,
                          void* stream) {
  FPB_REQUIRE(ngblocks == 0 || (rowcap >= 2 && rowcap <= 256), "row length %d out of range", rowcap);
  cudaStream_t s = as_stream(stream);
  if (ncanon > 0) {
    const int R = g_tuning_hex_canon_rows == 32 ? 32 : 64;
    unsigned grid = (unsigned)((ncanon + R - 1) / R);
    // TMA variant: CTAs loop over row blocks, one resident wave
    if (FPB_HEXR_TMA && !accumulate) grid = std::min<unsigned>(grid, kNumSMs * (R == 32 ? 2 * FPB_HEXR_MINB : FPB_HEXR_MINB));
#define FPB_HC(RR, AA, BB)                                                                                  \
  k_hex_rows_canon<RR, AA, BB><<<grid, 3 * RR, 0, s>>>(ncanon, canon_rows, canon_inc8, H, nelem, rowptr, nnz, out, \
                                                       box_nx, box_ny)
    const bool box = box_nx > 0 && box_ny > 0;
    if (R == 32) {
      if (box) {
        if (accumulate) FPB_HC(32, true, true); else FPB_HC(32, false, true);
      } else {
        if (accumulate) FPB_HC(32, true, false); else FPB_HC(32, false, false);
      }
    } else {
      if (accumulate) FPB_HC(64, true, false); else FPB_HC(64, false, false);
    }
#undef FPB_HC
    FPB_LAUNCH_CHECK();
  }
  if (ngblocks > 0) {
    const size_t smem = hb_generic_smem(rowcap);
    FPB_REQUIRE(smem <= 227 * 1024, "rows too long for the generic hex row kernel (%d entries)", rowcap);
    auto kern = accumulate ? k_hex_rows_generic<true> : k_hex_rows_generic<false>;
    FPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<ngblocks, 3 * kHbGenRows, smem, s>>>(maxinc, rowcap, gblk_rows, ginc,
                                                reinterpret_cast<const uint2*>(gslot), H, nelem, rowptr, colind, nnz,
                                                out);
    FPB_LAUNCH_CHECK();
  }
  return FPB_OK;
}

}  // extern "C"
