// Row-owned continuity matrices B_x, B_y, B_z for TET04 by column pairs
// (timeloop.py:159-171: CONVECTION with unit e_k; _kernels.py:238-266).
//
// For an affine tet rotated so the row node i is local node 0 (even
// permutation, rows.cu), det grad N_p for the other three nodes is the cross
// product of the two remaining edge vectors in cyclic order,
//   det grad N_1 = e_2 x e_3,  det grad N_2 = e_3 x e_1,  det grad N_3 = e_1 x e_2,
// e_l = x_l - x_0, and B_k[i][j] = mN_0 sum_{tets on edge ij} (det grad N_j)[k].
// So row i's entry in column j is a sum of edge-vector cross products over
// the tets containing edge ij, and the diagonal is minus the sum of all of
// them (sum_p grad N_p = 0).  k_rows_nb accumulates each incidence into its
// three columns (nine shared-memory read-modify-writes per incidence);
// here every row walks a precomputed stream of (q, r) slot pairs sorted by
// target column, keeps the column's sum in registers and writes it once:
// six staged-coordinate loads per pair, no read-modify-write.
//
// Stream: SELL-32 over the incidence slices (rows.cu), three 16-bit words
// per incidence: q | r << 7 | last << 14 (q, r = off-diagonal slots of the
// two edge vectors, last = final pair of the current target column; the
// targets run 0, 1, 2, ... because every off-diagonal column has at least
// one pair — a column no incident element touches, e.g. a slab's
// ghost-shaped interface rows, gets the dummy pair (t, t) = 0).  Slice s
// holds pair_ptr[s + 1] - pair_ptr[s] words per row (its longest row, even):
// row 32 s + l, entry k at uint32 (pair_ptr[s] / 2 + k / 2) 32 + l, half
// k & 1 (two words per load); padding 0 (the pair (0, 0): adds an exact
// zero, stores nothing).  Rows longer than 128 entries use k_rows_nb.
//
// Column pairs are ordered around the edge's tet ring, so consecutive
// pairs share an edge vector (bit 15: reuse the previous r as q); the next
// pair's vectors are fetched before the current column test; finished
// columns go straight into the warp's linear output rows.  Config 2
// (B200): 0.196 ms vs 0.264 ms for k_rows_nb (profiles/r01v_pairs ..
// r01y_step); 24-word batches = one third of an interior row's 72 pairs.
#include <algorithm>
#include <cub/device/device_scan.cuh>

#include "elemcore.cuh"

namespace fpb {

constexpr int kPairMaxInc = 64;      // incidences per row the setup sort handles
#ifndef FPB_PAIR_CHAIN
#define FPB_PAIR_CHAIN 1  // ring-ordered columns: reuse the previous pair's r as q
#endif
#ifndef FPB_PAIR_PACK2
#define FPB_PAIR_PACK2 1  // two stream words per 32-bit load ([2 m0 + k / 2][lane][2]; 0.242 vs 0.250 ms on config 2)
#endif
// padding word = pair (0, 0), not last: e_0 x e_0 = 0 joins no column, so
// the hot loop needs no end-of-row test
constexpr uint16_t kPairPad = 0;

// Canonical stream: the pair stream shared by every interior row of a
// structured mesh (on the Kuhn box all interior rows have the same 15
// columns, 24 incidences and therefore the same 72 (q, r) words).  The host
// finds it as the most frequent row stream, verifies rows against it word by
// word, and slices whose 32 rows all match run the kernel with the stream
// read from constant memory (uniform across the warp) instead of 2 bytes
// per pair per row from HBM.
constexpr int kPairCanonMax = 512;
__constant__ uint16_t c_pair_canon[kPairCanonMax];

// Pass FILL = false: per-slice stream width (the slice's longest row,
// rounded up to even) into width[sl]; FILL = true: the words.
template <bool FILL>
__global__ void k_pair_stream(int32_t n, const int32_t* __restrict__ slice_ptr, const uint32_t* __restrict__ slots,
                              const int32_t* __restrict__ rowptr, const int64_t* __restrict__ pair_ptr,
                              int64_t* __restrict__ width, uint16_t* __restrict__ words, int* err) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nsl = ((int64_t)n + 31) / 32;
  if (row >= nsl * 32) return;
  const int64_t sl = row >> 5;
  const int lane = (int)(row & 31);
  const int m0 = slice_ptr[sl], m1 = slice_ptr[sl + 1];
  uint32_t key[3 * kPairMaxInc + 128];  // target << 16 | r << 8 | q (+ bit 24: chained, bit 25: last)
  int np = 0;
  if (row < n) {
    for (int m = m0; m < m1; ++m) {
      const uint32_t w = slots[(int64_t)m * 32 + lane];
      if (w == 0xffffffffu) break;
      if (m - m0 >= kPairMaxInc) {
        atomicExch(err, 1);
        break;
      }
      const uint32_t s1 = (w >> 8) & 0xff, s2 = (w >> 16) & 0xff, s3 = (w >> 24) & 0xff;
      if (s1 > 127 || s2 > 127 || s3 > 127) atomicExch(err, 1);
      key[np++] = s1 << 16 | s3 << 8 | s2;  // column of node 1: e_2 x e_3
      key[np++] = s2 << 16 | s1 << 8 | s3;  // node 2: e_3 x e_1
      key[np++] = s3 << 16 | s2 << 8 | s1;  // node 3: e_1 x e_2
    }
  }
  // stable insertion sort by target column (incidence order within a column)
  for (int i = 1; i < np; ++i) {
    const uint32_t k = key[i];
    int j = i - 1;
    while (j >= 0 && (key[j] >> 16) > (k >> 16)) {
      key[j + 1] = key[j];
      --j;
    }
    key[j + 1] = k;
  }
  // chain each column's pairs around its edge: (q1, q2), (q2, q3), ... —
  // the tets around edge ij form a ring (open at the boundary), so a pair
  // whose q is the previous pair's r reuses that node's edge vector from
  // registers (bit 15); the column's summation order is the ring order
  for (int c0 = 0; c0 < np;) {
    int c1 = c0 + 1;
    while (c1 < np && (key[c1] >> 16) == (key[c0] >> 16)) ++c1;
    // start at a pair whose q is no other pair's r (open chain), else c0
    int start = c0;
    for (int i = c0; i < c1; ++i) {
      bool has_pred = false;
      for (int j = c0; j < c1; ++j) has_pred |= j != i && ((key[j] >> 8) & 0xff) == (key[i] & 0xff);
      if (!has_pred) {
        start = i;
        break;
      }
    }
    uint32_t t = key[c0];
    key[c0] = key[start];
    key[start] = t;
    for (int i = c0 + 1; i < c1; ++i) {  // greedy: next pair continues the chain if one does
      const uint32_t want = (key[i - 1] >> 8) & 0xff;
      for (int j = i; j < c1; ++j)
        if ((key[j] & 0xff) == want) {
          t = key[i];
          key[i] = key[j];
          key[j] = t;
          key[i] |= 1u << 24;  // chained to its predecessor
          break;
        }
    }
    key[c1 - 1] |= 1u << 25;  // last pair of the column
    c0 = c1;
  }
  // the targets are implicit (0, 1, 2, ... in order), so a pattern column no
  // incident element touches (a slab's ghost-shaped interface rows) gets a
  // dummy pair (t, t): e_t x e_t = 0 exactly, and the column stores 0
  int total = np;
  if (row < n) {
    const int ncol = rowptr[row + 1] - rowptr[row] - 1;
    if (ncol > 128) atomicExch(err, 1);
    int have = 0;
    for (int i = 0; i < np; ++i) have += (i == 0 || ((key[i] >> 16) & 0xff) != ((key[i - 1] >> 16) & 0xff)) ? 1 : 0;
    const int missing = ncol - have;
    if (missing < 0 || np + missing > 3 * kPairMaxInc + 128) atomicExch(err, 1);
    if (missing > 0 && missing <= 128 && np + missing <= 3 * kPairMaxInc + 128) {
      // merge from the back: targets ncol-1 .. 0
      int src = np - 1, dst = np + missing - 1;
      for (int t = ncol - 1; t >= 0; --t) {
        bool found = false;
        while (src >= 0 && (int)((key[src] >> 16) & 0xff) == t) {
          key[dst--] = key[src--];
          found = true;
        }
        if (!found) key[dst--] = (uint32_t)t << 16 | (uint32_t)t << 8 | (uint32_t)t | 1u << 25;
      }
      total = np + missing;
    }
  }
  if constexpr (!FILL) {
    int wdt = (total + 1) & ~1;  // even: two words per 32-bit load
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wdt = max(wdt, __shfl_xor_sync(0xffffffffu, wdt, o));
    if (lane == 0) width[sl] = wdt;
    return;
  } else {
    const int64_t p0 = pair_ptr[sl];
    const int wdt = (int)(pair_ptr[sl + 1] - p0);
    for (int k = 0; k < wdt; ++k) {
      uint16_t v = kPairPad;
      if (k < total)
        v = (uint16_t)((key[k] & 0x7f) | ((key[k] >> 8) & 0x7f) << 7 | (key[k] & (1u << 25) ? 1u << 14 : 0u) |
                       (FPB_PAIR_CHAIN && (key[k] & (1u << 24)) ? 1u << 15 : 0u));
#if FPB_PAIR_PACK2
      words[((((p0 >> 1) + (k >> 1)) * 32 + lane) << 1) | (k & 1)] = v;
#else
      words[(p0 + k) * 32 + lane] = v;
#endif
    }
  }
}

#ifndef FPB_PAIR_W
#define FPB_PAIR_W 24  // stream words per prefetch batch (one TET04 interior row = 72 pairs)
#endif

// Shared memory: the relative coordinates e_s of every thread's
// off-diagonal slots ([s][field][thread], region X) and the warp's three
// output row blocks (linear, one per matrix), where each finished column is
// stored once at its CSR position.
template <bool CANON>
__global__ void __launch_bounds__(32, 1)
k_rows_pairs(int32_t n, int32_t row0, const int32_t* __restrict__ slist, const int32_t* __restrict__ rlist,
             int32_t nlist, int canon_len, const int64_t* __restrict__ pair_ptr, const uint16_t* __restrict__ words,
             const double* __restrict__ xyz4, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
             int64_t nnz, int rowcap, int accumulate, double* __restrict__ out) {
  constexpr int DIM = 3, T = 32;
  constexpr int SS = DIM * T;  // doubles per slot in each region
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  // rows: a row list (rlist: any rows, each reading its own stream; the
  // generic rows next to the Kuhn kernel's), the 32-row slice slist[block],
  // else row0 + 32 block
  const bool listed = rlist != nullptr;
  int row;
  bool live;
  if (listed) {
    const int64_t i = (int64_t)blockIdx.x * T + tid;
    live = i < nlist;
    row = __ldg(rlist + (live ? i : 0));
  } else {
    row = (slist ? __ldg(slist + blockIdx.x) : row0 / T + blockIdx.x) * T + tid;
    live = row < n;
  }
  const int lane = row & 31;
  const int64_t p0 = CANON ? 0 : __ldg(pair_ptr + (row >> 5));
  // stream words of the slice
  const int k1 = !live ? 0 : CANON ? canon_len : (int)(__ldg(pair_ptr + (row >> 5) + 1) - p0);
  int rlo = 0, rlen = 0;
  double x0[DIM] = {0.0, 0.0, 0.0};
  if (live) {
    rlo = __ldg(rowptr + row);
    rlen = __ldg(rowptr + row + 1) - rlo;
    double r4[4];
    ld256(xyz4 + 4 * (int64_t)row, r4);
#pragma unroll
    for (int d = 0; d < DIM; ++d) x0[d] = r4[d];
  }
  const int nslot = rowcap > 1 ? rowcap - 1 : 1;
  double* __restrict__ X = sm + tid;                    // [s][d][thread]
  // the warp's output rows, one linear buffer per matrix: entry (row, c) at
  // rlo - base + c, so finished columns land where the coalesced write-out
  // reads them (no intermediate copy)
  double* __restrict__ Bo = sm + nslot * SS;          // [3][32 rowcap]
  const int bstride = 32 * rowcap;
  const int base = __shfl_sync(0xffffffffu, rlo, 0);
  const int boff = listed ? tid * rowcap : rlo - base;  // this row's first entry in Bo

  // ---- pair stream: the first two batches are requested before staging so
  // their latency hides behind it ----
  const double mN0 = refmN<FPB_TET04>(0);
  double acc[DIM] = {0.0, 0.0, 0.0}, tot[DIM] = {0.0, 0.0, 0.0};
  int target = 0;
  constexpr int kW = FPB_PAIR_W;
  uint16_t wc[kW], wn[kW];
#if FPB_PAIR_PACK2
  const uint32_t* wp = CANON ? nullptr : reinterpret_cast<const uint32_t*>(words) + (p0 >> 1) * 32 + lane;
  auto ld_w = [&](int k, uint16_t (&w)[kW]) {
    if constexpr (CANON) {  // uniform across the warp: constant-cache broadcast
#pragma unroll
      for (int j = 0; j < kW; ++j) w[j] = k + j < k1 ? c_pair_canon[k + j] : kPairPad;
      return;
    }
#pragma unroll
    for (int j = 0; j < kW; j += 2) {
      const uint32_t v = k + j < k1 ? __ldg(wp + (int64_t)((k + j) >> 1) * 32) : 0u;
      w[j] = (uint16_t)(v & 0xffffu);
      w[j + 1] = (uint16_t)(v >> 16);
    }
  };
#else
  const uint16_t* wp = words + p0 * 32 + lane;
  auto ld_w = [&](int k, uint16_t (&w)[kW]) {
#pragma unroll
    for (int j = 0; j < kW; ++j) w[j] = k + j < k1 ? __ldg(wp + (int64_t)(k + j) * 32) : kPairPad;
  };
#endif
  ld_w(0, wc);
  ld_w(kW, wn);
  // ---- stage the neighbours' edge vectors e_s = x_s - x_0 ----
#ifndef FPB_PAIR_STAGE
#define FPB_PAIR_STAGE 8
#endif
  constexpr int kStage = FPB_PAIR_STAGE;  // neighbour records in flight per staging batch
  int dslot = rlen - 1;
  {
    int s = 0;
    for (int c0 = 0; c0 < rlen; c0 += kStage) {
      int col[kStage];
      double rx[kStage][4];
#pragma unroll
      for (int j = 0; j < kStage; ++j) col[j] = c0 + j < rlen ? __ldg(colind + rlo + c0 + j) : -1;
#pragma unroll
      for (int j = 0; j < kStage; ++j)
        if (col[j] >= 0 && col[j] != row) ld256(xyz4 + 4 * (int64_t)col[j], rx[j]);
#pragma unroll
      for (int j = 0; j < kStage; ++j) {
        if (col[j] < 0) continue;
        if (col[j] == row) {
          dslot = c0 + j;
          continue;
        }
#pragma unroll
        for (int d = 0; d < DIM; ++d) X[s * SS + d * T] = rx[j][d] - x0[d];
        ++s;
      }
    }
  }

  // ---- walk the pair stream: column sums in registers ----
  // software-pipelined: the edge vectors of pair j + 1 are requested before
  // pair j's column test, so the shared-memory latency overlaps the FP64
  // work and the (rare) column store
  double a[DIM], b[DIM];
  auto fetch = [&](uint32_t w, const double (&pbv)[DIM], double (&na)[DIM], double (&nb)[DIM]) {
    const int q = w & 0x7f, r = (w >> 7) & 0x7f;
#pragma unroll
    for (int d = 0; d < DIM; ++d) nb[d] = X[r * SS + d * T];
    if (FPB_PAIR_CHAIN && (w & (1u << 15))) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) na[d] = pbv[d];
    } else {
#pragma unroll
      for (int d = 0; d < DIM; ++d) na[d] = X[q * SS + d * T];
    }
  };
  {
    const double z[DIM] = {0.0, 0.0, 0.0};
    fetch(wc[0], z, a, b);
  }
  for (int k = 0; k < k1; k += kW) {
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const uint32_t w = wc[j];
      const uint32_t wnext = j + 1 < kW ? wc[j + 1] : wn[0];
      double na[DIM], nb[DIM];
      fetch(wnext, b, na, nb);
      acc[0] += a[1] * b[2] - a[2] * b[1];
      acc[1] += a[2] * b[0] - a[0] * b[2];
      acc[2] += a[0] * b[1] - a[1] * b[0];
      if (w & (1u << 14)) {  // column finished: store once, fold into the diagonal
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          Bo[d * bstride + boff + target + (target >= dslot)] = mN0 * acc[d];
          tot[d] += acc[d];
          acc[d] = 0.0;
        }
        ++target;
      }
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        a[d] = na[d];
        b[d] = nb[d];
      }
    }
#pragma unroll
    for (int j = 0; j < kW; ++j) wc[j] = wn[j];
    ld_w(k + 2 * kW, wn);
  }
  double dacc[DIM];
#pragma unroll
  for (int d = 0; d < DIM; ++d) dacc[d] = -(mN0 * tot[d]);

  // ---- coalesced write-out of the warp's rows (diagonal added now) ----
  const int wlane = tid & 31;
  int wend = live ? rlo + rlen : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wend = max(wend, __shfl_xor_sync(0xffffffffu, wend, o));
  const int span = wend - base;  // <= 32 rowcap
  if (live) {
#pragma unroll
    for (int k = 0; k < DIM; ++k) Bo[k * bstride + boff + dslot] = dacc[k];
  }
  __syncwarp();
  if (!listed) {
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      double* o = out + k * nnz + base;
      for (int q = wlane; q < span; q += 32) {
        const double v = Bo[k * bstride + q];
        o[q] = accumulate ? o[q] + v : v;
      }
    }
  } else {  // listed rows are not consecutive: row by row (Bo slot rr rowcap)
    for (int rr = 0; rr < 32; ++rr) {
      const int lo = __shfl_sync(0xffffffffu, rlo, rr), len = __shfl_sync(0xffffffffu, rlen, rr);
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        double* o = out + k * nnz + lo;
        for (int q = wlane; q < len; q += 32) {  // len = 0 for padding lanes
          const double v = Bo[k * bstride + rr * rowcap + q];
          o[q] = accumulate ? o[q] + v : v;
        }
      }
    }
  }
}


// ---- compile-time Kuhn stream --------------------------------------------
// The canonical stream of an interior row of the generator's Kuhn TET04 box
// (mesh.py:212-213, :268-282: 24 tets around every interior node, 14
// neighbours, 72 pairs), as the stream builder above emits it (dumped with
// tools/pair_canon_dump.py).  The host uses this kernel only when the
// detected canonical stream equals this table word for word
// (fpb_pair_kuhn_table), so rows are still verified against the real
// pattern.  With the pairs known at compile time the 14 edge vectors live in
// registers and the walk is straight-line FP64 (no stream loads, no
// shared-memory edge fetches, no decode).
constexpr int kKuhnWords = 72, kKuhnCols = 14, kKuhnDiag = 7;
__host__ __device__ constexpr uint16_t kuhn_word(int i) {
  constexpr uint16_t t[kKuhnWords] = {
      0x0083, 0x8281, 0x8205, 0x8304, 0x8106, 0xc182, 0x0180, 0x8383, 0x8287, 0xc005, 0x0300, 0x8406,
      0x8188, 0xc003, 0x0001, 0x8100, 0x8402, 0x8488, 0x8389, 0xc087, 0x0280, 0x8505, 0x830a, 0xc006,
      0x0004, 0x8080, 0x8381, 0x8587, 0x850b, 0xc20a, 0x0002, 0x8200, 0x8504, 0x860a, 0x840c, 0xc108,
      0x0181, 0x8483, 0x8689, 0x858d, 0x828b, 0xc085, 0x0302, 0x8606, 0x868c, 0x848d, 0x8189, 0xc103,
      0x0187, 0x8403, 0x8688, 0xc38d, 0x0284, 0x8585, 0x868b, 0x860d, 0x830c, 0xc206, 0x028a, 0x8385,
      0x8687, 0xc50d, 0x0308, 0x8506, 0x868a, 0xc40d, 0x0487, 0x8409, 0x8608, 0x850c, 0x858a, 0xc38b};
  return t[i];
}


// acc += X[q] x X[r] with the pair taken in ascending order (the interior
// stream holds every face pair twice, once per adjacent tet and in opposite
// orders): the 36 distinct cross products become common subexpressions
// the compiler evaluates once.  Used by every Kuhn-stream kernel, so they
// stay bitwise equal to each other.
__device__ __forceinline__ void kuhn_pair_acc(const double (&X)[kKuhnCols][3], int q, int r, double (&acc)[3]) {
  const int a = q < r ? q : r, b = q < r ? r : q;  // compile-time after unrolling
  const double c0 = X[a][1] * X[b][2] - X[a][2] * X[b][1];
  const double c1 = X[a][2] * X[b][0] - X[a][0] * X[b][2];
  const double c2 = X[a][0] * X[b][1] - X[a][1] * X[b][0];
  if (q < r) {
    acc[0] += c0;
    acc[1] += c1;
    acc[2] += c2;
  } else {
    acc[0] -= c0;
    acc[1] -= c1;
    acc[2] -= c2;
  }
}

constexpr int kKuhnWarps = 2;  // warps (32-row slices) per CTA

#ifndef FPB_KUHN_MINB
#define FPB_KUHN_MINB 6
#endif
// BOX (R = nx + 1, L = (nx + 1)(ny + 1) > 0): the mesh is the generator's Kuhn
// box (assembly.py KuhnBox), whose interior rows hold the node and its 14
// neighbours at the offsets +-1, +-R, +-(1+R), +-L, +-(1+L), +-(R+L),
// +-(1+R+L) in ascending order: the neighbour ids are computed, not read
// from colind (one dependent load level and 4 B per entry less).
__host__ __device__ __forceinline__ int64_t kuhn_box_off(int t, int64_t R, int64_t L) {
  const int64_t o[7] = {1 + R + L, R + L, 1 + L, L, 1 + R, R, 1};
  return t < 7 ? -o[t] : o[13 - t];
}

template <bool BOX>
__global__ void __launch_bounds__(32 * kKuhnWarps, FPB_KUHN_MINB)
k_rows_pairs_kuhn(int32_t nrows, const int32_t* __restrict__ rows, const int32_t* __restrict__ rlos,
                  const int32_t* __restrict__ nbr, const double* __restrict__ xyz4,
                  const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind, int64_t nnz,
                  int accumulate, double* __restrict__ out, int64_t boxR = 0, int64_t boxL = 0, int nxi = 0,
                  int nyi = 0) {
  constexpr int DIM = 3, R = kKuhnCols + 1;  // entries per row
  __shared__ double Bo[kKuhnWarps][DIM][32 * R];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = ((int64_t)blockIdx.x * kKuhnWarps + warp) * 32;  // the warp's 32 list entries
  bool live;
  int row;
  if constexpr (BOX) {
    // interior node rows by arithmetic: warp -> (x segment, interior line
    // (j, k)), lane -> i; nrows = the number of warps
    const int64_t wg = i0 >> 5;
    if (wg >= nrows) return;
    const int segs = (nxi + 31) >> 5;
    const int64_t line = wg / segs;
    const int i = 1 + 32 * (int)(wg - line * segs) + lane;
    const int64_t j = 1 + line % nyi, k = 1 + line / nyi;
    live = i <= nxi;
    row = live ? (int)(i + boxR * j + boxL * k) : -1;
  } else {
    if (i0 >= nrows) return;
    live = i0 + lane < nrows;
    row = live ? __ldg(rows + i0 + lane) : -1;
  }
  // rlos / nbr (per list entry, nullable): the row's CSR start and its 14
  // neighbours ([14][nrows]) precomputed, so every load below is indexed by
  // the list position alone — one dependent level (-> coordinates) instead
  // of three (row -> rowptr -> colind -> coordinates)
  const int rlo = !live ? 0 : rlos ? __ldg(rlos + i0 + lane) : __ldg(rowptr + row);
  const int base = __shfl_sync(0xffffffffu, rlo, 0);
  // the diagonal sits at CSR offset kKuhnDiag of every canonical row (the
  // host checks it with the stream): off-diagonal slot t is offset t + (t >= 7)
  constexpr int dslot = kKuhnDiag;
  double x0[DIM] = {0.0, 0.0, 0.0}, X[kKuhnCols][DIM];
  if (live) {
    double r4[4];
    ld256(xyz4 + 4 * (int64_t)row, r4);
#pragma unroll
    for (int d = 0; d < DIM; ++d) x0[d] = r4[d];
#pragma unroll
    for (int t = 0; t < kKuhnCols; ++t) {
      const int64_t col = BOX ? row + kuhn_box_off(t, boxR, boxL)
                              : nbr ? __ldg(nbr + (int64_t)t * nrows + i0 + lane) : __ldg(colind + rlo + t + (t >= dslot));
      ld256(xyz4 + 4 * (int64_t)col, r4);
#pragma unroll
      for (int d = 0; d < DIM; ++d) X[t][d] = r4[d] - x0[d];
    }
  } else {
#pragma unroll
    for (int t = 0; t < kKuhnCols; ++t)
#pragma unroll
      for (int d = 0; d < DIM; ++d) X[t][d] = 0.0;
  }
  const double mN0 = refmN<FPB_TET04>(0);
  double acc[DIM] = {0.0, 0.0, 0.0}, tot[DIM] = {0.0, 0.0, 0.0};
  double* const bo = &Bo[warp][0][0];
  int target = 0;
#pragma unroll
  for (int i = 0; i < kKuhnWords; ++i) {
    const int w = kuhn_word(i);
    const int q = w & 0x7f, r = (w >> 7) & 0x7f;
    kuhn_pair_acc(X, q, r, acc);
    if (w & (1 << 14)) {  // column finished
      const int cpos = target + (target >= dslot);
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        bo[d * 32 * R + lane * R + cpos] = mN0 * acc[d];
        tot[d] += acc[d];
        acc[d] = 0.0;
      }
      ++target;
    }
  }
#pragma unroll
  for (int d = 0; d < DIM; ++d) bo[d * 32 * R + lane * R + dslot] = -(mN0 * tot[d]);
  __syncwarp();
  int nlive = live ? lane + 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nlive = max(nlive, __shfl_xor_sync(0xffffffffu, nlive, o));
  const int last = __shfl_sync(0xffffffffu, row, nlive - 1), first = __shfl_sync(0xffffffffu, row, 0);
  if (last - first == nlive - 1) {
    // consecutive rows (15 entries each): one contiguous CSR range per matrix
    const int span = nlive * R;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      double* o = out + d * nnz + base;
      for (int j = lane; j < span; j += 32) {
        const double v = bo[d * 32 * R + j];
        o[j] = accumulate ? o[j] + v : v;
      }
    }
  } else {
    // gaps (boundary rows between): two 15-entry rows per warp instruction
    const int half = lane >> 4, j = lane & 15;
    for (int r0 = 0; r0 < nlive; r0 += 2) {  // warp-uniform trip count (the shuffle needs every lane)
      const int rr = r0 + half;
      const int lo = __shfl_sync(0xffffffffu, rlo, rr & 31);
      if (rr < nlive && j < R) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          double* o = out + d * nnz + lo + j;
          const double v = bo[d * 32 * R + rr * R + j];
          *o = accumulate ? *o + v : v;
        }
      }
    }
  }
}


// ---- Kuhn box, z-marching interior lines -----------------------------------
// Same rows, values and order as k_rows_pairs_kuhn<true>, but each warp owns
// a 32-node segment of one interior node line (j) and walks the interior
// layers k of a z-chunk.  The coordinates of node rows j - 1 .. j + 1 over the
// segment's 34 node columns are staged per layer in the warp's shared-memory
// ring by cp.async two layers ahead, so the 14 edge vectors of every row
// come from shared memory and no load latency is exposed; the row's CSR
// start is one load per warp and layer.  Warps are independent (no
// barriers).
#ifndef FPB_KGRAD_WARPS
#define FPB_KGRAD_WARPS 1  // one warp per CTA, 6 CTAs/SM (33 KB of staging each)
#endif
constexpr int kGradWarps = FPB_KGRAD_WARPS;
#ifdef FPB_KGRAD_STCS  // streaming (evict-first) stores of the output runs: A/B only, 1.92 vs 1.36 ms at C5
#define FPB_KGRAD_STORE(p, v) __stcs((p), (v))
#else
#define FPB_KGRAD_STORE(p, v) (*(p) = (v))
#endif
#ifndef FPB_KGRAD_MINB
// CTAs per SM: 6 one-warp CTAs with the double-buffered TMA output staging
// (plain stores: 4 two-warp CTAs, ~249 registers, 8 warps/SM: 1.40 ms at C5
// vs 1.59 at 168 registers / 10 warps)
#define FPB_KGRAD_MINB 6
#endif
int g_tuning_kgrad_march = 1;  // fpb_set_tuning("kgrad_march", 0|1): z-marching lines (1) or the row kernel (0)
int g_tuning_kgrad_kchunk = 0;  // 0: from the grid size
int g_tuning_kgrad_bthreads = 128;  // threads per CTA of the Kuhn boundary-row kernel
constexpr int kGradStg = 4 * 3 * 3 * 34 + 2;  // [layer slot][node row][comp][34 columns] + 4 CSR starts (int)
// output staging per matrix: 32 rows x 15 entries + 2 doubles of padding, so
// the block can be shifted by one double to match the 16-byte phase of its
// CSR destination (TMA bulk stores need 16-byte aligned ends)
constexpr int kGradOut = 32 * (kKuhnCols + 1) + 2;
// output path: 0 = coalesced st.global from the staging buffer; 1 = one TMA
// bulk store per matrix and plane (single buffer: the next plane waits for
// the store to drain, C5 B_xyz 1.35 -> 1.44 ms); 2 = the same, double
// buffered (1.35 -> 1.29 ms; L1 wavefronts 80 -> 48 % of peak)
#ifndef FPB_KGRAD_TMA
#define FPB_KGRAD_TMA 2
#endif
__device__ __forceinline__ void g_cp8(double* smem_dst, const double* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}

__global__ void __launch_bounds__(32 * kGradWarps, FPB_KGRAD_MINB)
k_kuhn_grad_march(int nx, int ny, int nz, int kz0, int kz1, int kchunk, int64_t nwarps, const double* __restrict__ xyz4,
                  const int32_t* __restrict__ rowptr, int64_t nnz, int accumulate, double* __restrict__ out) {
  constexpr int DIM = 3, RE = kKuhnCols + 1;  // entries per row
  extern __shared__ __align__(16) double gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wg = (int64_t)blockIdx.x * kGradWarps + warp;
  if (wg >= nwarps) return;
  constexpr int NBUF = FPB_KGRAD_TMA == 2 ? 2 : 1;  // TMA 2: double-buffered output staging
  double* const stg = gsm + (size_t)warp * (kGradStg + NBUF * DIM * kGradOut);
  const int nxi = nx - 1, nyi = ny - 1;
  const int segs = (nxi + 31) >> 5;
  const int64_t per_chunk = (int64_t)segs * nyi;
  const int c = (int)(wg / per_chunk);
  const int rem = (int)(wg - (int64_t)c * per_chunk);
  const int j = 1 + rem / segs, s = rem - (rem / segs) * segs;
  const int i = 1 + 32 * s + lane;
  const int nlive = min(32, nxi - 32 * s);
  const bool live = lane < nlive;
  const int kb = kz0 + c * kchunk, ke = min(kz1 + 1, kb + kchunk);  // node planes [kz0, kz1]
  const int64_t R = nx + 1, L = R * (ny + 1);

  int* const rlo_s = reinterpret_cast<int*>(stg + 4 * 3 * 3 * 34);  // [layer slot]
  auto stage = [&](int kl) {  // node layer kl, node rows j - 1 .. j + 1, columns 32 s .. 32 s + 33
    double* t0 = stg + (kl & 3) * 3 * 3 * 34;
    if (lane == 0 && kl >= kb && kl < ke) {  // the segment's CSR start in layer kl (4-byte cp.async)
      const unsigned d = (unsigned)__cvta_generic_to_shared(rlo_s + (kl & 3));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(rowptr + (1 + 32 * s) + R * j + L * kl)
                   : "memory");
    }
    for (int q = lane; q < 34; q += 32) {
      const int col = 32 * s + q;
      if (col <= nx) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double* src = xyz4 + 4 * (col + R * (j - 1 + r) + L * kl);
          double* t = t0 + r * 3 * 34 + q;
          g_cp8(t, src);
          g_cp8(t + 34, src + 1);
          g_cp8(t + 68, src + 2);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  stage(kb - 1);
  stage(kb);
  stage(kb + 1);
  const double mN0 = refmN<FPB_TET04>(0);
  constexpr int dslot = kKuhnDiag;
  for (int k = kb; k < ke; ++k) {
    if (k + 2 <= nz) stage(k + 2);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
#if FPB_KGRAD_TMA
    // the bulk stores that last used this plane's staging buffer (two planes
    // back when double-buffered, the previous plane otherwise) must have read it
    if (lane == 0) {
      if (NBUF == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
#endif
    __syncwarp();
    double* const bo0 = stg + kGradStg + (NBUF == 2 ? (k & 1) * DIM * kGradOut : 0);
    const int base = rlo_s[k & 3];
    // per matrix d: staging block at bo0 + d kGradOut, shifted by the CSR
    // destination's 16-byte phase (one double when its address is odd in doubles)
    int sh[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d)
      sh[d] = FPB_KGRAD_TMA && !accumulate ? (int)((reinterpret_cast<uintptr_t>(out + d * nnz + base) >> 3) & 1) : 0;
    double x0[DIM], X[kKuhnCols][DIM];
    {
      const double* c0 = stg + (k & 3) * 3 * 3 * 34 + 1 * 3 * 34 + lane + 1;
#pragma unroll
      for (int d = 0; d < DIM; ++d) x0[d] = c0[d * 34];
#pragma unroll
      for (int t = 0; t < kKuhnCols; ++t) {
        // neighbour offsets in ascending node order (kuhn_box_off): (di, dj, dk)
        constexpr int8_t off[14][3] = {{-1, -1, -1}, {0, -1, -1}, {-1, 0, -1}, {0, 0, -1}, {-1, -1, 0},
                                       {0, -1, 0},   {-1, 0, 0},  {1, 0, 0},   {0, 1, 0},  {1, 1, 0},
                                       {0, 0, 1},    {1, 0, 1},   {0, 1, 1},   {1, 1, 1}};
        const double* cp = stg + ((k + off[t][2]) & 3) * 3 * 3 * 34 + (1 + off[t][1]) * 3 * 34 + lane + 1 + off[t][0];
#pragma unroll
        for (int d = 0; d < DIM; ++d) X[t][d] = cp[d * 34] - x0[d];
      }
    }
    double acc[DIM] = {0.0, 0.0, 0.0}, tot[DIM] = {0.0, 0.0, 0.0};
    int target = 0;
#pragma unroll
    for (int q8 = 0; q8 < kKuhnWords; ++q8) {
      const int w = kuhn_word(q8);
      const int q = w & 0x7f, r = (w >> 7) & 0x7f;
      kuhn_pair_acc(X, q, r, acc);
      if (w & (1 << 14)) {  // column finished
        const int cpos = target + (target >= dslot);
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          bo0[d * kGradOut + sh[d] + lane * RE + cpos] = mN0 * acc[d];
          tot[d] += acc[d];
          acc[d] = 0.0;
        }
        ++target;
      }
    }
#pragma unroll
    for (int d = 0; d < DIM; ++d) bo0[d * kGradOut + sh[d] + lane * RE + dslot] = -(mN0 * tot[d]);
#if FPB_KGRAD_TMA
    // every writer makes its staging stores visible to the async proxy
    // before lane 0 hands the block to the TMA unit
    if (!accumulate) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
    __syncwarp();
    // the segment's rows are consecutive (15 entries each): one contiguous CSR range per matrix
    const int span = nlive * RE;
    if (FPB_KGRAD_TMA && !accumulate) {
      // one TMA bulk store per matrix for the 16-byte aligned middle of the
      // range; an unaligned first / last double by plain stores (lane 0)
      if (lane == 0) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          double* o = out + d * nnz + base;
          const double* b = bo0 + d * kGradOut + sh[d];
          const int h = sh[d];                 // 0 or 1 leading double
          const int nb = ((span - h) >> 1) << 1;  // doubles in the bulk part
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
      }
    } else {
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double* o = out + d * nnz + base;
        for (int q = lane; q < span; q += 32) {
          const double v = bo0[d * kGradOut + q];
          if (accumulate) o[q] += v;
          else FPB_KGRAD_STORE(o + q, v);
        }
      }
    }
    (void)live;
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#if FPB_KGRAD_TMA
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
}

// ---- Kuhn box, boundary rows -----------------------------------------------
// A boundary node of the Kuhn box keeps the subset of the interior stream
// whose tets exist: word (target t, pair q, r) belongs to the tet {node, t,
// q, r}, which lies in the cell at offset min(0, off_t, off_q, off_r) per
// axis; the word counts iff that cell is inside the box.  The row's columns
// are the neighbours with at least one counting word, in ascending order
// (the t order), the diagonal among them — so the CSR slot of column t is a
// popcount.  Values equal the generic pair-stream kernel's to rounding (the
// summation order is the interior stream's).
__host__ __device__ constexpr int kuhn_off3(int t, int d) {
  // (di, dj, dk) of neighbour t in ascending node order (kuhn_box_off)
  return d == 0 ? ((t == 0 || t == 2 || t == 4 || t == 6) ? -1 : (t == 7 || t == 9 || t == 11 || t == 13) ? 1 : 0)
       : d == 1 ? ((t == 0 || t == 1 || t == 4 || t == 5) ? -1 : (t == 8 || t == 9 || t == 12 || t == 13) ? 1 : 0)
                : ((t <= 3) ? -1 : (t >= 10) ? 1 : 0);
}
__host__ __device__ constexpr int cmin0(int a, int b, int c) { return (a < b ? (a < c ? a : c) : (b < c ? b : c)) < 0 ? -1 : 0; }

#ifndef FPB_KGRAD_BMINB
#define FPB_KGRAD_BMINB 4
#endif
__global__ void __launch_bounds__(128, FPB_KGRAD_BMINB)
k_kuhn_grad_boundary(int32_t nrows, const int32_t* __restrict__ rows, int nx, int ny, int nz, int vk0, int vk1,
                     const double* __restrict__ xyz4, const int32_t* __restrict__ rowptr, int64_t nnz,
                     int accumulate, double* __restrict__ out) {
  constexpr int DIM = 3;
  const int64_t R = nx + 1, L = R * (ny + 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nrows; e += (int64_t)gridDim.x * blockDim.x) {
    const int row = __ldg(rows + e);
    const int k = (int)(row / L), rem = (int)(row - k * L), j = rem / (int)R, i = rem - j * (int)R;
    // the 8 cells around the node: bit (cx + 1) + 2 (cy + 1) + 4 (cz + 1)
    // cells in the box (they shape the CSR row) and cells integrated (layers
    // [vk0, vk1): a slab's own layers) — the latter contribute values
    unsigned cells = 0, vcells = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int ci = i + (b & 1) - 1, cj = j + ((b >> 1) & 1) - 1, ck = k + ((b >> 2) & 1) - 1;
      if (ci >= 0 && ci < nx && cj >= 0 && cj < ny && ck >= 0 && ck < nz) {
        cells |= 1u << b;
        if (ck >= vk0 && ck < vk1) vcells |= 1u << b;
      }
    }
    double x0[DIM], X[kKuhnCols][DIM];
    {
      double r4[4];
      ld256(xyz4 + 4 * (int64_t)row, r4);
#pragma unroll
      for (int d = 0; d < DIM; ++d) x0[d] = r4[d];
#pragma unroll
      for (int t = 0; t < kKuhnCols; ++t) {
        const int ii = i + kuhn_off3(t, 0), jj = j + kuhn_off3(t, 1), kk = k + kuhn_off3(t, 2);
        const bool ok = ii >= 0 && ii <= nx && jj >= 0 && jj <= ny && kk >= 0 && kk <= nz;
        if (ok) ld256(xyz4 + 4 * (row + kuhn_box_off(t, R, L)), r4);
#pragma unroll
        for (int d = 0; d < DIM; ++d) X[t][d] = ok ? r4[d] - x0[d] : 0.0;
      }
    }
    // columns are stored as they finish (their CSR slot is known by then:
    // the present columns before them, +1 past the diagonal), so no
    // per-column register copy is kept — 195 -> ~120 registers
    const double mN0 = refmN<FPB_TET04>(0);
    const int lo = __ldg(rowptr + row);
    double acc[DIM] = {0.0, 0.0, 0.0}, tot[DIM] = {0.0, 0.0, 0.0};
    unsigned present = 0;
    bool any = false;
    int target = 0;
#pragma unroll
    for (int q8 = 0; q8 < kKuhnWords; ++q8) {
      const int w = kuhn_word(q8);
      const int q = w & 0x7f, r = (w >> 7) & 0x7f;
      const int cb = (cmin0(kuhn_off3(target, 0), kuhn_off3(q, 0), kuhn_off3(r, 0)) + 1) +
                     2 * (cmin0(kuhn_off3(target, 1), kuhn_off3(q, 1), kuhn_off3(r, 1)) + 1) +
                     4 * (cmin0(kuhn_off3(target, 2), kuhn_off3(q, 2), kuhn_off3(r, 2)) + 1);
      if ((vcells >> cb) & 1u) {
        kuhn_pair_acc(X, q, r, acc);
      }
      if ((cells >> cb) & 1u) any = true;
      if (w & (1 << 14)) {  // column finished
        if (any) {
          const int cp = __popc(present) + (target >= kKuhnDiag ? 1 : 0);
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            double* o = out + d * nnz + lo + cp;
            const double v = mN0 * acc[d];
            *o = accumulate ? *o + v : v;
          }
          present |= 1u << target;
        }
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          tot[d] += acc[d];
          acc[d] = 0.0;
        }
        any = false;
        ++target;
      }
    }
    const int dpos = __popc(present & 0x7fu);
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      double* o = out + d * nnz + lo + dpos;
      const double dv = -(mN0 * tot[d]);
      *o = accumulate ? *o + dv : dv;
    }
  }
}
}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_pair_stream_build(int32_t n, const int32_t* slice_ptr, const uint32_t* slots, const int32_t* rowptr,
                          int64_t* pair_ptr, uint16_t* words, int64_t* total_h, void* stream) {
  FPB_REQUIRE(n >= 0 && slice_ptr && slots && rowptr && pair_ptr, "bad pair-stream arguments");
  cudaStream_t s = as_stream(stream);
  const int64_t nsl = ((int64_t)n + 31) / 32;
  int* err = nullptr;
  FPB_CUDA(cudaMallocAsync(&err, sizeof(int), s));
  FPB_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
  const unsigned grid = (unsigned)((nsl * 32 + 127) / 128);
  if (!words) {  // pass 1: slice widths -> pair_ptr (exclusive scan), *total_h
    FPB_CUDA(cudaMemsetAsync(pair_ptr, 0, sizeof(int64_t), s));
    if (nsl > 0) {
      k_pair_stream<false><<<grid, 128, 0, s>>>(n, slice_ptr, slots, rowptr, nullptr, pair_ptr + 1, nullptr, err);
      FPB_LAUNCH_CHECK();
      size_t tmp_bytes = 0;
      void* tmp = nullptr;
      cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, pair_ptr + 1, pair_ptr + 1, nsl, s);
      FPB_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
      FPB_CUDA(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, pair_ptr + 1, pair_ptr + 1, nsl, s));
      FPB_CUDA(cudaFreeAsync(tmp, s));
    }
    FPB_CUDA(cudaMemcpyAsync(total_h, pair_ptr + nsl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  } else if (nsl > 0) {  // pass 2: the words [pair_ptr[nsl] * 32]
    k_pair_stream<true><<<grid, 128, 0, s>>>(n, slice_ptr, slots, rowptr, pair_ptr, nullptr, words, err);
    FPB_LAUNCH_CHECK();
  }
  int h = 0;
  FPB_CUDA(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  FPB_CUDA(cudaFreeAsync(err, s));
  FPB_CUDA(cudaStreamSynchronize(s));
  if (h) {
    set_error("pair stream: a row has more than %d incidences or 128 entries", kPairMaxInc);
    return FPB_ECONFIG;
  }
  return FPB_OK;
}

int fpb_assemble_gradient_pairs(int32_t n, int32_t row0, int32_t row1, const int64_t* pair_ptr,
                                const uint16_t* words, const double* xyz4, const int32_t* rowptr,
                                const int32_t* colind, int64_t nnz, int rowcap, int accumulate, double* out,
                                void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  FPB_REQUIRE(pair_ptr && words && xyz4 && rowptr && colind && out && rowcap >= 2 && rowcap <= 129,
              "pair-stream gradient assembly needs the stream, the CSR pattern and rows <= 129 entries");
  FPB_REQUIRE(row0 >= 0 && row0 % 32 == 0 && row1 <= n && row0 <= row1,
              "row window [%d, %d) must start on a 32-row slice", row0, row1);
  if (row1 <= row0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  // edge vectors [rowcap - 1][3][32] + output rows [3][32 rowcap]
  const size_t smem = ((size_t)3 * (rowcap - 1) * 32 + (size_t)3 * 32 * rowcap) * sizeof(double);
  if (smem > 48 * 1024)
    FPB_CUDA(cudaFuncSetAttribute(k_rows_pairs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_rows_pairs<false><<<(unsigned)((row1 - row0 + 31) / 32), 32, smem, s>>>(
      row1, row0, nullptr, nullptr, 0, 0, pair_ptr, words, xyz4, rowptr, colind, nnz, rowcap, accumulate, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_assemble_gradient_pairs_rows(int32_t n, int32_t nrows, const int32_t* rows, const int64_t* pair_ptr,
                                     const uint16_t* words, const double* xyz4, const int32_t* rowptr,
                                     const int32_t* colind, int64_t nnz, int rowcap, int accumulate, double* out,
                                     void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  if (nrows <= 0) return FPB_OK;
  FPB_REQUIRE(rows && pair_ptr && words && xyz4 && rowptr && colind && out && rowcap >= 2 && rowcap <= 129,
              "pair-stream row-list assembly needs the stream, the CSR pattern and rows <= 129 entries");
  cudaStream_t s = as_stream(stream);
  const size_t smem = ((size_t)3 * (rowcap - 1) * 32 + (size_t)3 * 32 * rowcap) * sizeof(double);
  if (smem > 48 * 1024)
    FPB_CUDA(cudaFuncSetAttribute(k_rows_pairs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_rows_pairs<false><<<(unsigned)((nrows + 31) / 32), 32, smem, s>>>(n, 0, nullptr, rows, nrows, 0, pair_ptr, words,
                                                                      xyz4, rowptr, colind, nnz, rowcap, accumulate,
                                                                      out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_pair_kuhn_table(uint16_t* words_h) {
  for (int i = 0; i < kKuhnWords; ++i) words_h[i] = kuhn_word(i);
  return kKuhnWords;
}

int fpb_assemble_gradient_pairs_kuhn(int32_t nrows, const int32_t* rows, const int32_t* rlos, const int32_t* nbr,
                                     const double* xyz4, const int32_t* rowptr, const int32_t* colind, int64_t nnz,
                                     int accumulate, double* out, void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  FPB_REQUIRE(rows && xyz4 && rowptr && colind && out, "missing arrays for the Kuhn-stream kernel");
  if (nrows <= 0) return FPB_OK;
  const int64_t warps = ((int64_t)nrows + 31) / 32;
  k_rows_pairs_kuhn<false><<<(unsigned)((warps + kKuhnWarps - 1) / kKuhnWarps), 32 * kKuhnWarps, 0, as_stream(stream)>>>(
      nrows, rows, rlos, nbr, xyz4, rowptr, colind, nnz, accumulate, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_assemble_gradient_kuhn_boundary(int32_t nrows, const int32_t* rows, int nx, int ny, int nz, int vk0,
                                        int vk1, const double* xyz4, const int32_t* rowptr, int64_t nnz,
                                        int accumulate, double* out, void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  FPB_REQUIRE(rows && xyz4 && rowptr && out && nx >= 1 && ny >= 1 && nz >= 1, "bad Kuhn-boundary arguments");
  if (nrows <= 0) return FPB_OK;
  const int bt = g_tuning_kgrad_bthreads;
  k_kuhn_grad_boundary<<<grid_for(nrows, bt), bt, 0, as_stream(stream)>>>(nrows, rows, nx, ny, nz, vk0, vk1, xyz4,
                                                                          rowptr, nnz, accumulate, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_assemble_gradient_kuhn_lines(int nx, int ny, int nz, int kz0, int kz1, const double* xyz4,
                                     const int32_t* rowptr, int64_t nnz, int accumulate, double* out, void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  FPB_REQUIRE(xyz4 && rowptr && out && nx >= 2 && ny >= 2 && 1 <= kz0 && kz1 <= nz - 1,
              "bad Kuhn-line arguments (box %d x %d x %d, planes [%d, %d])", nx, ny, nz, kz0, kz1);
  if (kz1 < kz0) return FPB_OK;
  const int nxi = nx - 1, nyi = ny - 1, np = kz1 - kz0 + 1;
  // z-chunks: about four waves of 10 resident warps per SM, 4..32 layers each
  const int64_t lines = (int64_t)((nxi + 31) / 32) * nyi;
  const int kauto = (int)std::min<int64_t>(32, std::max<int64_t>(4, lines * np / (4 * 10 * kNumSMs)));
  const int kchunk = std::max(1, std::min(g_tuning_kgrad_kchunk > 0 ? g_tuning_kgrad_kchunk : kauto, np));
  const int nchunk = (np + kchunk - 1) / kchunk;
  const int64_t nwarps = lines * nchunk;
  const size_t smem = (size_t)kGradWarps * (kGradStg + (FPB_KGRAD_TMA == 2 ? 2 : 1) * 3 * kGradOut) * sizeof(double);
  FPB_CUDA(cudaFuncSetAttribute(k_kuhn_grad_march, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_kuhn_grad_march<<<(unsigned)((nwarps + kGradWarps - 1) / kGradWarps), 32 * kGradWarps, smem,
                      as_stream(stream)>>>(nx, ny, nz, kz0, kz1, kchunk, nwarps, xyz4, rowptr, nnz, accumulate, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_assemble_gradient_pairs_kuhn_box(int32_t nrows, const int32_t* rows, int nx, int ny, const double* xyz4,
                                         const int32_t* rowptr, int64_t nnz, int accumulate, double* out,
                                         void* stream) {
  if (g_tuning_kgrad_march && nx >= 2 && ny >= 2 && nrows > 0) {
    const int nxi = nx - 1, nyi = ny - 1;
    FPB_REQUIRE((int64_t)nrows % ((int64_t)nxi * nyi) == 0, "%d interior rows: not whole interior planes", nrows);
    const int nz = nrows / (nxi * nyi) + 1;
    return fpb_assemble_gradient_kuhn_lines(nx, ny, nz, 1, nz - 1, xyz4, rowptr, nnz, accumulate, out, stream);
  }
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  FPB_REQUIRE(rows && xyz4 && rowptr && out && nx >= 1 && ny >= 1, "bad Kuhn-box gradient arguments");
  if (nrows <= 0) return FPB_OK;
  const int64_t R = nx + 1, L = R * (ny + 1);
  const int nxi = nx - 1, nyi = ny - 1;
  FPB_REQUIRE(nxi >= 1 && nyi >= 1 && (int64_t)nrows % ((int64_t)nxi * nyi) == 0,
              "%d interior rows is not a whole number of interior node planes of %d x %d", nrows, nxi, nyi);
  const int64_t warps = (int64_t)(nrows / nxi) * ((nxi + 31) / 32);  // interior lines x segments
  k_rows_pairs_kuhn<true><<<(unsigned)((warps + kKuhnWarps - 1) / kKuhnWarps), 32 * kKuhnWarps, 0, as_stream(stream)>>>(
      (int32_t)warps, nullptr, nullptr, nullptr, xyz4, rowptr, nullptr, nnz, accumulate, out, R, L, nxi, nyi);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_pair_canon_set(const uint16_t* words_h, int len) {
  FPB_REQUIRE(len >= 0 && len <= kPairCanonMax && len % 2 == 0, "canonical stream length %d out of range", len);
  if (len) FPB_CUDA(cudaMemcpyToSymbol(c_pair_canon, words_h, (size_t)len * sizeof(uint16_t)));
  return FPB_OK;
}

int fpb_assemble_gradient_pairs_slices(int32_t n, int32_t nslices, const int32_t* slist, int canon_len,
                                       const int64_t* pair_ptr, const uint16_t* words, const double* xyz4,
                                       const int32_t* rowptr, const int32_t* colind, int64_t nnz, int rowcap,
                                       int accumulate, double* out, void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  if (nslices <= 0) return FPB_OK;
  FPB_REQUIRE(slist && xyz4 && rowptr && colind && out && rowcap >= 2 && rowcap <= 129,
              "pair-stream gradient assembly needs the slice list, the CSR pattern and rows <= 129 entries");
  FPB_REQUIRE(canon_len > 0 || (pair_ptr && words), "generic slices need the pair stream");
  FPB_REQUIRE(canon_len <= kPairCanonMax, "canonical stream too long");
  if (nslices <= 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  const size_t smem = ((size_t)3 * (rowcap - 1) * 32 + (size_t)3 * 32 * rowcap) * sizeof(double);
  if (canon_len > 0) {
    if (smem > 48 * 1024)
      FPB_CUDA(cudaFuncSetAttribute(k_rows_pairs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_rows_pairs<true><<<(unsigned)nslices, 32, smem, s>>>(n, 0, slist, nullptr, 0, canon_len, nullptr, nullptr,
                                                           xyz4, rowptr, colind, nnz, rowcap, accumulate, out);
  } else {
    if (smem > 48 * 1024)
      FPB_CUDA(cudaFuncSetAttribute(k_rows_pairs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_rows_pairs<false><<<(unsigned)nslices, 32, smem, s>>>(n, 0, slist, nullptr, 0, 0, pair_ptr, words, xyz4,
                                                            rowptr, colind, nnz, rowcap, accumulate, out);
  }
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

}  // extern "C"
