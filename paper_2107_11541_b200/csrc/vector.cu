// Solver vector kernels (sparse.py:78-130) and a device-resident Jacobi-PCG
// (krylov.py:27-89).  All reductions are deterministic: a fixed grid of
// kDotBlocks blocks reduces fixed strided slices in a fixed tree order, and
// the last block to finish (atomic ticket) folds the per-block partials in
// index order.  Repeated calls are therefore bitwise reproducible, like the
// reference's sequential loops (test_sparse.py:93-107).
#include <cub/device/device_scan.cuh>
#include "common.cuh"

namespace fpb {

// One resident wave of 512-thread blocks (2 per SM = 1024 threads): the
// fused SELL solver kernels hold 2 such blocks per SM, so a larger grid runs
// a second partial wave (profiles/r01o_sell: config-2 PCG 51.7 -> 47.2 us
// per iteration, BiCGSTAB 118 -> 108 us; 3 per SM is the worst of all)
#ifndef FPB_DOT_BLOCKS_PER_SM
#define FPB_DOT_BLOCKS_PER_SM 2
#endif
#ifndef FPB_DOT_THREADS
#define FPB_DOT_THREADS 512
#endif
constexpr int kDotBlocks = FPB_DOT_BLOCKS_PER_SM * kNumSMs;
constexpr int kDotThreads = FPB_DOT_THREADS;
// work layout (doubles): [0, 4*kDotBlocks) partials for up to 4 fused dots,
// then 4 ticket counters (as unsigned int in the low word).
constexpr int kWorkDoubles = 4 * kDotBlocks + 8;
#ifndef FPB_DOT_UNROLL
#define FPB_DOT_UNROLL 1
#endif

// alpha*x + y with the reference's two roundings (no DFMA contraction), so
// axpy is bitwise identical to sparse.py:96-99
__device__ __forceinline__ double axpy1(double a, double x, double y) {
  return __dadd_rn(__dmul_rn(a, x), y);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide fixed-order sum of NV values per thread; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
  __shared__ double sh[NV][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) sh[q][wid] = v[q];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double t = lane < nw ? sh[q][lane] : 0.0;
      v[q] = warp_sum(t);
    }
  }
}

// Publish this block's NV partials; returns true in thread 0 of the last
// block, with the grand totals in tot[] (summed in block-index order).
template <int NV>
__device__ __forceinline__ bool grid_finish(double (&v)[NV], double* work, int slot, double (&tot)[NV]) {
  __shared__ bool last;
  double* part = work;  // [NV][gridDim.x]
  unsigned int* ticket = reinterpret_cast<unsigned int*>(work + 4 * kDotBlocks) + 2 * slot;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) part[q * gridDim.x + blockIdx.x] = v[q];
    __threadfence();
    unsigned int t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  // last block: fold partials in fixed order with the whole block
  __threadfence();
  double s[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) s[q] = 0.0;
  // fixed assignment: thread t sums partials t, t+blockDim, ... in order
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
    for (int q = 0; q < NV; ++q) s[q] += __ldcg(part + q * gridDim.x + b);
  block_sum<NV>(s);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) tot[q] = s[q];
    *ticket = 0u;  // re-arm for the next launch
  }
  return threadIdx.x == 0;
}

// ---------------------------------------------------------------------------
// CSR SpMV, G lanes per row (G = 4/8/16 picked from the mean row length).
// ---------------------------------------------------------------------------
// G lanes per row; each lane owns entries lo+sub, lo+sub+G, ...  The first
// ITEMS of them are loaded together (all index/value loads issued before the
// dependent x gathers) — rows up to G*ITEMS entries (tet ~15, hex ~27) take
// one round trip; longer rows continue in a remainder loop.  Each lane sums
// its entries in ascending order, then a fixed xor-tree: deterministic.
template <int G, int ITEMS = (G == 16 ? 4 : 2)>
__device__ __forceinline__ double row_dot(const int32_t* __restrict__ rowptr,
                                          const int32_t* __restrict__ colind,
                                          const double* __restrict__ vals,
                                          const double* __restrict__ x, int64_t row, bool valid,
                                          int sub) {
  double acc = 0.0;
  if (valid) {
    const int lo = __ldg(rowptr + row), hi = __ldg(rowptr + row + 1);
    int col[ITEMS];
    double v[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const int k = lo + sub + it * G;
      col[it] = k < hi ? __ldcs(colind + k) : -1;
      v[it] = k < hi ? __ldcs(vals + k) : 0.0;
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it)
      if (col[it] >= 0) acc += v[it] * __ldg(x + col[it]);
    for (int k = lo + sub + ITEMS * G; k < hi; k += G) acc += __ldcs(vals + k) * __ldg(x + __ldcs(colind + k));
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
  return acc;
}

// R groups of 32/G rows per warp pass (rows base + r * 32/G + lane/G): every
// index/value load of the R groups is issued before the first dependent x
// gather (the single-group loop is latency-bound on large matrices); per
// row the same order as row_dot.  Returns the dots in out[r] (all lanes of
// a row group), row ids in row[r] (>= n: no row).
template <int G, int R, int ITEMS = (G == 16 ? 4 : 2)>
__device__ __forceinline__ void row_dot_grp(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                                            const double* __restrict__ vals, const double* __restrict__ x,
                                            int64_t base, int64_t n, int sub, int64_t (&row)[R],
                                            double (&out)[R]) {
  constexpr int RPW = 32 / G;
  int lo[R], hi[R], col[R][ITEMS];
  double v[R][ITEMS];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    row[r] = base + r * RPW + (threadIdx.x & 31) / G;
    lo[r] = row[r] < n ? __ldg(rowptr + row[r]) : 0;
    hi[r] = row[r] < n ? __ldg(rowptr + row[r] + 1) : 0;
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const int k = lo[r] + sub + it * G;
      col[r][it] = k < hi[r] ? __ldcs(colind + k) : -1;
      v[r][it] = k < hi[r] ? __ldcs(vals + k) : 0.0;
    }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double a = 0.0;
#pragma unroll
    for (int it = 0; it < ITEMS; ++it)
      if (col[r][it] >= 0) a += v[r][it] * __ldg(x + col[r][it]);
    for (int k = lo[r] + sub + ITEMS * G; k < hi[r]; k += G) a += __ldcs(vals + k) * __ldg(x + __ldcs(colind + k));
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o, G);
    out[r] = a;
  }
}

#ifndef FPB_FUSED_GROUPS
#define FPB_FUSED_GROUPS 4
#endif
// grid-stride loop over warp passes of R row groups
#define FPB_ROW_LOOP_R(G, R, n)                                                          \
  const int sub = threadIdx.x & ((G) - 1);                                              \
  const int64_t wid_ = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;           \
  const int64_t nwarps_ = ((int64_t)gridDim.x * blockDim.x) >> 5;                       \
  for (int64_t base_ = wid_ * (32 / (G)) * (R); base_ < (n); base_ += nwarps_ * (32 / (G)) * (R))

// Warp-uniform row loop: each warp covers 32/G consecutive rows per trip, so
// every lane of a warp runs the same number of trips (the shuffles above need
// the full warp).
#define FPB_ROW_LOOP(G, n)                                                               \
  const int sub = threadIdx.x & ((G) - 1);                                              \
  const int64_t wid_ = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;           \
  const int64_t nwarps_ = ((int64_t)gridDim.x * blockDim.x) >> 5;                       \
  for (int64_t base_ = wid_ * (32 / (G)); base_ < (n); base_ += nwarps_ * (32 / (G)))  \
    for (int64_t row = base_ + (threadIdx.x & 31) / (G), once_ = 0; once_ < 1; ++once_)

// Multi-group SpMV: each warp pass covers R groups of 32/G rows and issues
// every (column, value) load of all R groups before the first dependent x
// gather, so a warp keeps R times more bytes in flight across the
// load -> gather -> reduce chain (one group per pass was latency-bound at
// ~53 % of HBM on config 2; R = 4 reaches ~58 %).  Same per-row order: lane
// sums in ascending entry order, then the fixed xor tree.
template <int G, int R, int ITEMS = (G == 16 ? 4 : 2)>
__global__ void __launch_bounds__(256) k_spmv_r(int32_t n, const int32_t* __restrict__ rowptr,
                                                const int32_t* __restrict__ colind,
                                                const double* __restrict__ vals,
                                                const double* __restrict__ x, double* __restrict__ y) {
  constexpr int RPW = 32 / G;  // rows per group
  const int sub = threadIdx.x & (G - 1);
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = wid * RPW * R; base < n; base += nw * RPW * R) {
    int lo[R], hi[R], col[R][ITEMS];
    double v[R][ITEMS], acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t row = base + r * RPW + (threadIdx.x & 31) / G;
      lo[r] = row < n ? __ldg(rowptr + row) : 0;
      hi[r] = row < n ? __ldg(rowptr + row + 1) : 0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int it = 0; it < ITEMS; ++it) {
        const int k = lo[r] + sub + it * G;
        col[r][it] = k < hi[r] ? __ldcs(colind + k) : -1;
        v[r][it] = k < hi[r] ? __ldcs(vals + k) : 0.0;
      }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double a = 0.0;
#pragma unroll
      for (int it = 0; it < ITEMS; ++it)
        if (col[r][it] >= 0) a += v[r][it] * __ldg(x + col[r][it]);
      for (int k = lo[r] + sub + ITEMS * G; k < hi[r]; k += G) a += __ldcs(vals + k) * __ldg(x + __ldcs(colind + k));
      acc[r] = a;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o, G);
      const int64_t row = base + r * RPW + (threadIdx.x & 31) / G;
      if (row < n && sub == 0) y[row] = acc[r];
    }
  }
}

#ifndef FPB_SPMV_GROUPS
#define FPB_SPMV_GROUPS 4
#endif

// ---- SELL-32 copy of a CSR matrix (solver-side format) -------------------------
// Slice s = rows [32 s, 32 s + 32), width w_s = its longest row; entry k of
// row 32 s + l at sell_ptr[s] + 32 k + l (padding never read: each row stops
// at its own length).  One thread per row: every index / value load of a
// warp is one contiguous 128 / 256-byte line (no rowptr -> entry dependency,
// no idle lanes on short rows), and the row is summed in ascending column
// order with separately rounded products and sums — the reference's order
// and rounding (sparse.py:80-84), bit for bit.
__global__ void k_sell_width(int32_t n, const int32_t* __restrict__ rowptr, int64_t* __restrict__ width) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int len = row < n ? rowptr[row + 1] - rowptr[row] : 0;
  len = __reduce_max_sync(0xffffffffu, len);
  if ((threadIdx.x & 31) == 0 && (row >> 5) < ((int64_t)n + 31) / 32) width[row >> 5] = 32 * (int64_t)len;
}

// column storage: int32 columns (padding -1), or int16 offsets col - row
// (padding -32768) when every |col - row| < 32768 — 2 bytes less per entry
// of a bandwidth-bound SpMV (10 instead of 12 bytes per entry)
constexpr int kSellPad16 = -32768;

__global__ void k_sell_fill(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                            const double* __restrict__ vals, const int64_t* __restrict__ sell_ptr,
                            void* __restrict__ scol, int idx16, double* __restrict__ sval, int* bad) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // rows past n: padding only
  if (row >= ((int64_t)n + 31) / 32 * 32) return;
  const int64_t base = sell_ptr[row >> 5] + (row & 31);
  const int w = (int)((sell_ptr[(row >> 5) + 1] - sell_ptr[row >> 5]) >> 5);
  const int lo = row < n ? rowptr[row] : 0, len = row < n ? rowptr[row + 1] - lo : 0;
  for (int k = 0; k < w; ++k) {
    const int64_t at = base + 32 * (int64_t)k;
    if (scol && idx16) {
      int o = kSellPad16;
      if (k < len) {
        o = colind[lo + k] - (int)row;
        if (o <= kSellPad16 || o > 32767) atomicExch(bad, 1);
      }
      static_cast<int16_t*>(scol)[at] = (int16_t)o;
    } else if (scol) {
      static_cast<int32_t*>(scol)[at] = k < len ? colind[lo + k] : -1;
    }
    if (sval) sval[at] = k < len ? vals[lo + k] : 0.0;
  }
}

__global__ void k_max_offset(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                             int* out) {
  int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) m = max(m, abs(colind[k] - (int)i));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// entries per load batch (index + value loads of a batch in flight
// together, then its x gathers): 16 (tools/spmv_probe.py, tools/flow_probe.py:
// config-2 MASS 75 % of HBM vs 71 % with 8, pressure operator 0.111 vs
// 0.117 ms; configs 4 / 5 ~100 %)
#ifndef FPB_SELL_BATCH
#define FPB_SELL_BATCH 16
#endif
constexpr int kSellBatch = FPB_SELL_BATCH;
// row . x for one SELL row; rows of a warp are one slice (row >> 5
// uniform).  Padding entries are marked in the column array, so a row needs
// no length lookup: index and value loads of a batch go out together, then
// the x gathers of the valid entries.
template <typename IDX>
__device__ __forceinline__ int sell_col(const IDX* scol, int64_t at, int64_t row) {
  if constexpr (sizeof(IDX) == 2) {
    const int o = __ldcs(reinterpret_cast<const short*>(scol) + at);
    return o == kSellPad16 ? -1 : (int)row + o;
  } else {
    return __ldcs(scol + at);
  }
}

template <int B, typename IDX>
__device__ __forceinline__ double sell_row_dot(const int64_t* __restrict__ sell_ptr,
                                               const IDX* __restrict__ scol,
                                               const double* __restrict__ sval,
                                               const double* __restrict__ x, int64_t row) {
  const int64_t s0 = __ldg(sell_ptr + (row >> 5));
  const int w = (int)((__ldg(sell_ptr + (row >> 5) + 1) - s0) >> 5);
  const int64_t base = s0 + (row & 31);
  double acc = 0.0;
  for (int k0 = 0; k0 < w; k0 += B) {
    int c[B];
    double v[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const bool ok = k0 + j < w;
      c[j] = ok ? sell_col(scol, base + 32 * (int64_t)(k0 + j), row) : -1;
      v[j] = ok ? __ldcs(sval + base + 32 * (int64_t)(k0 + j)) : 0.0;
    }
    double xv[B];
#pragma unroll
    for (int j = 0; j < B; ++j) xv[j] = c[j] >= 0 ? __ldg(x + c[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < B; ++j)
      if (c[j] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[j], xv[j]));
  }
  return acc;
}

template <int B, typename IDX>
__global__ void __launch_bounds__(256) k_spmv_sell(int32_t n, const int64_t* __restrict__ sell_ptr,
                                                   const IDX* __restrict__ scol,
                                                   const double* __restrict__ sval,
                                                   const double* __restrict__ x, double* __restrict__ y) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if ((row & ~31LL) >= n) return;  // whole warps past the end
  const double a = sell_row_dot<B, IDX>(sell_ptr, scol, sval, x, row);
  if (row < n) y[row] = a;
}

__global__ void k_axpy(int64_t n, double alpha, const double* __restrict__ x,
                       const double* __restrict__ y, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = axpy1(alpha, x[i], y[i]);
}

__global__ void k_axpy2(int64_t n2, double alpha, const double2* __restrict__ x,
                        const double2* __restrict__ y, double2* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 a = __ldcs(x + i), b = __ldcs(y + i);
    __stcs(out + i, make_double2(axpy1(alpha, a.x, b.x), axpy1(alpha, a.y, b.y)));
  }
}

__global__ void __launch_bounds__(kDotThreads) k_dot(int64_t n, const double* __restrict__ x,
                                                     const double* __restrict__ y,
                                                     double* __restrict__ result, double* work) {
  double v[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
#if FPB_DOT_UNROLL > 1
  // FPB_DOT_UNROLL independent loads per operand in flight per trip
  constexpr int U = FPB_DOT_UNROLL;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    double a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = __ldcs(x + i + u * stride);
      b[u] = __ldcs(y + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) v[0] += a[u] * b[u];
  }
#endif
  for (; i < n; i += stride) v[0] += __ldcs(x + i) * __ldcs(y + i);
  block_sum<1>(v);
  double tot[1];
  if (grid_finish<1>(v, work, 0, tot)) *result = tot[0];
}

__global__ void k_diagonal(int32_t n, const int32_t* __restrict__ rowptr,
                           const int32_t* __restrict__ colind, const double* __restrict__ vals,
                           double* __restrict__ d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int lo = rowptr[i], hi = rowptr[i + 1], end = hi;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (colind[mid] < i) lo = mid + 1; else hi = mid;
    }
    d[i] = (lo < end && colind[lo] == i) ? vals[lo] : 0.0;
  }
}

__global__ void k_row_sums(int32_t n, const int32_t* __restrict__ rowptr,
                           const double* __restrict__ vals, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) s += vals[k];
    out[i] = s;
  }
}

// ---------------------------------------------------------------------------
// Device-resident PCG.  state: [0] rz, [1] bnorm, [2] tol, [3] status,
// [4] iterations, [5] relres, [6] pq, [7] beta
// ---------------------------------------------------------------------------
enum { S_RZ = 0, S_BNORM, S_TOL, S_STATUS, S_IT, S_RELRES, S_PQ, S_BETA };

// init part 1: x = x0 | 0, r = b - A x0 | b, partial ||b||^2, ||r||^2
template <int G>
__global__ void __launch_bounds__(kDotThreads)
k_pcg_init(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
           const double* __restrict__ vals, const double* __restrict__ b,
           const double* __restrict__ x0, double* __restrict__ x, double* __restrict__ r,
           double* state, double* hist, double tol, double* work) {
  double v[2] = {0.0, 0.0};
  FPB_ROW_LOOP(G, n) {
    const bool valid = row < n;
    double ri = 0.0;
    if (x0) {
      double ax = row_dot<G>(rowptr, colind, vals, x0, row, valid, sub);
      if (valid) ri = axpy1(-1.0, ax, b[row]);  // axpy(-1.0, spmv(A, x), b) (krylov.py:59)
      if (valid && sub == 0) x[row] = x0[row];
    } else {
      if (valid) ri = b[row];
      if (valid && sub == 0) x[row] = 0.0;
    }
    if (valid && sub == 0) {
      r[row] = ri;
      v[0] += b[row] * b[row];
      v[1] += ri * ri;
    }
  }
  block_sum<2>(v);
  double tot[2];
  if (grid_finish<2>(v, work, 0, tot)) {
    double bnorm = sqrt(tot[0]);
    double relres = bnorm == 0.0 ? 0.0 : sqrt(tot[1]) / bnorm;
    state[S_BNORM] = bnorm;
    state[S_TOL] = tol;
    state[S_IT] = 0.0;
    state[S_RELRES] = relres;
    state[S_PQ] = 0.0;
    state[S_STATUS] = (bnorm == 0.0 || relres <= tol) ? 1.0 : 0.0;
    hist[0] = relres;
  }
}

// init part 2: z = r / d, p = z, rz = r.z
__global__ void __launch_bounds__(kDotThreads)
k_pcg_init2(int64_t n, const double* __restrict__ r, const double* __restrict__ d,
            double* __restrict__ z, double* __restrict__ p, double* state, double* work) {
  double v[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double zi = r[i] / d[i];
    z[i] = zi;
    p[i] = zi;
    v[0] += r[i] * zi;
  }
  block_sum<1>(v);
  double tot[1];
  if (grid_finish<1>(v, work, 1, tot)) state[S_RZ] = tot[0];
}

// iteration step 1: q = A p, pq = p.q; breakdown if pq <= 0
template <int G>
__global__ void __launch_bounds__(kDotThreads)
k_pcg_spmv(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
           const double* __restrict__ vals, const double* __restrict__ p, double* __restrict__ q,
           double* state, double* work) {
  if (state[S_STATUS] != 0.0) return;
  double v[1] = {0.0};
  constexpr int R = FPB_FUSED_GROUPS;
  FPB_ROW_LOOP_R(G, R, n) {
    int64_t row[R];
    double qi[R];
    row_dot_grp<G, R>(rowptr, colind, vals, p, base_, n, sub, row, qi);
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (row[r] < n && sub == 0) {
        q[row[r]] = qi[r];
        v[0] += p[row[r]] * qi[r];
      }
  }
  block_sum<1>(v);
  double tot[1];
  if (grid_finish<1>(v, work, 2, tot)) {
    state[S_PQ] = tot[0];
    if (tot[0] <= 0.0) state[S_STATUS] = 2.0;
  }
}

// iteration step 2: x += alpha p; r -= alpha q; relres; z = r/d; rz_new = r.z
__global__ void __launch_bounds__(kDotThreads)
k_pcg_update(int64_t n, double* __restrict__ x, double* __restrict__ r,
             const double* __restrict__ p, const double* __restrict__ q,
             const double* __restrict__ d, double* __restrict__ z, double* state, double* hist,
             int64_t hist_cap, double* work) {
  if (state[S_STATUS] != 0.0) return;
  const double alpha = state[S_RZ] / state[S_PQ];
  double v[2] = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double pi = p[i];
    x[i] = axpy1(alpha, pi, x[i]);
    const double ri = axpy1(-alpha, q[i], r[i]);
    r[i] = ri;
    const double zi = ri / d[i];
    z[i] = zi;
    v[0] += ri * ri;
    v[1] += ri * zi;
  }
  block_sum<2>(v);
  double tot[2];
  if (grid_finish<2>(v, work, 3, tot)) {
    const double relres = sqrt(tot[0]) / state[S_BNORM];
    const double it = state[S_IT] + 1.0;
    state[S_IT] = it;
    state[S_RELRES] = relres;
    hist[(int64_t)it % hist_cap] = relres;
    if (relres <= state[S_TOL]) {
      state[S_STATUS] = 1.0;
    } else {
      state[S_BETA] = tot[1] / state[S_RZ];
      state[S_RZ] = tot[1];
    }
  }
}

// iteration step 3: p = beta p + z
__global__ void k_pcg_direction(int64_t n, double* __restrict__ p, const double* __restrict__ z,
                                const double* state) {
  if (state[S_STATUS] != 0.0) return;
  const double beta = state[S_BETA];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = axpy1(beta, p[i], z[i]);
}

// ---------------------------------------------------------------------------
// Device-resident Jacobi-preconditioned BiCGSTAB (config 5's solver; not in
// the reference, so it follows the published van der Vorst recurrence as
// scipy.sparse.linalg.bicgstab states it, operation for operation: rtilde =
// r0, p = r + beta (p - omega v), phat = M^-1 p, v = A phat, alpha =
// rho / (rtilde, v), s = r - alpha v, shat = M^-1 s, t = A shat,
// omega = (t, s) / (t, t), x += alpha phat; x += omega shat, r = s - omega t,
// stop when ||r|| < tol ||b||).  Five fused kernels per iteration, scalars
// and status on the device, like the PCG above.
//
// Domain decomposition (distributed.py): elementwise updates run over all n
// local entries, reductions only over the owned range [own_lo, own_hi).
// With defer = 0 the last block finishes the scalars in place (one GPU);
// with defer = 1 it leaves the partial sums in state[B_RED..] for a
// cross-rank allreduce, after which fpb_bicgstab_finish applies the same
// scalar step.
// state: see the B_* enum; status 0 running, 1 converged, 2 rho breakdown,
// 3 (rtilde, v) = 0, 4 omega breakdown, 5 converged on s (half step pending)
// ---------------------------------------------------------------------------
enum {
  B_RHO = 0, B_RHO_PREV, B_ALPHA, B_OMEGA, B_BNORM, B_ATOL, B_STATUS, B_IT, B_RELRES, B_BETA, B_RV,
  B_TS, B_TT, B_FIRST, B_RED = 16, B_NSTATE = 20  // B_RED..B_RED+2: deferred partial sums
};
enum { BSTEP_INIT = 0, BSTEP_AV, BSTEP_S, BSTEP_AT, BSTEP_UPDATE };
constexpr double kBreakTol = 4.930380657631324e-32;  // eps^2 (scipy's rhotol / omegatol)

// scalar step after reduction `step` with totals tot[] (identical on every rank)
__device__ void bicg_finish(int step, const double* tot, double* state, double* hist, int64_t hist_cap,
                            double tol) {
  switch (step) {
    case BSTEP_INIT: {
      const double bnorm = sqrt(tot[0]), rnorm = sqrt(tot[1]);
      const double atol = tol * bnorm;
      state[B_BNORM] = bnorm;
      state[B_ATOL] = atol;
      state[B_IT] = 0.0;
      state[B_RELRES] = bnorm == 0.0 ? 0.0 : rnorm / bnorm;
      state[B_RHO] = tot[1];  // (rtilde, r) with rtilde = r
      state[B_RHO_PREV] = 1.0;
      state[B_ALPHA] = 1.0;
      state[B_OMEGA] = 1.0;
      state[B_BETA] = 0.0;  // first spin: p = r
      state[B_FIRST] = 1.0;
      hist[0] = state[B_RELRES];
      double st = 0.0;
      if (bnorm == 0.0 || rnorm < atol) st = 1.0;
      else if (fabs(tot[1]) < kBreakTol) st = 2.0;
      state[B_STATUS] = st;
      break;
    }
    case BSTEP_AV:
      if (state[B_STATUS] != 0.0) break;
      state[B_RV] = tot[0];
      if (tot[0] == 0.0) state[B_STATUS] = 3.0;
      else state[B_ALPHA] = state[B_RHO] / tot[0];
      break;
    case BSTEP_S:
      if (state[B_STATUS] != 0.0) break;
      if (sqrt(tot[0]) < state[B_ATOL]) {
        state[B_STATUS] = 5.0;
        state[B_RELRES] = sqrt(tot[0]) / state[B_BNORM];
      }
      break;
    case BSTEP_AT:
      if (state[B_STATUS] != 0.0) break;
      state[B_TS] = tot[0];
      state[B_TT] = tot[1];
      state[B_OMEGA] = tot[0] / tot[1];
      break;
    case BSTEP_UPDATE: {
      const double status = state[B_STATUS];
      if (status != 0.0 && status != 5.0) break;
      const bool half = status == 5.0;
      const double alpha = state[B_ALPHA], omega = state[B_OMEGA];
      const double it = state[B_IT] + 1.0;
      const double rnorm = sqrt(tot[0]);
      state[B_IT] = it;
      state[B_RELRES] = rnorm / state[B_BNORM];
      hist[(int64_t)it % hist_cap] = state[B_RELRES];
      state[B_FIRST] = 0.0;
      if (half || rnorm < state[B_ATOL]) {
        state[B_STATUS] = 1.0;
      } else if (fabs(tot[1]) < kBreakTol) {
        state[B_STATUS] = 2.0;
      } else if (fabs(omega) < kBreakTol) {
        state[B_STATUS] = 4.0;
      } else {
        state[B_BETA] = (tot[1] / state[B_RHO]) * (alpha / omega);
        state[B_RHO_PREV] = state[B_RHO];
        state[B_RHO] = tot[1];
      }
      break;
    }
  }
}

struct BicgRed {  // where a kernel's totals go
  int64_t own_lo, own_hi;
  int defer;
  double* hist;
  int64_t hist_cap;
  double tol;
};

template <int NV>
__device__ __forceinline__ void bicg_reduce(double (&acc)[NV], int step, double* state, double* work,
                                            int slot, const BicgRed& R, int red_off = 0) {
  block_sum<NV>(acc);
  double tot[NV];
  if (grid_finish<NV>(acc, work, slot, tot)) {
    if (R.defer) {
#pragma unroll
      for (int q = 0; q < NV; ++q) state[B_RED + red_off + q] = tot[q];
    } else {
      bicg_finish(step, tot, state, R.hist, R.hist_cap, R.tol);
    }
  }
}

template <int G>
__global__ void __launch_bounds__(kDotThreads)
k_bicg_init(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
            const double* __restrict__ vals, const double* __restrict__ b, const double* __restrict__ x0,
            double* __restrict__ x, double* __restrict__ r, double* __restrict__ rt, double* __restrict__ p,
            double* __restrict__ v, double* state, double* work, BicgRed R) {
  double acc[2] = {0.0, 0.0};
  FPB_ROW_LOOP(G, n) {
    const bool valid = row < n;
    double ri = 0.0;
    if (x0) {
      const double ax = row_dot<G>(rowptr, colind, vals, x0, row, valid, sub);
      if (valid) ri = __dsub_rn(b[row], ax);  // r = b - A x0
    } else if (valid) {
      ri = b[row];
    }
    if (valid && sub == 0) {
      x[row] = x0 ? x0[row] : 0.0;
      r[row] = ri;
      rt[row] = ri;
      p[row] = 0.0;
      v[row] = 0.0;
      if (row >= R.own_lo && row < R.own_hi) {
        acc[0] += b[row] * b[row];
        acc[1] += ri * ri;
      }
    }
  }
  bicg_reduce<2>(acc, BSTEP_INIT, state, work, 0, R);
}

// K1: p = r + beta (p - omega v) (first spin: p = r); phat = p / d
__global__ void k_bicg_dir(int64_t n, const double* __restrict__ r, const double* __restrict__ v,
                           const double* __restrict__ d, double* __restrict__ p, double* __restrict__ ph,
                           const double* state) {
  if (state[B_STATUS] != 0.0) return;
  const bool first = state[B_FIRST] != 0.0;
  const double beta = state[B_BETA], omega = state[B_OMEGA];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double pi;
    if (first) {
      pi = r[i];
    } else {  // p -= omega*v; p *= beta; p += r
      pi = __dadd_rn(__dmul_rn(__dsub_rn(p[i], __dmul_rn(omega, v[i])), beta), r[i]);
    }
    p[i] = pi;
    ph[i] = d ? __ddiv_rn(pi, d[i]) : pi;
  }
}

// K2: v = A phat; rv = (rtilde, v); alpha = rho / rv
template <int G>
__global__ void __launch_bounds__(kDotThreads)
k_bicg_av(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
          const double* __restrict__ vals, const double* __restrict__ ph, const double* __restrict__ rt,
          double* __restrict__ v, double* state, double* work, BicgRed R) {
  if (state[B_STATUS] != 0.0) return;
  double acc[1] = {0.0};
  constexpr int NG = FPB_FUSED_GROUPS;
  FPB_ROW_LOOP_R(G, NG, n) {
    int64_t row[NG];
    double vi[NG];
    row_dot_grp<G, NG>(rowptr, colind, vals, ph, base_, n, sub, row, vi);
#pragma unroll
    for (int r = 0; r < NG; ++r)
      if (row[r] < n && sub == 0) {
        v[row[r]] = vi[r];
        if (row[r] >= R.own_lo && row[r] < R.own_hi) acc[0] += rt[row[r]] * vi[r];
      }
  }
  bicg_reduce<1>(acc, BSTEP_AV, state, work, 1, R);
}

// K3: s = r - alpha v; shat = s / d; ||s|| < atol -> converged on s
__global__ void __launch_bounds__(kDotThreads)
k_bicg_s(int64_t n, const double* __restrict__ r, const double* __restrict__ v, const double* __restrict__ d,
         double* __restrict__ sv, double* __restrict__ sh, double* state, double* work, BicgRed R) {
  if (state[B_STATUS] != 0.0) return;
  const double alpha = state[B_ALPHA];
  double acc[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double si = __dsub_rn(r[i], __dmul_rn(alpha, v[i]));
    sv[i] = si;
    sh[i] = d ? __ddiv_rn(si, d[i]) : si;
    if (i >= R.own_lo && i < R.own_hi) acc[0] += si * si;
  }
  // deferred: ||s||^2 goes to state[B_RED + 2] and rides on the allreduce
  // after K4 (three reductions per iteration cross ranks, not four)
  bicg_reduce<1>(acc, BSTEP_S, state, work, 2, R, 2);
}

// K4: t = A shat; (t, s), (t, t); omega = ts / tt
template <int G>
__global__ void __launch_bounds__(kDotThreads)
k_bicg_at(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
          const double* __restrict__ vals, const double* __restrict__ sh, const double* __restrict__ sv,
          double* __restrict__ t, double* state, double* work, BicgRed R) {
  if (state[B_STATUS] != 0.0) return;
  double acc[2] = {0.0, 0.0};
  constexpr int NG = FPB_FUSED_GROUPS;
  FPB_ROW_LOOP_R(G, NG, n) {
    int64_t row[NG];
    double ti[NG];
    row_dot_grp<G, NG>(rowptr, colind, vals, sh, base_, n, sub, row, ti);
#pragma unroll
    for (int r = 0; r < NG; ++r)
      if (row[r] < n && sub == 0) {
        t[row[r]] = ti[r];
        if (row[r] >= R.own_lo && row[r] < R.own_hi) {
          acc[0] += ti[r] * sv[row[r]];
          acc[1] += ti[r] * ti[r];
        }
      }
  }
  bicg_reduce<2>(acc, BSTEP_AT, state, work, 3, R);
}

// K5: x += alpha phat; x += omega shat; r = s - omega t; ||r||, rho_new =
// (rtilde, r); stopping and breakdown tests, beta for the next spin.  With
// status 5 (converged on s) only x += alpha phat and r = s are applied.
__global__ void __launch_bounds__(kDotThreads)
k_bicg_update(int64_t n, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ ph,
              const double* __restrict__ sh, const double* __restrict__ sv, const double* __restrict__ t,
              const double* __restrict__ rt, double* state, double* work, BicgRed R) {
  const double status = state[B_STATUS];
  if (status != 0.0 && status != 5.0) return;
  const bool half = status == 5.0;
  const double alpha = state[B_ALPHA], omega = state[B_OMEGA];
  double acc[2] = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double xi = axpy1(alpha, ph[i], x[i]);
    double ri = sv[i];
    if (!half) {
      xi = axpy1(omega, sh[i], xi);
      ri = __dsub_rn(ri, __dmul_rn(omega, t[i]));
    }
    x[i] = xi;
    r[i] = ri;
    if (i >= R.own_lo && i < R.own_hi) {
      acc[0] += ri * ri;
      acc[1] += rt[i] * ri;
    }
  }
  bicg_reduce<2>(acc, BSTEP_UPDATE, state, work, 0, R);
}

__global__ void k_bicg_finish(int step, double* state, double* hist, int64_t hist_cap, double tol) {
  double tot[2] = {state[B_RED], state[B_RED + 1]};
  if (step == BSTEP_S) tot[0] = state[B_RED + 2];
  bicg_finish(step, tot, state, hist, hist_cap, tol);
}

// ---- SELL-32 twins of the fused solver kernels (sparse.SellCopy) -----------
// Same epilogues as the CSR kernels above; the matrix rows come from
// sell_row_dot (one thread per row, the reference's per-row order).  Rows
// are walked grid-stride in whole slices (n32 = n rounded up to 32).
#define FPB_SELL_LOOP(n)                                                          \
  const int64_t n32_ = ((int64_t)(n) + 31) & ~31LL;                              \
  const int64_t stride_ = (int64_t)gridDim.x * blockDim.x;                       \
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < n32_; row += stride_)

struct SellMat {
  const int64_t* ptr;
  const void* col;  // int32 columns or int16 offsets (idx16)
  const double* val;
  int idx16;
};
template <typename IDX>
__device__ __forceinline__ const IDX* sell_cols(const SellMat& A) { return static_cast<const IDX*>(A.col); }

template <int B, typename IDX>
__global__ void __launch_bounds__(kDotThreads)
k_pcg_init_sell(int32_t n, SellMat A, const double* __restrict__ b, const double* __restrict__ x0,
                double* __restrict__ x, double* __restrict__ r, double* state, double* hist, double tol,
                double* work) {
  double v[2] = {0.0, 0.0};
  FPB_SELL_LOOP(n) {
    const double ax = x0 ? sell_row_dot<B, IDX>(A.ptr, sell_cols<IDX>(A), A.val, x0, row) : 0.0;
    if (row < n) {
      const double ri = x0 ? axpy1(-1.0, ax, b[row]) : b[row];  // krylov.py:59
      x[row] = x0 ? x0[row] : 0.0;
      r[row] = ri;
      v[0] += b[row] * b[row];
      v[1] += ri * ri;
    }
  }
  block_sum<2>(v);
  double tot[2];
  if (grid_finish<2>(v, work, 0, tot)) {
    double bnorm = sqrt(tot[0]);
    double relres = bnorm == 0.0 ? 0.0 : sqrt(tot[1]) / bnorm;
    state[S_BNORM] = bnorm;
    state[S_TOL] = tol;
    state[S_IT] = 0.0;
    state[S_RELRES] = relres;
    state[S_PQ] = 0.0;
    state[S_STATUS] = (bnorm == 0.0 || relres <= tol) ? 1.0 : 0.0;
    hist[0] = relres;
  }
}

template <int B, typename IDX>
__global__ void __launch_bounds__(kDotThreads)
k_pcg_spmv_sell(int32_t n, SellMat A, const double* __restrict__ p, double* __restrict__ q, double* state,
                double* work) {
  if (state[S_STATUS] != 0.0) return;
  double v[1] = {0.0};
  FPB_SELL_LOOP(n) {
    const double qi = sell_row_dot<B, IDX>(A.ptr, sell_cols<IDX>(A), A.val, p, row);
    if (row < n) {
      q[row] = qi;
      v[0] += p[row] * qi;
    }
  }
  block_sum<1>(v);
  double tot[1];
  if (grid_finish<1>(v, work, 2, tot)) {
    state[S_PQ] = tot[0];
    if (tot[0] <= 0.0) state[S_STATUS] = 2.0;
  }
}

template <int B, typename IDX>
__global__ void __launch_bounds__(kDotThreads)
k_bicg_init_sell(int32_t n, SellMat A, const double* __restrict__ b, const double* __restrict__ x0,
                 double* __restrict__ x, double* __restrict__ r, double* __restrict__ rt, double* __restrict__ p,
                 double* __restrict__ v, double* state, double* work, BicgRed R) {
  double acc[2] = {0.0, 0.0};
  FPB_SELL_LOOP(n) {
    const double ax = x0 ? sell_row_dot<B, IDX>(A.ptr, sell_cols<IDX>(A), A.val, x0, row) : 0.0;
    if (row < n) {
      const double ri = x0 ? __dsub_rn(b[row], ax) : b[row];  // r = b - A x0
      x[row] = x0 ? x0[row] : 0.0;
      r[row] = ri;
      rt[row] = ri;
      p[row] = 0.0;
      v[row] = 0.0;
      if (row >= R.own_lo && row < R.own_hi) {
        acc[0] += b[row] * b[row];
        acc[1] += ri * ri;
      }
    }
  }
  bicg_reduce<2>(acc, BSTEP_INIT, state, work, 0, R);
}

template <int B, typename IDX>
__global__ void __launch_bounds__(kDotThreads)
k_bicg_av_sell(int32_t n, SellMat A, const double* __restrict__ ph, const double* __restrict__ rt,
               double* __restrict__ v, double* state, double* work, BicgRed R) {
  if (state[B_STATUS] != 0.0) return;
  double acc[1] = {0.0};
  FPB_SELL_LOOP(n) {
    const double vi = sell_row_dot<B, IDX>(A.ptr, sell_cols<IDX>(A), A.val, ph, row);
    if (row < n) {
      v[row] = vi;
      if (row >= R.own_lo && row < R.own_hi) acc[0] += rt[row] * vi;
    }
  }
  bicg_reduce<1>(acc, BSTEP_AV, state, work, 1, R);
}

template <int B, typename IDX>
__global__ void __launch_bounds__(kDotThreads)
k_bicg_at_sell(int32_t n, SellMat A, const double* __restrict__ sh, const double* __restrict__ sv,
               double* __restrict__ t, double* state, double* work, BicgRed R) {
  if (state[B_STATUS] != 0.0) return;
  double acc[2] = {0.0, 0.0};
  FPB_SELL_LOOP(n) {
    const double ti = sell_row_dot<B, IDX>(A.ptr, sell_cols<IDX>(A), A.val, sh, row);
    if (row < n) {
      t[row] = ti;
      if (row >= R.own_lo && row < R.own_hi) {
        acc[0] += ti * sv[row];
        acc[1] += ti * ti;
      }
    }
  }
  bicg_reduce<2>(acc, BSTEP_AT, state, work, 3, R);
}

// launch a SELL kernel for the matrix's column storage
#define FPB_SELL_LAUNCH(KER, GRID, BLOCK, N, A, ...)                                \
  do {                                                                              \
    if ((A).idx16) KER<kSellBatch, int16_t><<<GRID, BLOCK, 0, s>>>(N, A, __VA_ARGS__); \
    else KER<kSellBatch, int32_t><<<GRID, BLOCK, 0, s>>>(N, A, __VA_ARGS__);           \
  } while (0)

inline int lanes_per_row(int32_t n, int64_t nnz) {
  const double mean = n > 0 ? (double)nnz / n : 0.0;
  return mean <= 6.0 ? 4 : (mean <= 20.0 ? 8 : 16);
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_spmv(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
             const double* vals, const double* x, double* y, void* stream) {
  if (n <= 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  // lanes per row from the mean row length (tet ~15 -> 8, hex ~27 -> 16)
  const double mean = (double)nnz / n;
#ifdef FPB_SPMV_G
  const int G = FPB_SPMV_G;
#else
  const int G = mean <= 6.0 ? 4 : (mean <= 20.0 ? 8 : 16);
#endif
  constexpr int R = FPB_SPMV_GROUPS;
  int grid = grid_for(((int64_t)n * G + R - 1) / R, 256, 16);
  if (G == 4) k_spmv_r<4, R><<<grid, 256, 0, s>>>(n, rowptr, colind, vals, x, y);
  else if (G == 8) k_spmv_r<8, R><<<grid, 256, 0, s>>>(n, rowptr, colind, vals, x, y);
  else k_spmv_r<16, R><<<grid, 256, 0, s>>>(n, rowptr, colind, vals, x, y);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_sell_build(int32_t n, const int32_t* rowptr, const int32_t* colind, const double* vals, int64_t* sell_ptr,
                   void* scol, int idx16, double* sval, int64_t* total_h, int32_t* maxoff_h, void* stream) {
  FPB_REQUIRE(n >= 0 && rowptr && sell_ptr, "bad SELL arguments");
  cudaStream_t s = as_stream(stream);
  const int64_t nsl = ((int64_t)n + 31) / 32;
  if (!scol && !sval) {  // widths and slice offsets (+ the largest |col - row|)
    FPB_CUDA(cudaMemsetAsync(sell_ptr, 0, sizeof(int64_t), s));
    int* dmax = nullptr;
    if (maxoff_h) {
      FPB_REQUIRE(colind, "the offset range needs colind");
      FPB_CUDA(cudaMallocAsync(&dmax, sizeof(int), s));
      FPB_CUDA(cudaMemsetAsync(dmax, 0, sizeof(int), s));
      if (n > 0) k_max_offset<<<grid_for(n, 256), 256, 0, s>>>(n, rowptr, colind, dmax);
    }
    if (nsl > 0) {
      k_sell_width<<<(unsigned)((nsl * 32 + 255) / 256), 256, 0, s>>>(n, rowptr, sell_ptr + 1);
      FPB_LAUNCH_CHECK();
      size_t tmp_bytes = 0;
      void* tmp = nullptr;
      cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, sell_ptr + 1, sell_ptr + 1, nsl, s);
      FPB_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
      FPB_CUDA(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, sell_ptr + 1, sell_ptr + 1, nsl, s));
      FPB_CUDA(cudaFreeAsync(tmp, s));
    }
    FPB_CUDA(cudaMemcpyAsync(total_h, sell_ptr + nsl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (dmax) {
      FPB_CUDA(cudaMemcpyAsync(maxoff_h, dmax, sizeof(int), cudaMemcpyDeviceToHost, s));
      FPB_CUDA(cudaFreeAsync(dmax, s));
    }
    FPB_CUDA(cudaStreamSynchronize(s));
    return FPB_OK;
  }
  if (n > 0) {
    int* bad = nullptr;
    if (scol && idx16) {
      FPB_CUDA(cudaMallocAsync(&bad, sizeof(int), s));
      FPB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    }
    k_sell_fill<<<(unsigned)((nsl * 32 + 255) / 256), 256, 0, s>>>(n, rowptr, colind, vals, sell_ptr, scol, idx16,
                                                                  sval, bad);
    FPB_LAUNCH_CHECK();
    if (bad) {
      int h = 0;
      FPB_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
      FPB_CUDA(cudaFreeAsync(bad, s));
      FPB_CUDA(cudaStreamSynchronize(s));
      FPB_REQUIRE(!h, "column offsets do not fit 16 bits (check maxoff first)");
    }
  }
  return FPB_OK;
}

int fpb_spmv_sell(int32_t n, const int64_t* sell_ptr, const void* scol, int idx16, const double* sval,
                  const double* x, double* y, void* stream) {
  if (n <= 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  const unsigned grid = (unsigned)(((int64_t)n + 255) / 256);
  if (idx16)
    k_spmv_sell<kSellBatch, int16_t><<<grid, 256, 0, s>>>(n, sell_ptr, static_cast<const int16_t*>(scol), sval, x, y);
  else
    k_spmv_sell<kSellBatch, int32_t><<<grid, 256, 0, s>>>(n, sell_ptr, static_cast<const int32_t*>(scol), sval, x, y);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_axpy(int64_t n, double alpha, const double* x, const double* y, double* out, void* stream) {
  if (n <= 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  bool aligned = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) && ((uintptr_t)out % 16 == 0);
  if (aligned && n % 2 == 0) {
    k_axpy2<<<grid_for(n / 2, 256, 8), 256, 0, s>>>(n / 2, alpha, (const double2*)x, (const double2*)y,
                                                    (double2*)out);
  } else {
    k_axpy<<<grid_for(n, 256, 8), 256, 0, s>>>(n, alpha, x, y, out);
  }
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int64_t fpb_dot_work_size(void) { return kWorkDoubles; }

int fpb_dot(int64_t n, const double* x, const double* y, double* result, double* work, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_dot<<<kDotBlocks, kDotThreads, 0, s>>>(n, x, y, result, work);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_diagonal(int32_t n, const int32_t* rowptr, const int32_t* colind, const double* vals,
                 double* d, void* stream) {
  if (n <= 0) return FPB_OK;
  k_diagonal<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, rowptr, colind, vals, d);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_row_sums(int32_t n, const int32_t* rowptr, const double* vals, double* out, void* stream) {
  if (n <= 0) return FPB_OK;
  k_row_sums<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, rowptr, vals, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_pcg_init(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind, const double* vals,
                 const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16, const double* b, const double* x0, double* x, double* r, double* p, double* z,
                 const double* d, double* state, double* hist, double tol, double* work,
                 void* stream) {
  cudaStream_t s = as_stream(stream);
  const SellMat A{sell_ptr, scol, sval, sell_idx16};
  if (sell_ptr)
    FPB_SELL_LAUNCH(k_pcg_init_sell, kDotBlocks, kDotThreads, n, A, b, x0, x, r, state, hist, tol, work);
  else switch (lanes_per_row(n, nnz)) {
    case 4: k_pcg_init<4><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, b, x0, x, r, state, hist, tol, work); break;
    case 8: k_pcg_init<8><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, b, x0, x, r, state, hist, tol, work); break;
    default: k_pcg_init<16><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, b, x0, x, r, state, hist, tol, work); break;
  }
  FPB_LAUNCH_CHECK();
  k_pcg_init2<<<kDotBlocks, kDotThreads, 0, s>>>(n, r, d, z, p, state, work);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_pcg_iterate(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind, const double* vals,
                    const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16, double* x, double* r, double* p, double* q, double* z, const double* d,
                    double* state, double* hist, int64_t hist_cap, int iters, double* work,
                    void* stream) {
  cudaStream_t s = as_stream(stream);
  const int G = lanes_per_row(n, nnz);
  const SellMat A{sell_ptr, scol, sval, sell_idx16};
  const bool SB = sell_ptr != nullptr;
  for (int it = 0; it < iters; ++it) {
    if (SB) FPB_SELL_LAUNCH(k_pcg_spmv_sell, kDotBlocks, kDotThreads, n, A, p, q, state, work);
    else if (G == 4) k_pcg_spmv<4><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, p, q, state, work);
    else if (G == 8) k_pcg_spmv<8><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, p, q, state, work);
    else k_pcg_spmv<16><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, p, q, state, work);
    k_pcg_update<<<kDotBlocks, kDotThreads, 0, s>>>(n, x, r, p, q, d, z, state, hist, hist_cap, work);
    k_pcg_direction<<<grid_for(n, 256, 8), 256, 0, s>>>(n, p, z, state);
  }
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}


int fpb_bicgstab_state_size(void) { return B_NSTATE; }

int fpb_bicgstab_init(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind, const double* vals,
                      const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16, const double* b, const double* x0, double* x, double* r, double* rt, double* p, double* v,
                      double* state, double* hist, double tol, int64_t own_lo, int64_t own_hi, int defer,
                      double* work, void* stream) {
  cudaStream_t s = as_stream(stream);
  const BicgRed R{own_lo, own_hi, defer, hist, 1, tol};
  const SellMat A{sell_ptr, scol, sval, sell_idx16};
  if (sell_ptr)
    FPB_SELL_LAUNCH(k_bicg_init_sell, kDotBlocks, kDotThreads, n, A, b, x0, x, r, rt, p, v, state, work, R);
  else switch (lanes_per_row(n, nnz)) {
    case 4: k_bicg_init<4><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, b, x0, x, r, rt, p, v, state, work, R); break;
    case 8: k_bicg_init<8><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, b, x0, x, r, rt, p, v, state, work, R); break;
    default: k_bicg_init<16><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, b, x0, x, r, rt, p, v, state, work, R); break;
  }
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_bicgstab_iterate(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
                         const double* vals, const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16,
                         const double* d, double* x, double* r, const double* rt, double* p,
                         double* ph, double* v, double* sv, double* sh, double* t, double* state, double* hist,
                         int64_t hist_cap, int iters, double* work, void* stream) {
  cudaStream_t s = as_stream(stream);
  for (int it = 0; it < iters; ++it)
    for (int step = BSTEP_AV; step <= BSTEP_UPDATE; ++step) {
      int rc = fpb_bicgstab_step(step, n, nnz, rowptr, colind, vals, sell_ptr, scol, sval, sell_idx16, d, x, r, rt, p, ph, v, sv, sh, t, state,
                                 hist, hist_cap, 0, n, 0, work, stream);
      if (rc) return rc;
    }
  (void)s;
  return FPB_OK;
}

int fpb_bicgstab_step(int step, int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
                      const double* vals, const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16,
                      const double* d, double* x, double* r, const double* rt, double* p,
                      double* ph, double* v, double* sv, double* sh, double* t, double* state, double* hist,
                      int64_t hist_cap, int64_t own_lo, int64_t own_hi, int defer, double* work, void* stream) {
  cudaStream_t s = as_stream(stream);
  const int G = lanes_per_row(n, nnz);
  const BicgRed R{own_lo, own_hi, defer, hist, hist_cap, 0.0};
  const SellMat A{sell_ptr, scol, sval, sell_idx16};
  const bool SB = sell_ptr != nullptr;
  switch (step) {
    case BSTEP_AV:  // K1 + K2
      k_bicg_dir<<<grid_for(n, 256, 8), 256, 0, s>>>(n, r, v, d, p, ph, state);
      if (SB) FPB_SELL_LAUNCH(k_bicg_av_sell, kDotBlocks, kDotThreads, n, A, ph, rt, v, state, work, R);
      else if (G == 4) k_bicg_av<4><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, ph, rt, v, state, work, R);
      else if (G == 8) k_bicg_av<8><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, ph, rt, v, state, work, R);
      else k_bicg_av<16><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, ph, rt, v, state, work, R);
      break;
    case BSTEP_S:
      k_bicg_s<<<kDotBlocks, kDotThreads, 0, s>>>(n, r, v, d, sv, sh, state, work, R);
      break;
    case BSTEP_AT:
      if (SB) FPB_SELL_LAUNCH(k_bicg_at_sell, kDotBlocks, kDotThreads, n, A, sh, sv, t, state, work, R);
      else if (G == 4) k_bicg_at<4><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, sh, sv, t, state, work, R);
      else if (G == 8) k_bicg_at<8><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, sh, sv, t, state, work, R);
      else k_bicg_at<16><<<kDotBlocks, kDotThreads, 0, s>>>(n, rowptr, colind, vals, sh, sv, t, state, work, R);
      break;
    case BSTEP_UPDATE:
      k_bicg_update<<<kDotBlocks, kDotThreads, 0, s>>>(n, x, r, ph, sh, sv, t, rt, state, work, R);
      break;
    default:
      set_error("bad BiCGSTAB step %d", step);
      return FPB_ECONFIG;
  }
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_bicgstab_finish(int step, double* state, double* hist, int64_t hist_cap, double tol, void* stream) {
  FPB_REQUIRE(step >= BSTEP_INIT && step <= BSTEP_UPDATE, "bad BiCGSTAB step %d", step);
  k_bicg_finish<<<1, 1, 0, as_stream(stream)>>>(step, state, hist, hist_cap, tol);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

}  // extern "C"
