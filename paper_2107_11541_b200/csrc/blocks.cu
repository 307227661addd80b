// Element-block RHS assembly: element-centric integration with a
// deterministic, atomic-free two-level reduction.
//
// Elements are cut into blocks of kBlockElems consecutive elements (4 packs
// of 32 lanes — consecutive elements of the reference's k-major cell order
// share nodes heavily: ~0.72 distinct nodes per element inside a 128-element
// block versus 4 node references per element).  128-element blocks with
// 6 CTAs/SM measured fastest on B200 (profiles/r01_blocks_variants.txt).  One CTA per block:
//   phase 1 (k_blk_rhs): every thread integrates one element in registers
//     (closed form for affine simplices, the reference Gauss loop otherwise),
//     parks its NN x NV contributions in shared memory, and after one barrier
//     each distinct node of the block sums its contributions in ascending
//     element order (pre-sorted gather list) into a per-(block, node) partial;
//   phase 2 (k_blk_gather): one thread per mesh node sums its partials in
//     ascending block order and writes the RHS entry once.
// Each element is integrated exactly once, nothing is zero-filled, and the
// summation order is fixed — the output is bitwise reproducible.
//
// Setup (k_blk_setup): a CTA radix-sorts its block's (node, slot) pairs with
// CUB's BlockRadixSort (stable, so equal nodes keep ascending slot order),
// giving the distinct node list, the per-node gather ranges and the gather
// slots in one pass; the node -> partial lists for phase 2 are a counting
// sort plus a per-node insertion sort.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <climits>

#include "simplex.cuh"

namespace fpb {

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }


#ifndef FPB_BLK_ELEMS
#define FPB_BLK_ELEMS 256  // affine simplices: 2 elements per thread
#endif
#ifndef FPB_BLK_ELEMS_GAUSS
#define FPB_BLK_ELEMS_GAUSS 128  // Gauss-loop types: 1 element per thread
#endif
#ifndef FPB_BLK_THREADS
#define FPB_BLK_THREADS 128
#endif
#ifndef FPB_BLK_MINB
#define FPB_BLK_MINB 4  // affine, other kinds
#endif
// affine momentum / scalar RHS: CTAs per SM measured on config 2
// (profiles/r01n_blk: momentum 0.222 -> 0.208 ms at 5, scalar 0.155 -> 0.151 at 6)
#ifndef FPB_BLK_MINB_MOMENTUM
#define FPB_BLK_MINB_MOMENTUM 5
#endif
#ifndef FPB_BLK_MINB_SCALAR
#define FPB_BLK_MINB_SCALAR 6
#endif
#ifndef FPB_BLK_MINB_SCALAR3
#define FPB_BLK_MINB_SCALAR3 5
#endif
#ifndef FPB_BLK_TET_ADJ
#define FPB_BLK_TET_ADJ 1  // TET04 momentum in the adjugate closed form (fewer FP64 operations)
#endif
#ifndef FPB_BLK_INTERLEAVE
#define FPB_BLK_INTERLEAVE 1  // the compiler interleaves a thread's two elements (ILP)
#endif
#ifndef FPB_BLK_MINB_NONAFFINE
#define FPB_BLK_MINB_NONAFFINE 2  // Gauss-loop elements (QUAD04, PYR05, HEX08): registers, not spills
#endif
constexpr int kBlockThreads = FPB_BLK_THREADS;  // threads of the RHS kernel
int g_tuning_blk_pipe = 0;  // fpb_set_tuning("blk_pipe", 0|1): pipelined persistent block kernel (A/B: slower, profiles/r02e_mom)
// elements per block (= setup threads): the affine kernels integrate EPT = 2
// elements per thread so the CTA's fixed latencies (node-id and record
// gathers, two barriers) are paid once per 256 elements; the Gauss-loop
// kernels (~230 registers, two CTAs per SM) keep one element per thread
template <int ET> constexpr int blk_elems() { return Elem<ET>::AFFINE ? FPB_BLK_ELEMS : FPB_BLK_ELEMS_GAUSS; }
inline int blk_elems_rt(int et) { return (et == FPB_TRI03 || et == FPB_TET04) ? FPB_BLK_ELEMS : FPB_BLK_ELEMS_GAUSS; }
static_assert(FPB_BLK_ELEMS % FPB_BLK_THREADS == 0 && FPB_BLK_ELEMS / FPB_BLK_THREADS <= 2, "EPT must be 1 or 2");
static_assert(FPB_BLK_ELEMS_GAUSS % FPB_BLK_THREADS == 0 && FPB_BLK_ELEMS_GAUSS / FPB_BLK_THREADS <= 2, "EPT");

// ---- setup -------------------------------------------------------------------
template <int NN, int kBlockElems>
__global__ void __launch_bounds__(kBlockElems)
k_blk_setup(int64_t nelem, const int32_t* __restrict__ conn, int pass, int32_t* __restrict__ blk_count,
            const int32_t* __restrict__ blk_ptr, int32_t* __restrict__ blk_nodes,
            uint16_t* __restrict__ blk_gptr, uint16_t* __restrict__ blk_gslot,
            uint16_t* __restrict__ blk_lidx) {
  using Sort = cub::BlockRadixSort<int, kBlockElems, NN, unsigned short>;
  using Scan = cub::BlockScan<int, kBlockElems>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ int sorted[kBlockElems * NN + 1];
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.x;
  const int64_t e = b * kBlockElems + tid;
  int keys[NN];
  unsigned short vals[NN];
#pragma unroll
  for (int q = 0; q < NN; ++q) {
    keys[q] = e < nelem ? conn[e * NN + q] : INT_MAX;
    vals[q] = (unsigned short)(tid * NN + q);  // slot = local element * NN + local node
  }
  Sort(tmp.sort).Sort(keys, vals);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NN; ++q) sorted[tid * NN + q] = keys[q];
  __syncthreads();
  int head[NN], nhead = 0;
#pragma unroll
  for (int q = 0; q < NN; ++q) {
    const int pos = tid * NN + q;
    head[q] = keys[q] != INT_MAX && (pos == 0 || sorted[pos - 1] != keys[q]);
    nhead += head[q];
  }
  int first, total;
  Scan(tmp.scan).ExclusiveSum(nhead, first, total);
  if (pass == 0) {
    if (tid == 0) blk_count[b] = total;
    return;
  }
  const int64_t base = blk_ptr[b];
  uint16_t* gptr = blk_gptr + base + b;  // total + 1 entries
  int u = first;
#pragma unroll
  for (int q = 0; q < NN; ++q) {
    const int pos = tid * NN + q;
    if (head[q]) {
      blk_nodes[base + u] = keys[q];
      gptr[u] = (uint16_t)pos;
      ++u;
    }
    blk_gslot[b * kBlockElems * NN + pos] = vals[q];
    // slot -> local node (u - 1 is the run this sorted item belongs to)
    if (keys[q] != INT_MAX) blk_lidx[b * kBlockElems * NN + vals[q]] = (uint16_t)(u - 1);
  }
  // end of the last gather range = number of valid (node, slot) pairs
  int64_t nvalid = nelem - b * kBlockElems;
  if (nvalid > kBlockElems) nvalid = kBlockElems;
  if (tid == 0) gptr[total] = (uint16_t)(nvalid * NN);
}

__global__ void k_max_count(int64_t m, const int32_t* cnt, int32_t* out) {
  int best = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    best = max(best, cnt[i]);
  best = __reduce_max_sync(0xffffffffu, best);
  if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

__global__ void k_p2_count(int64_t P, const int32_t* blk_nodes, int32_t* cnt) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[blk_nodes[p]], 1);
}

__global__ void k_p2_fill(int64_t P, const int32_t* blk_nodes, const int32_t* ptr, int32_t* cursor,
                          int32_t* list) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const int node = blk_nodes[p];
    list[ptr[node] + atomicAdd(&cursor[node], 1)] = (int32_t)p;
  }
}

__global__ void k_p2_sort(int32_t n, const int32_t* ptr, int32_t* list) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t* l = list + ptr[i];
    const int len = ptr[i + 1] - ptr[i];
    for (int x = 1; x < len; ++x) {
      const int v = l[x];
      int y = x - 1;
      while (y >= 0 && l[y] > v) {
        l[y + 1] = l[y];
        --y;
      }
      l[y + 1] = v;
    }
  }
}

// ---- phase 1: stage nodes, integrate, in-block gather ---------------------------
// kBlockThreads threads per CTA integrate kBlockElems = EPT x kBlockThreads
// elements (EPT per thread, one after the other): the CTA's fixed
// latencies — node-id and node-record gathers, two barriers — are paid once
// per EPT elements of compute.
// Shared memory: [contributions: NN * NV x kBlockElems], [gather slots:
// NN x kBlockElems uint16], [node data of the block's distinct nodes:
// maxnu x NDAT].
template <int ET, int KIND>
__global__ void __launch_bounds__(kBlockThreads,
                                  !Elem<ET>::AFFINE              ? FPB_BLK_MINB_NONAFFINE
                                  : KIND == FPB_MOMENTUM_RHS     ? FPB_BLK_MINB_MOMENTUM
                                  : KIND == FPB_SCALAR_RHS       ? FPB_BLK_MINB_SCALAR
                                  : KIND == KIND_SCALAR3         ? FPB_BLK_MINB_SCALAR3
                                                                 : FPB_BLK_MINB)
k_blk_rhs(int64_t nelem, int64_t blk0, const uint16_t* __restrict__ blk_lidx, const double* __restrict__ xyz4,
          const double* __restrict__ uvw4, const double* __restrict__ vel, const double* __restrict__ phi,
          int64_t fstride, double rho, double mu, double kappa, const int32_t* __restrict__ blk_ptr, const int32_t* __restrict__ blk_nodes,
          const uint16_t* __restrict__ blk_gptr, const uint16_t* __restrict__ blk_gslot, int maxnu,
          double* __restrict__ partial) {
  constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM;
  constexpr int NV = Out<ET, KIND>::NV;
  constexpr int NF = KIND == FPB_SCALAR_RHS ? 1 : KIND == KIND_SCALAR3 ? 3 : 0;  // scalar fields
  constexpr int NDAT = 2 * DIM + NF;  // x, u (, phi...)
  constexpr int TPB = kBlockThreads;
  constexpr int kBlockElems = blk_elems<ET>();
  constexpr int EPT = kBlockElems / TPB;
  constexpr int NGR = EPT == 2 ? 3 : 2;  // gather ranges prefetched per thread (nu <= NGR * TPB)
  extern __shared__ __align__(16) double smem[];
  double* sm = smem;                                                    // [NN * NV][kBlockElems]
  uint16_t* sgslot = reinterpret_cast<uint16_t*>(sm + NN * NV * kBlockElems);  // [NN * kBlockElems]
  double* snode = sm + NN * NV * kBlockElems + NN * kBlockElems / 4;  // [maxnu][NDAT]
  const int tid = threadIdx.x;
  const int64_t b = blk0 + blockIdx.x;  // blocks [blk0, blk0 + gridDim.x)
  // gather metadata of phase 3 is fetched now so its latency hides behind
  // staging and integration: slots via cp.async, range bounds in registers
  {
    const uint16_t* g = blk_gslot + b * kBlockElems * NN;
    for (int c = tid; c < NN * kBlockElems / 8; c += TPB) cp_async16(sgslot + 8 * c, g + 8 * c);
    cp_async_commit();
  }
  const int64_t base = blk_ptr[b];
  const int nu = blk_ptr[b + 1] - (int)base;
  const uint16_t* gptr = blk_gptr + base + b;
  int glo[NGR], ghi[NGR];
#pragma unroll
  for (int j = 0; j < NGR; ++j) {
    const int u = tid + j * TPB;
    glo[j] = u < nu ? __ldg(gptr + u) : 0;
    ghi[j] = u < nu ? __ldg(gptr + u + 1) : 0;
  }
  int li[EPT][NN];
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const int64_t e = b * kBlockElems + tid + j * TPB;
    if (e < nelem) {
      const uint16_t* lp = blk_lidx + e * NN;
      if constexpr (NN == 4) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(lp));
        li[j][0] = v.x & 0xffff; li[j][1] = v.x >> 16; li[j][2] = v.y & 0xffff; li[j][3] = v.y >> 16;
      } else {
#pragma unroll
        for (int a = 0; a < NN; ++a) li[j][a] = __ldg(lp + a);
      }
    }
  }
  // stage the block's distinct nodes: two 256-bit loads per node record
  for (int u = tid; u < nu; u += TPB) {
    const int64_t node = __ldg(blk_nodes + base + u);
    double rx[4], ru[4] = {0.0, 0.0, 0.0, 0.0};
    ld256(xyz4 + 4 * node, rx);
    if (uvw4) {
      ld256(uvw4 + 4 * node, ru);
    } else {  // the caller's velocity rows [n][dim] (+ scalar) directly: no packing pass
#pragma unroll
      for (int d = 0; d < DIM; ++d) ru[d] = __ldg(vel + node * DIM + d);
      if constexpr (KIND == FPB_SCALAR_RHS) ru[3] = __ldg(phi + node);
    }
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      snode[u * NDAT + d] = rx[d];
      snode[u * NDAT + DIM + d] = ru[d];
    }
    if constexpr (KIND == FPB_SCALAR_RHS) snode[u * NDAT + 2 * DIM] = ru[3];
    if constexpr (KIND == KIND_SCALAR3) {  // fields [3][fstride], read in place
#pragma unroll
      for (int f = 0; f < 3; ++f) snode[u * NDAT + 2 * DIM + f] = __ldg(phi + f * fstride + node);
    }
  }
  __syncthreads();
#if FPB_BLK_INTERLEAVE
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int j = 0; j < EPT; ++j) {
    const int el = tid + j * TPB;
    if (b * kBlockElems + el >= nelem) break;
    double xe[NN][DIM], ue[Out<ET, KIND>::NU][DIM], fe[Out<ET, KIND>::NF];
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      const int l = j == 0 ? li[0][a] : li[EPT - 1][a];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        xe[a][d] = snode[l * NDAT + d];
        ue[a][d] = snode[l * NDAT + DIM + d];
      }
      if constexpr (KIND == FPB_SCALAR_RHS) fe[a] = snode[l * NDAT + 2 * DIM];
      if constexpr (KIND == KIND_SCALAR3) {
#pragma unroll
        for (int f = 0; f < 3; ++f) fe[f * NN + a] = snode[l * NDAT + 2 * DIM + f];
      }
    }
    double acc[Out<ET, KIND>::NOUT];
    if constexpr (ET == FPB_TET04 && KIND == FPB_MOMENTUM_RHS && FPB_BLK_TET_ADJ) {
      // adjugate closed form (simplex.cuh tet_mom_adj, the Kuhn kernels' residual)
      double res[4][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
      tet_mom_adj(xe, ue, rho * refM<ET>(0, 1), mu * refWsum<ET>(), res);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[a * 3 + k] = res[a][k];
    } else if constexpr (Elem<ET>::AFFINE) {
      simplex_rhs_all<ET, KIND>(xe, ue, fe, rho, mu, kappa, acc);
    } else if constexpr (KIND == KIND_SCALAR3 && ET == FPB_HEX08) {  // one geometry, three fields (Walsh forms)
      hex_rhs_integrate<KIND_SCALAR3>(xe, ue, fe, rho, mu, kappa, acc);
    } else if constexpr (KIND == KIND_SCALAR3) {  // Gauss loop per field (staging shared)
      const double kap[3] = {rho, mu, kappa};
#pragma unroll 1
      for (int f = 0; f < 3; ++f) {
        double ff[NN], af[NN];
#pragma unroll
        for (int a = 0; a < NN; ++a) ff[a] = fe[f * NN + a];
        element_integrate<ET, FPB_SCALAR_RHS>(xe, ue, ff, 0.0, 0.0, kap[f], 0, af);
#pragma unroll
        for (int a = 0; a < NN; ++a) acc[a * 3 + f] = af[a];
      }
    } else {
      element_integrate<ET, KIND>(xe, ue, fe, rho, mu, kappa, 0, acc);
    }
#pragma unroll
    for (int a = 0; a < NN; ++a)
#pragma unroll
      for (int k = 0; k < NV; ++k) sm[(a * NV + k) * kBlockElems + el] = acc[a * NV + k];
  }
  cp_async_wait_all();
  __syncthreads();
  for (int u = tid, j = 0; u < nu; u += TPB, ++j) {
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = 0.0;
    int lo, hi;
    if (j < NGR) {
      lo = glo[0];
      hi = ghi[0];
#pragma unroll
      for (int q = 1; q < NGR; ++q)
        if (j == q) {
          lo = glo[q];
          hi = ghi[q];
        }
    } else {
      lo = __ldg(gptr + u);
      hi = __ldg(gptr + u + 1);
    }
    for (int q = lo; q < hi; ++q) {
      const int slot = sgslot[q];
      const int el = slot / NN, a = slot - el * NN;
#pragma unroll
      for (int k = 0; k < NV; ++k) s[k] += sm[(a * NV + k) * kBlockElems + el];
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) partial[(base + u) * NV + k] = s[k];
  }
}

// ---- pipelined persistent variant (affine simplices) ---------------------------
// Same arithmetic and summation order as k_blk_rhs (bitwise identical
// partials), but each CTA walks blocks blk0 + blockIdx.x, + gridDim.x, ... and
// double-buffers the node staging: while block b is integrated and gathered,
// block b + gridDim.x's node records, velocity rows and gather slots are
// already in flight into the other buffer with cp.async (16-byte record
// halves, 8-byte velocity components), and its node ids, element-local
// indices and gather ranges are fetched into registers one block ahead.  The
// gather -> record -> stage dependency chain that k_blk_rhs exposes once per
// block (profiles/r02d_mom: ~31 % of its stall samples) overlaps the
// previous block's FP64 work.
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <int ET, int KIND>
__global__ void __launch_bounds__(kBlockThreads, 4)
k_blk_rhs_pipe(int64_t nelem, int64_t blk0, int64_t blk1, const uint16_t* __restrict__ blk_lidx,
               const double* __restrict__ xyz4, const double* __restrict__ vel, const double* __restrict__ phi,
               int64_t fstride, double rho, double mu, double kappa, const int32_t* __restrict__ blk_ptr,
               const int32_t* __restrict__ blk_nodes, const uint16_t* __restrict__ blk_gptr,
               const uint16_t* __restrict__ blk_gslot, int maxnu, double* __restrict__ partial) {
  constexpr int NN = Elem<ET>::NN, DIM = Elem<ET>::DIM;
  constexpr int NV = Out<ET, KIND>::NV;
  constexpr int NF = KIND == FPB_SCALAR_RHS ? 1 : KIND == KIND_SCALAR3 ? 3 : 0;
  constexpr int NU = DIM + NF;  // velocity (+ scalars) per staged node
  constexpr int TPB = kBlockThreads;
  constexpr int kBlockElems = blk_elems<ET>();
  constexpr int EPT = kBlockElems / TPB;
  constexpr int NGR = 3;  // node slots per thread (nu <= 3 TPB)
  static_assert(Elem<ET>::AFFINE && EPT == 2 && NN == 4 - (DIM == 2),
                "pipelined block kernel: affine simplices, 2 elements per thread");
  extern __shared__ __align__(16) double smem[];
  double* const sm = smem;                                                      // [NN * NV][kBlockElems]
  uint16_t* const sgs = reinterpret_cast<uint16_t*>(sm + NN * NV * kBlockElems);  // [2][NN * kBlockElems] slots
  uint16_t* const sli = sgs + 2 * NN * kBlockElems;                             // [2][kBlockElems * NN] local ids
  double* const sx = sm + NN * NV * kBlockElems + NN * kBlockElems;             // [2][maxnu][4]
  double* const su = sx + 2 * maxnu * 4;                                        // [2][maxnu][NU]
  const int tid = threadIdx.x;
  const int64_t stride = gridDim.x;

  // a block's staging inputs, fetched one block ahead: partial base, node
  // count, the node ids of my staging slots
  struct Ids {
    int64_t base;
    int nu;
    int node[NGR];
  };
  auto fetch_ids = [&](int64_t b, Ids& m) {
    m.nu = 0;
    m.base = 0;
    if (b >= blk1) return;
    m.base = __ldg(blk_ptr + b);
    m.nu = __ldg(blk_ptr + b + 1) - (int)m.base;
#pragma unroll
    for (int j = 0; j < NGR; ++j) {
      const int u = tid + j * TPB;
      m.node[j] = u < m.nu ? __ldg(blk_nodes + m.base + u) : 0;
    }
  };
  // cp.async the block's node data, gather slots and local ids into buffer q
  auto stage = [&](int64_t b, const Ids& m, int q) {
    if (b < blk1) {
      const uint16_t* gs = blk_gslot + b * kBlockElems * NN;
      const uint16_t* li = blk_lidx + b * kBlockElems * NN;
      uint16_t* g = sgs + q * NN * kBlockElems;
      uint16_t* l = sli + q * NN * kBlockElems;
      const int64_t nvalid = min((int64_t)kBlockElems, nelem - b * kBlockElems) * NN;  // lidx ends with the mesh
      for (int c = tid; c < NN * kBlockElems / 8; c += TPB) {
        cp_async16(g + 8 * c, gs + 8 * c);
        if (8 * c < nvalid) cp_async16(l + 8 * c, li + 8 * c);
      }
      double* x = sx + q * maxnu * 4;
      double* u = su + q * maxnu * NU;
#pragma unroll
      for (int j = 0; j < NGR; ++j) {
        const int v = tid + j * TPB;
        if (v < m.nu) {
          const int64_t nd = m.node[j];
          cp_async16(x + v * 4, xyz4 + 4 * nd);
          cp_async16(x + v * 4 + 2, xyz4 + 4 * nd + 2);
#pragma unroll
          for (int d = 0; d < DIM; ++d) cp_async8(u + v * NU + d, vel + nd * DIM + d);
          if constexpr (KIND == FPB_SCALAR_RHS) cp_async8(u + v * NU + DIM, phi + nd);
          if constexpr (KIND == KIND_SCALAR3) {
#pragma unroll
            for (int f = 0; f < 3; ++f) cp_async8(u + v * NU + DIM + f, phi + f * fstride + nd);
          }
        }
      }
    }
    cp_async_commit();  // (an empty group past the window keeps the wait count uniform)
  };

  int64_t b = blk0 + blockIdx.x;
  Ids cur, nxt;
  fetch_ids(b, cur);
  stage(b, cur, 0);
  fetch_ids(b + stride, nxt);
  int q = 0;
  for (; b < blk1; b += stride, q ^= 1) {
    stage(b + stride, nxt, q ^ 1);  // the next block is in flight while this one computes
    Ids nn2;
    fetch_ids(b + 2 * stride, nn2);  // ids two blocks ahead, for the next iteration's stage
    // this block's gather ranges (consumed after the integration)
    int glo[NGR], ghi[NGR];
    const uint16_t* gptr = blk_gptr + cur.base + b;
#pragma unroll
    for (int j = 0; j < NGR; ++j) {
      const int v = tid + j * TPB;
      glo[j] = v < cur.nu ? __ldg(gptr + v) : 0;
      ghi[j] = v < cur.nu ? __ldg(gptr + v + 1) : 0;
    }
    cp_async_wait_1();  // this block's group has landed
    __syncthreads();
    const double* x = sx + q * maxnu * 4;
    const double* u = su + q * maxnu * NU;
    const uint16_t* l = sli + q * NN * kBlockElems;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int el = tid + j * TPB;
      if (b * kBlockElems + el >= nelem) break;
      int li[NN];
      if constexpr (NN == 4) {
        const uint2 v = *reinterpret_cast<const uint2*>(l + el * NN);
        li[0] = v.x & 0xffff; li[1] = v.x >> 16; li[2] = v.y & 0xffff; li[3] = v.y >> 16;
      } else {
#pragma unroll
        for (int a = 0; a < NN; ++a) li[a] = l[el * NN + a];
      }
      double xe[NN][DIM], ue[Out<ET, KIND>::NU][DIM], fe[Out<ET, KIND>::NF];
#pragma unroll
      for (int a = 0; a < NN; ++a) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          xe[a][d] = x[li[a] * 4 + d];
          ue[a][d] = u[li[a] * NU + d];
        }
        if constexpr (KIND == FPB_SCALAR_RHS) fe[a] = u[li[a] * NU + DIM];
        if constexpr (KIND == KIND_SCALAR3) {
#pragma unroll
          for (int f = 0; f < 3; ++f) fe[f * NN + a] = u[li[a] * NU + DIM + f];
        }
      }
      double acc[Out<ET, KIND>::NOUT];
      simplex_rhs_all<ET, KIND>(xe, ue, fe, rho, mu, kappa, acc);
#pragma unroll
      for (int a = 0; a < NN; ++a)
#pragma unroll
        for (int k = 0; k < NV; ++k) sm[(a * NV + k) * kBlockElems + el] = acc[a * NV + k];
    }
    __syncthreads();
    const uint16_t* g = sgs + q * NN * kBlockElems;
#pragma unroll
    for (int j = 0; j < NGR; ++j) {
      const int v = tid + j * TPB;
      if (v >= cur.nu) break;
      double sv[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) sv[k] = 0.0;
      for (int t = glo[j]; t < ghi[j]; ++t) {
        const int slot = g[t];
        const int el = slot / NN, a = slot - el * NN;
#pragma unroll
        for (int k = 0; k < NV; ++k) sv[k] += sm[(a * NV + k) * kBlockElems + el];
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) partial[(cur.base + v) * NV + k] = sv[k];
    }
    __syncthreads();  // sm and buffer q are reused two stages on
    cur = nxt;
    nxt = nn2;
  }
  cp_async_wait_all();
}

// ---- phase 2: per-node gather of block partials ---------------------------------
// out[i][k] (node-major), or out[k][fstride] (field-major) when fstride > 0
template <int NV>
__global__ void k_blk_gather(int32_t node0, int32_t node1, const int32_t* __restrict__ ptr,
                             const int32_t* __restrict__ list, const double* __restrict__ partial, int accumulate,
                             double* __restrict__ out, int64_t fstride = 0) {
  for (int64_t i = node0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < node1;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = 0.0;
    const int lo = __ldg(ptr + i), hi = __ldg(ptr + i + 1);
    for (int q = lo; q < hi; ++q) {
      const int64_t p = __ldg(list + q);
#pragma unroll
      for (int k = 0; k < NV; ++k) s[k] += __ldg(partial + p * NV + k);
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double* o = fstride > 0 ? out + k * fstride + i : out + i * NV + k;
      *o = accumulate ? *o + s[k] : s[k];
    }
  }
}

template <int ET, int KIND>
static int launch_blk(int64_t nelem, int64_t blk0, int64_t blk1, const uint16_t* lidx, const double* xyz4, const double* uvw4,
                      const double* vel, const double* phi, int64_t fstride,
                      double rho, double mu, double kappa, const int32_t* blk_ptr,
                      const int32_t* blk_nodes, const uint16_t* blk_gptr, const uint16_t* blk_gslot,
                      int maxnu, double* partial, cudaStream_t s) {
  constexpr int NV = Out<ET, KIND>::NV;
  constexpr int NDAT = 2 * Elem<ET>::DIM + (KIND == FPB_SCALAR_RHS ? 1 : KIND == KIND_SCALAR3 ? 3 : 0);
  constexpr int kBlockElems = blk_elems<ET>();
  const int64_t nblocks = (nelem + kBlockElems - 1) / kBlockElems;
  const size_t contrib = (size_t)Elem<ET>::NN * NV * kBlockElems * sizeof(double) +
                         (size_t)Elem<ET>::NN * kBlockElems * sizeof(uint16_t);
  const size_t smem = contrib + (size_t)maxnu * NDAT * sizeof(double);
  FPB_REQUIRE(smem <= 227 * 1024, "element block needs %zu bytes of shared memory", smem);
  if (smem > 48 * 1024)
    FPB_CUDA(cudaFuncSetAttribute(k_blk_rhs<ET, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  FPB_REQUIRE(blk0 >= 0 && blk0 <= blk1 && blk1 <= nblocks, "block window [%lld, %lld) outside [0, %lld)",
              (long long)blk0, (long long)blk1, (long long)nblocks);
  if (blk1 == blk0) return FPB_OK;
  if constexpr (Elem<ET>::AFFINE && kBlockElems / kBlockThreads == 2) {
    if (g_tuning_blk_pipe && uvw4 == nullptr && maxnu <= 3 * kBlockThreads) {
      constexpr int NU = Elem<ET>::DIM + (KIND == FPB_SCALAR_RHS ? 1 : KIND == KIND_SCALAR3 ? 3 : 0);
      const size_t psmem = (size_t)Elem<ET>::NN * NV * kBlockElems * sizeof(double) +
                           4 * (size_t)Elem<ET>::NN * kBlockElems * sizeof(uint16_t) +
                           2 * (size_t)maxnu * (4 + NU) * sizeof(double);
      FPB_REQUIRE(psmem <= 227 * 1024, "element block needs %zu bytes of shared memory", psmem);
      auto kern = k_blk_rhs_pipe<ET, KIND>;
      FPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
      int per_sm = 0;
      FPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlockThreads, psmem));
      int dev = 0, nsm = kNumSMs;
      FPB_CUDA(cudaGetDevice(&dev));
      FPB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      const int64_t grid = std::min<int64_t>(blk1 - blk0, (int64_t)std::max(per_sm, 1) * nsm);
      kern<<<(unsigned)grid, kBlockThreads, psmem, s>>>(nelem, blk0, blk1, lidx, xyz4, vel, phi, fstride, rho, mu,
                                                        kappa, blk_ptr, blk_nodes, blk_gptr, blk_gslot, maxnu,
                                                        partial);
      FPB_LAUNCH_CHECK();
      return FPB_OK;
    }
  }
  k_blk_rhs<ET, KIND><<<(unsigned)(blk1 - blk0), kBlockThreads, smem, s>>>(nelem, blk0, lidx, xyz4, uvw4, vel, phi, fstride,
                                                                   rho, mu, kappa,
                                                                   blk_ptr, blk_nodes, blk_gptr, blk_gslot, maxnu,
                                                                   partial);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

template <int ET>
static int blk_kind(int kind, int64_t nelem, int64_t blk0, int64_t blk1, const uint16_t* lidx, const double* xyz4, const double* uvw4,
                    const double* vel, const double* phi, int64_t fstride,
                    double rho, double mu, double kappa, const int32_t* blk_ptr,
                    const int32_t* blk_nodes, const uint16_t* blk_gptr, const uint16_t* blk_gslot, int maxnu,
                    double* partial, cudaStream_t s) {
  if (kind == FPB_MOMENTUM_RHS)
    return launch_blk<ET, FPB_MOMENTUM_RHS>(nelem, blk0, blk1, lidx, xyz4, uvw4, vel, phi, 0, rho, mu, kappa, blk_ptr,
                                            blk_nodes, blk_gptr, blk_gslot, maxnu, partial, s);
  if (kind == KIND_SCALAR3)
    return launch_blk<ET, KIND_SCALAR3>(nelem, blk0, blk1, lidx, xyz4, nullptr, vel, phi, fstride, rho, mu, kappa,
                                        blk_ptr, blk_nodes, blk_gptr, blk_gslot, maxnu, partial, s);
  return launch_blk<ET, FPB_SCALAR_RHS>(nelem, blk0, blk1, lidx, xyz4, uvw4, vel, phi, 0, rho, mu, kappa, blk_ptr,
                                        blk_nodes, blk_gptr, blk_gslot, maxnu, partial, s);
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_block_elems(int etype) { return blk_elems_rt(etype); }

// setup kernel launch for (node count, block size)
static void launch_setup(int nn, int be, int64_t nblocks, cudaStream_t s, int64_t nelem, const int32_t* conn,
                         int pass, int32_t* cnt, const int32_t* blk_ptr, int32_t* blk_nodes, uint16_t* blk_gptr,
                         uint16_t* blk_gslot, uint16_t* blk_lidx) {
#define FPB_SETUP(NN_, BE_)                                                                                      \
  k_blk_setup<NN_, BE_><<<(unsigned)nblocks, BE_, 0, s>>>(nelem, conn, pass, cnt, blk_ptr, blk_nodes, blk_gptr, \
                                                          blk_gslot, blk_lidx)
  if (be == FPB_BLK_ELEMS) {
    if (nn == 3) FPB_SETUP(3, FPB_BLK_ELEMS);
    else FPB_SETUP(4, FPB_BLK_ELEMS);
  } else {
    if (nn == 4) FPB_SETUP(4, FPB_BLK_ELEMS_GAUSS);
    else if (nn == 5) FPB_SETUP(5, FPB_BLK_ELEMS_GAUSS);
    else FPB_SETUP(8, FPB_BLK_ELEMS_GAUSS);
  }
#undef FPB_SETUP
}

int fpb_blocks_build(int etype, int64_t nelem, const int32_t* conn, int32_t n, int32_t* blk_ptr,
                     int32_t* blk_nodes, uint16_t* blk_gptr, uint16_t* blk_gslot, uint16_t* blk_lidx,
                     int32_t* node_pptr, int32_t* node_plist, int64_t* npartial_h, int* maxnu_h,
                     void* stream) {
  FPB_REQUIRE(etype >= 0 && etype < 5, "unsupported element type %d", etype);
  FPB_REQUIRE(nelem >= 0 && n >= 0, "bad sizes");
  cudaStream_t s = as_stream(stream);
  const int nn = etype_nn(etype), be = blk_elems_rt(etype);
  const int64_t nblocks = (nelem + be - 1) / be;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  if (blk_nodes == nullptr) {  // pass 0: sizes
    int32_t* cnt = nullptr;
    FPB_CUDA(cudaMallocAsync(&cnt, sizeof(int32_t) * (nblocks + 1), s));
    FPB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nblocks + 1), s));
    if (nblocks > 0) {
      launch_setup(nn, be, nblocks, s, nelem, conn, 0, cnt, nullptr, nullptr, nullptr, nullptr, nullptr);
      FPB_LAUNCH_CHECK();
    }
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, blk_ptr, nblocks + 1, s);
    FPB_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
    FPB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, blk_ptr, nblocks + 1, s));
    int32_t P = 0;
    FPB_CUDA(cudaMemcpyAsync(&P, blk_ptr + nblocks, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    int32_t* mx = nullptr;
    FPB_CUDA(cudaMallocAsync(&mx, sizeof(int32_t), s));
    FPB_CUDA(cudaMemsetAsync(mx, 0, sizeof(int32_t), s));
    if (nblocks > 0) k_max_count<<<grid_for(nblocks, 256), 256, 0, s>>>(nblocks, cnt, mx);
    int32_t mxh = 0;
    FPB_CUDA(cudaMemcpyAsync(&mxh, mx, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    FPB_CUDA(cudaFreeAsync(mx, s));
    FPB_CUDA(cudaFreeAsync(tmp, s));
    FPB_CUDA(cudaFreeAsync(cnt, s));
    FPB_CUDA(cudaStreamSynchronize(s));
    *npartial_h = P;
    *maxnu_h = mxh;
    return FPB_OK;
  }
  const int64_t P = *npartial_h;
  if (nblocks > 0) {
    launch_setup(nn, be, nblocks, s, nelem, conn, 1, nullptr, blk_ptr, blk_nodes, blk_gptr, blk_gslot, blk_lidx);
    FPB_LAUNCH_CHECK();
  }
  int32_t* cnt = nullptr;
  FPB_CUDA(cudaMallocAsync(&cnt, sizeof(int32_t) * (n + 1), s));
  FPB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), s));
  if (P > 0) k_p2_count<<<grid_for(P, 256), 256, 0, s>>>(P, blk_nodes, cnt);
  FPB_LAUNCH_CHECK();
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, node_pptr, n + 1, s);
  FPB_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
  FPB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, node_pptr, n + 1, s));
  FPB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), s));
  if (P > 0) k_p2_fill<<<grid_for(P, 256), 256, 0, s>>>(P, blk_nodes, node_pptr, cnt, node_plist);
  if (n > 0) k_p2_sort<<<grid_for(n, 256), 256, 0, s>>>(n, node_pptr, node_plist);
  FPB_LAUNCH_CHECK();
  FPB_CUDA(cudaFreeAsync(tmp, s));
  FPB_CUDA(cudaFreeAsync(cnt, s));
  return FPB_OK;
}

int fpb_assemble_blocks(int kind, int etype, int64_t nelem, int64_t blk0, int64_t blk1, const double* xyz4,
                        const double* uvw4, const double* vel, const double* phi,
                        double rho, double mu, double kappa, const int32_t* blk_ptr,
                        const int32_t* blk_nodes, const uint16_t* blk_gptr, const uint16_t* blk_gslot,
                        const uint16_t* blk_lidx, int maxnu, double* partial, int32_t n, int32_t node0,
                        int32_t node1, const int32_t* node_pptr, const int32_t* node_plist, int accumulate,
                        double* out, void* stream) {
  FPB_REQUIRE(etype >= 0 && etype < 5 && g_ref_loaded[etype],
              "reference tables for element type %d not uploaded", etype);
  FPB_REQUIRE(kind == FPB_MOMENTUM_RHS || kind == FPB_SCALAR_RHS,
              "element-block assembly covers the RHS kinds (got %d)", kind);
  FPB_REQUIRE(xyz4 != nullptr && (uvw4 != nullptr || (vel != nullptr && (kind != FPB_SCALAR_RHS || phi))),
              "kind %d needs node records or the velocity (+ scalar) arrays", kind);
  cudaStream_t s = as_stream(stream);
  if (nelem > 0) {
    int rc = FPB_OK;
    switch (etype) {
      case FPB_TRI03: rc = blk_kind<FPB_TRI03>(kind, nelem, blk0, blk1, blk_lidx, xyz4, uvw4, vel, phi, 0, rho, mu, kappa, blk_ptr, blk_nodes, blk_gptr, blk_gslot, maxnu, partial, s); break;
      case FPB_QUAD04: rc = blk_kind<FPB_QUAD04>(kind, nelem, blk0, blk1, blk_lidx, xyz4, uvw4, vel, phi, 0, rho, mu, kappa, blk_ptr, blk_nodes, blk_gptr, blk_gslot, maxnu, partial, s); break;
      case FPB_TET04: rc = blk_kind<FPB_TET04>(kind, nelem, blk0, blk1, blk_lidx, xyz4, uvw4, vel, phi, 0, rho, mu, kappa, blk_ptr, blk_nodes, blk_gptr, blk_gslot, maxnu, partial, s); break;
      case FPB_PYR05: rc = blk_kind<FPB_PYR05>(kind, nelem, blk0, blk1, blk_lidx, xyz4, uvw4, vel, phi, 0, rho, mu, kappa, blk_ptr, blk_nodes, blk_gptr, blk_gslot, maxnu, partial, s); break;
      case FPB_HEX08: rc = blk_kind<FPB_HEX08>(kind, nelem, blk0, blk1, blk_lidx, xyz4, uvw4, vel, phi, 0, rho, mu, kappa, blk_ptr, blk_nodes, blk_gptr, blk_gslot, maxnu, partial, s); break;
    }
    if (rc) return rc;
  }
  FPB_REQUIRE(node0 >= 0 && node0 <= node1 && node1 <= n, "node window [%d, %d) outside [0, %d)", node0, node1, n);
  if (node1 > node0) {
    const int64_t w = node1 - node0;
    if (kind == FPB_MOMENTUM_RHS && etype_dim(etype) == 3)
      k_blk_gather<3><<<grid_for(w, 256), 256, 0, s>>>(node0, node1, node_pptr, node_plist, partial, accumulate, out);
    else if (kind == FPB_MOMENTUM_RHS)
      k_blk_gather<2><<<grid_for(w, 256), 256, 0, s>>>(node0, node1, node_pptr, node_plist, partial, accumulate, out);
    else
      k_blk_gather<1><<<grid_for(w, 256), 256, 0, s>>>(node0, node1, node_pptr, node_plist, partial, accumulate, out);
    FPB_LAUNCH_CHECK();
  }
  return FPB_OK;
}

int fpb_assemble_blocks_scalar3(int etype, int64_t nelem, int64_t blk0, int64_t blk1, const double* xyz4,
                                const double* vel, const double* phi3, double kappa0, double kappa1, double kappa2,
                                const int32_t* blk_ptr, const int32_t* blk_nodes, const uint16_t* blk_gptr,
                                const uint16_t* blk_gslot, const uint16_t* blk_lidx, int maxnu, double* partial,
                                int32_t n, int32_t node0, int32_t node1, const int32_t* node_pptr,
                                const int32_t* node_plist, int accumulate, double* out3, void* stream) {
  FPB_REQUIRE(etype >= 0 && etype < 5 && g_ref_loaded[etype],
              "reference tables for element type %d not uploaded", etype);
  FPB_REQUIRE(xyz4 && vel && phi3 && out3, "three-scalar RHS needs node records, velocity, phi[3][n], out[3][n]");
  cudaStream_t s = as_stream(stream);
  if (nelem > 0) {
    int rc = FPB_OK;
#define FPB_S3(ET_)                                                                                               \
  rc = blk_kind<ET_>(KIND_SCALAR3, nelem, blk0, blk1, blk_lidx, xyz4, nullptr, vel, phi3, n, kappa0, kappa1, kappa2, \
                     blk_ptr, blk_nodes, blk_gptr, blk_gslot, maxnu, partial, s)
    switch (etype) {
      case FPB_TRI03: FPB_S3(FPB_TRI03); break;
      case FPB_QUAD04: FPB_S3(FPB_QUAD04); break;
      case FPB_TET04: FPB_S3(FPB_TET04); break;
      case FPB_PYR05: FPB_S3(FPB_PYR05); break;
      case FPB_HEX08: FPB_S3(FPB_HEX08); break;
    }
#undef FPB_S3
    if (rc) return rc;
  }
  FPB_REQUIRE(node0 >= 0 && node0 <= node1 && node1 <= n, "node window [%d, %d) outside [0, %d)", node0, node1, n);
  if (node1 > node0) {
    const int64_t w = node1 - node0;
    k_blk_gather<3><<<grid_for(w, 256), 256, 0, s>>>(node0, node1, node_pptr, node_plist, partial, accumulate, out3, n);
    FPB_LAUNCH_CHECK();
  }
  return FPB_OK;
}

}  // extern "C"
