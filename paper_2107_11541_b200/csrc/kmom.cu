// Momentum RHS on a Kuhn box mesh by z-marching cell lines (TET04).
//
// The reference's generate_box_mesh(TET04, nx, ny, nz) (mesh.py:258-282)
// cuts every grid cell (i, j, k) into six tetrahedra that all contain the
// cell origin v0 as local node 0 and the far corner v7.  When a mesh's
// connectivity is exactly that (checked element by element on the device at
// setup, assembly.py KuhnBox) the momentum RHS of _kernels.py:320-382 +
// the scatter of :511-519 is assembled without any per-element metadata:
//
//   CTA (chunk c, cell row j) owns the x-line of cells (0..nx-1, j) and walks
//   the cell layers k of its z-chunk, one thread per cell column i.  Node
//   data of two node layers x two node rows are staged in shared memory
//   (structure of arrays, cp.async one layer ahead); each thread integrates
//   its cell's six tets (tet_mom_adj, simplex.cuh) into eight corner
//   accumulators held in registers.  Reductions:
//     z: the top-face accumulators become the next cell's bottom face;
//     x: a thread's right-hand corners go through shared memory to the
//        thread on its right;
//     y: node row j+1 also receives row j+1's cells: this CTA publishes its
//        partial of node row j+1 (pup, an n x 3 scratch) layer by layer
//        with a release flag, and the CTA of row j+1 adds it when it writes
//        node row j, one layer later (no chain waits in the steady state).
//   z-chunks: a chunk first integrates the cell layer below it (halo) for
//   the contributions to its lowest node layer, so chunks are independent.
// CTAs take (chunk, row) tickets in launch order, so the CTA a row waits for
// has always started: no deadlock whatever the residency.
// Every node is written exactly once, each sum has a fixed order (bitwise
// reproducible) and nothing is zero-filled.
#include "simplex.cuh"

namespace fpb {

// corner c = di + 2 dj + 4 dk of the cell; tets in the generator's
// permutation order (mesh.py:212-213), odd ones with the last two swapped
// {0,1,3,7} {0,2,6,7} {0,4,5,7} {0,1,7,5} {0,4,7,6} {0,2,7,3}, one nibble per node
__host__ __device__ constexpr int kuhn_corner(int t, int a) {
  return (int)(((t == 0 ? 0x7310u : t == 1 ? 0x7620u : t == 2 ? 0x7540u : t == 3 ? 0x5710u : t == 4 ? 0x6740u : 0x3720u) >>
                (4 * a)) & 15u);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cp8(double* smem_dst, const double* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

#ifndef FPB_KMOM_MINB
#define FPB_KMOM_MINB 2
#endif

template <int MAXT>
__global__ void __launch_bounds__(MAXT, FPB_KMOM_MINB)
k_kuhn_mom(int nx, int ny, int nz, int kchunk, const double* __restrict__ xyz4, const double* __restrict__ vel,
           double rho, double mu, int* __restrict__ sync, double* __restrict__ pup, double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  const int NP = nx + 1;                      // nodes per node row
  const int T = blockDim.x, tid = threadIdx.x;
  double* const stg = sm;                     // [3 layers][2 rows][6 comps][NP]
  double* const xl = stg + 36 * NP;           // [2 rows][3][NP]: corners di = 0 of thread i
  double* const xr = xl + 6 * NP;             // [2 rows][3][NP]: corners di = 1 of thread i - 1
  double* const own = xr + 6 * NP;            // [2 slots][3][NP]: node row j, thread-private
  const double r = rho * c_ref[FPB_TET04].M[1];  // M[0][1] = W / 20
  const double muW = mu * c_ref[FPB_TET04].W;
  __shared__ int s_ticket;
  if (tid == 0) s_ticket = atomicAdd(sync, 1);
  for (int i = tid; i < 6 * NP; i += T) {  // xr[.][.][0] and xl[.][.][nx] stay zero
    xl[i] = 0.0;
    xr[i] = 0.0;
  }
  __syncthreads();
  const int ticket = s_ticket;
  const int c = ticket / ny, j = ticket - c * ny;
  const int nchunk = (nz + kchunk - 1) / kchunk;
  const int kb = c * kchunk, ke = min(nz, kb + kchunk);
  const int kfirst = c > 0 ? kb - 1 : kb;          // halo cell layer below the chunk
  const int klast = c == nchunk - 1 ? nz : ke - 1;  // last node layer written (nz: the top face)
  const int ktop = ke;                               // highest node layer staged
  int* const flags = sync + 1 + (size_t)c * ny;      // layers of row j+1's partial published
  const int64_t row = NP, layer = (int64_t)NP * (ny + 1);

  auto stage = [&](int kl) {  // node layer kl, node rows j, j+1 -> stg[kl % 3]
    double* s = stg + (kl % 3) * 12 * NP;
    for (int i = tid; i < NP; i += T) {
#pragma unroll
      for (int dj = 0; dj < 2; ++dj) {
        const int64_t nd = i + (j + dj) * row + kl * layer;
        double* t = s + dj * 6 * NP + i;
        cp8(t, xyz4 + 4 * nd);
        cp8(t + NP, xyz4 + 4 * nd + 1);
        cp8(t + 2 * NP, xyz4 + 4 * nd + 2);
        cp8(t + 3 * NP, vel + 3 * nd);
        cp8(t + 4 * NP, vel + 3 * nd + 1);
        cp8(t + 5 * NP, vel + 3 * nd + 2);
      }
    }
    cp_commit();
  };

  stage(kfirst);
  stage(kfirst + 1);
  double bot[4][3];  // corners dk = 0: (di, dj) = c & 3
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int d = 0; d < 3; ++d) bot[q][d] = 0.0;
  const bool cell = tid < nx;

  for (int k = kfirst; k <= klast; ++k) {
    cp_wait_all();
    // node row j of layer k - 1 is written below: row j - 1's partial of it
    // must be published (it was, one layer ago, unless that CTA lags)
    if (tid == 0 && j > 0 && k - 1 >= kb) {
      const int need = k - kb;
      while (ld_acquire(flags + j - 1) < need) __nanosleep(64);
    }
    __syncthreads();
    if (tid == 0 && j + 1 < ny && k - 1 >= kb) st_release(flags + j, k - kb);  // layer k - 1 of row j + 1
    if (k + 2 <= ktop) stage(k + 2);
    if (k - 1 >= kb) {  // deferred write-out of node row j, layer k - 1
      const int sl = (k - 1) & 1;
      for (int i = tid; i < NP; i += T) {
        const int64_t nd = i + j * row + (int64_t)(k - 1) * layer;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double o = own[(sl * 3 + d) * NP + i];
          out[3 * nd + d] = j > 0 ? __ldcg(pup + 3 * nd + d) + o : o;
        }
      }
    }
    double top[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int d = 0; d < 3; ++d) top[q][d] = 0.0;
    if (cell && k < nz) {
      const double* s0 = stg + (k % 3) * 12 * NP + tid;
      const double* s1 = stg + ((k + 1) % 3) * 12 * NP + tid;
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        asm volatile("" ::: "memory");  // one tet's node loads at a time (register pressure)
        double xe[4][3], ue[4][3];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int cc = kuhn_corner(t, a);
          const double* s = ((cc & 4) ? s1 : s0) + ((cc >> 1) & 1) * 6 * NP + (cc & 1);
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            xe[a][d] = s[d * NP];
            ue[a][d] = s[(3 + d) * NP];
          }
        }
        tet_mom_adj_f(xe, ue, r, muW, [&](int a, int d, double v) {
          const int cc = kuhn_corner(t, a);
          if (cc & 4) top[cc & 3][d] -= v;
          else bot[cc & 3][d] -= v;
        });
      }
    }
    if (cell && k >= kb) {  // bottom face complete in z: split by x owner
#pragma unroll
      for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          xl[(dj * 3 + d) * NP + tid] = bot[2 * dj][d];
          xr[(dj * 3 + d) * NP + tid + 1] = bot[2 * dj + 1][d];
        }
    }
    __syncthreads();
    if (k >= kb) {
      const int sl = k & 1;
      bool wrote = false;
      for (int i = tid; i < NP; i += T) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          own[(sl * 3 + d) * NP + i] = xl[d * NP + i] + xr[d * NP + i];
          const double s1v = xl[(3 + d) * NP + i] + xr[(3 + d) * NP + i];
          const int64_t nd = i + (j + 1) * row + (int64_t)k * layer;
          if (j + 1 < ny) pup[3 * nd + d] = s1v;
          else out[3 * nd + d] = s1v;
        }
        wrote = true;
      }
      if (wrote && j + 1 < ny) __threadfence();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int d = 0; d < 3; ++d) bot[q][d] = top[q][d];
  }
  // last node layer of row j: publish ours first, then wait for row j - 1
  __syncthreads();
  if (tid == 0) {
    if (j + 1 < ny) st_release(flags + j, klast - kb + 1);
    if (j > 0)
      while (ld_acquire(flags + j - 1) < klast - kb + 1) __nanosleep(64);
  }
  __syncthreads();
  {
    const int sl = klast & 1;
    for (int i = tid; i < NP; i += T) {
      const int64_t nd = i + j * row + (int64_t)klast * layer;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double o = own[(sl * 3 + d) * NP + i];
        out[3 * nd + d] = j > 0 ? __ldcg(pup + 3 * nd + d) + o : o;
      }
    }
  }
}

inline size_t kmom_smem(int nx) { return (size_t)(36 + 6 + 6 + 6) * (nx + 1) * sizeof(double); }

}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_kuhn_mom_sync_len(int ny, int nz, int kchunk) {
  if (ny < 1 || nz < 1 || kchunk < 1) return 0;
  return 1 + ny * ((nz + kchunk - 1) / kchunk);
}

int fpb_assemble_momentum_kuhn(int nx, int ny, int nz, int kchunk, const double* xyz4, const double* vel,
                               double rho, double mu, int32_t* sync, double* pup, double* out, void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  FPB_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && nx <= 256, "Kuhn box %d x %d x %d: need 1 <= nx <= 256", nx, ny, nz);
  FPB_REQUIRE(kchunk >= 1, "bad z chunk %d", kchunk);
  FPB_REQUIRE(xyz4 && vel && sync && pup && out, "null argument");
  cudaStream_t s = as_stream(stream);
  const int nchunk = (nz + kchunk - 1) / kchunk;
  const int nsync = 1 + ny * nchunk;
  FPB_CUDA(cudaMemsetAsync(sync, 0, sizeof(int32_t) * nsync, s));
  const size_t smem = kmom_smem(nx);
  const int T = (nx + 31) / 32 * 32;
  auto kern = k_kuhn_mom<256>;
  FPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)(ny * nchunk), T, smem, s>>>(nx, ny, nz, kchunk, xyz4, vel, rho, mu, sync, pup, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

}  // extern "C"
