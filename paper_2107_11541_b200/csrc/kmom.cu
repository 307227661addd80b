// Momentum RHS on a Kuhn box mesh by z-marching cell pencils (TET04).
//
// The reference's generate_box_mesh(TET04, nx, ny, nz) (mesh.py:258-282)
// cuts every grid cell (i, j, k) into six tetrahedra that all contain the
// cell origin v0 as local node 0 and the far corner v7.  When a mesh's
// connectivity is exactly that (checked element by element on the device at
// setup, assembly.py KuhnBox) the momentum RHS of _kernels.py:320-382 + the
// scatter of :511-519 is assembled with no per-element metadata at all:
//
//   CTA (x-block a, y-block b, z-chunk c) owns the 32 x kKmomTY cell
//   columns (i0 + lane, j0 + warp) and walks the cell layers k of its
//   z-chunk; one thread per cell column.  Each warp stages the node data it
//   needs (two node layers x two node rows x 33 node columns, structure of
//   arrays, cp.async two layers ahead) in its own shared-memory slice and
//   integrates its cell's six tets (tet_mom_adj_f, simplex.cuh) into eight
//   corner accumulators held in registers.  Reductions:
//     z: the top-face accumulators become the next cell's bottom face;
//     x: right-hand corners move one lane up by a warp shuffle;
//     y: a warp's top node row goes to the warp above through a
//        shared-memory ring (volatile full / consumed counters);
//   the warps of a CTA never meet at a barrier.  Contributions that cross a
//   CTA boundary — the right-edge node column and the CTA's top node row —
//   go to small per-CTA partial buffers (Px, Py), and k_kuhn_fixup adds
//   them to the boundary nodes afterwards (stream order; no inter-CTA
//   synchronisation).  z-chunks integrate the cell layer below them (halo)
//   for the contributions to their lowest node layer, so they are
//   independent too.  Every sum has a fixed order: bitwise reproducible.
//
// The same pencils run four per-cell integrands (template KIND): 0 = TET04
// momentum (six Kuhn tets, shared-node cycle, tet_mom_core), 1 = TET04 three
// scalars (tet_s3_core), 2 / 3 = HEX08 momentum / three scalars (one Q1 hex
// per cell of the generator's hex box, hex_rhs_integrate).  A cell-layer
// range [kc0, kc1) restricts the integration to a z-slab's own layers.
#include <algorithm>

#include "simplex.cuh"

namespace fpb {

// corner c = di + 2 dj + 4 dk of the cell; tets in the generator's
// permutation order (mesh.py:212-213), odd ones with the last two swapped:
// {0,1,3,7} {0,2,6,7} {0,4,5,7} {0,1,7,5} {0,4,7,6} {0,2,7,3}, one nibble per node
__host__ __device__ constexpr int kuhn_corner(int t, int a) {
  return (int)(((t == 0 ? 0x7310u : t == 1 ? 0x7620u : t == 2 ? 0x7540u : t == 3 ? 0x5710u : t == 4 ? 0x6740u : 0x3720u) >>
                (4 * a)) & 15u);
}

__device__ __forceinline__ void cp8(double* smem_dst, const double* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// y-ring counters: acquire / release at CTA scope on shared memory
__device__ __forceinline__ int yc_acquire(volatile int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
               : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared((const void*)p)) : "memory");
  return v;
}
__device__ __forceinline__ void yc_release(volatile int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;"
               ::"r"((unsigned)__cvta_generic_to_shared((const void*)p)), "r"(v) : "memory");
}

#ifndef FPB_KMOM_TY
#define FPB_KMOM_TY 8
#endif
constexpr int kKmomTY = FPB_KMOM_TY;            // cell rows (warps) per CTA
static_assert(kKmomTY >= 1 && 32 * kKmomTY * 255 <= 65536,
              "the uncapped kinds (up to 255 registers) must fit one CTA of 32 x TY threads per SM");
constexpr int kKmomRing = 4;                    // y-forward slots per warp
constexpr int kKmomSlot = 33 * 3;               // one forwarded node row: [33][3]
constexpr int kKmomHold = 2 * 3 * 33;           // node row j held two layers: [parity][comp][33]
// KIND 0: momentum RHS (x, y, z, u, v, w staged per node); KIND 1: three
// scalar RHS sharing the velocity (+ phi_0, phi_1, phi_2)
// KIND 2 / 3: the same for a HEX08 box (one Q1 hex per cell, hex_rhs_integrate)
template <int KIND> constexpr int kmom_nc() { return (KIND & 1) ? 9 : 6; }
template <int KIND> constexpr int kmom_stg() { return 3 * 2 * kmom_nc<KIND>() * 33; }  // [layer][row][comp][33]
template <int KIND> constexpr int kmom_warp_d() { return kmom_stg<KIND>() + kKmomRing * kKmomSlot + kKmomHold; }

// boundary partials, per CTA (a, b) and node layer k:
//   Px[a][b][k][lr][3], lr = 0..kKmomTY: node column i0 + 32 (the next x-block's
//       first), local node row lr (lr = TY_b: the top-right corner)
//   Py[a][b][k][l][3], l = 0..32: node row j0 + TY_b (the next y-block's first),
//       node column i0 + l (l = 32 only when i0 + 32 == nx)
struct KuhnGrid {
  int nx, ny, nz, nxb, nyb;
  int kc0, kc1;  // cell layers integrated: [kc0, kc1) of the box's nz (a slab's own layers; 0, nz otherwise)
  __host__ __device__ int64_t px(int a, int b, int k, int lr) const {
    return ((((int64_t)a * nyb + b) * (nz + 1) + k) * (kKmomTY + 1) + lr) * 3;
  }
  __host__ __device__ int64_t py(int a, int b, int k, int l) const {
    return (int64_t)nxb * nyb * (nz + 1) * (kKmomTY + 1) * 3 + ((((int64_t)a * nyb + b) * (nz + 1) + k) * 33 + l) * 3;
  }
  __host__ __device__ int64_t scratch() const { return py(nxb, 0, 0, 0); }
};

#ifndef FPB_KMOM_SHARED
#define FPB_KMOM_SHARED 1
#endif
#ifndef FPB_KMOM_S3_SHARED
#define FPB_KMOM_S3_SHARED 1
#endif
#ifdef FPB_KMOM_TETBARRIER  // one tet's node loads at a time (A/B: tighter registers, slower without spills)
#define FPB_KMOM_TETBAR() asm volatile("" ::: "memory")
#else
#define FPB_KMOM_TETBAR() ((void)0)
#endif
// One Kuhn cell, its six tets in the cycle T0 (0,1,3,7), T3 (0,1,7,5), T2
// (0,4,5,7), T4 (0,4,7,6), T1 (0,2,6,7), T5 (0,2,7,3): consecutive tets share
// the cell diagonal, one middle node and one cross product with the diagonal
// edge e7, so each tet after the first loads one new node and forms two new
// cross products.  Edges / velocity differences against corner 0 (e_c, d_c),
// adjugate rows from the crosses (tet_mom_core, simplex.cuh).
template <int KIND>
__device__ __forceinline__ void kuhn_cell_shared(const double* s0, const double* s1, double r, double muW,
                                                 const double (&kW)[3], double (&bot)[4][3], double (&top)[4][3]) {
  constexpr int NC = kmom_nc<KIND>();
  struct Nd {  // differences of one corner against corner 0
    double e[3], du[3], dp[3];
  };
  double x0[3], u0[3], p0[3], u05[3];
  auto ldc = [&](int cc, double (&x)[3], double (&u)[3], double (&ph)[3]) {
    const double* sp = ((cc & 4) ? s1 : s0) + ((cc >> 1) & 1) * NC * 33 + (cc & 1);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      x[d] = sp[d * 33];
      u[d] = sp[(3 + d) * 33];
      ph[d] = KIND ? sp[(6 + d) * 33] : 0.0;
    }
  };
  auto node = [&](int cc, Nd& n) {
    double x[3], u[3], ph[3];
    ldc(cc, x, u, ph);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      n.e[d] = x[d] - x0[d];
      n.du[d] = u[d] - u0[d];
      n.dp[d] = KIND ? ph[d] - p0[d] : 0.0;
    }
  };
  Nd n7;
  ldc(0, x0, u0, p0);
  node(7, n7);
#pragma unroll
  for (int d = 0; d < 3; ++d) u05[d] = 5.0 * u0[d] + n7.du[d];  // 5 u_0 + (u_7 - u_0): shared by every tet's U + u_0
  auto acc = [&](int cc, int k, double v) {
    if (cc & 4) top[cc & 3][k] -= v;
    else bot[cc & 3][k] -= v;
  };
  // one tet: local nodes 1..3 = (na, nb, nc) at corners (ca, cb, cc); the two
  // that are not corner 7 are (p, q) in local order
  auto tet = [&](const double (&A)[3][3], double det, const Nd& na, const Nd& nb, const Nd& nc, const Nd& np,
                 const Nd& nq, int ca, int cb, int cc) {
    double du[3][3], w0[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      du[0][d] = na.du[d];
      du[1][d] = nb.du[d];
      du[2][d] = nc.du[d];
      w0[d] = u05[d] + (np.du[d] + nq.du[d]);
    }
    auto sub = [&](int a, int k, double v) { acc(a == 0 ? 0 : a == 1 ? ca : a == 2 ? cb : cc, k, v); };
    if constexpr (KIND) {
      double dp[3][3];
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        dp[f][0] = na.dp[f];
        dp[f][1] = nb.dp[f];
        dp[f][2] = nc.dp[f];
      }
      tet_s3_core(A, det, du, dp, w0, r, kW, sub);
    } else {
      tet_mom_core(A, det, du, w0, r, muW, sub);
    }
  };
  Nd n1, n3;
  double c71[3], c75[3], c74[3], c76[3], c72[3];
  node(1, n1);
  node(3, n3);
  {  // T0 (0, 1, 3, 7): E = (e1, e3, e7)
    double A[3][3];
    cross3(n3.e, n7.e, A[0]);
    cross3(n7.e, n1.e, A[1]);
    cross3(n1.e, n3.e, A[2]);
#pragma unroll
    for (int d = 0; d < 3; ++d) c71[d] = A[1][d];
    tet(A, dot3(n1.e, A[0]), n1, n3, n7, n1, n3, 1, 3, 7);
  }
  FPB_KMOM_TETBAR();
  Nd n5;
  node(5, n5);
  {  // T3 (0, 1, 7, 5): E = (e1, e7, e5)
    double A[3][3];
    cross3(n7.e, n5.e, A[0]);
    cross3(n5.e, n1.e, A[1]);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      c75[d] = A[0][d];
      A[2][d] = -c71[d];
    }
    tet(A, dot3(n1.e, A[0]), n1, n7, n5, n1, n5, 1, 7, 5);
  }
  FPB_KMOM_TETBAR();
  Nd n4;
  node(4, n4);
  {  // T2 (0, 4, 5, 7): E = (e4, e5, e7)
    double A[3][3];
    cross3(n7.e, n4.e, A[1]);
    cross3(n4.e, n5.e, A[2]);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      A[0][d] = -c75[d];
      c74[d] = A[1][d];
    }
    tet(A, dot3(n4.e, A[0]), n4, n5, n7, n4, n5, 4, 5, 7);
  }
  FPB_KMOM_TETBAR();
  Nd n6;
  node(6, n6);
  {  // T4 (0, 4, 7, 6): E = (e4, e7, e6)
    double A[3][3];
    cross3(n7.e, n6.e, A[0]);
    cross3(n6.e, n4.e, A[1]);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      c76[d] = A[0][d];
      A[2][d] = -c74[d];
    }
    tet(A, dot3(n4.e, A[0]), n4, n7, n6, n4, n6, 4, 7, 6);
  }
  FPB_KMOM_TETBAR();
  Nd n2;
  node(2, n2);
  {  // T1 (0, 2, 6, 7): E = (e2, e6, e7)
    double A[3][3];
    cross3(n7.e, n2.e, A[1]);
    cross3(n2.e, n6.e, A[2]);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      A[0][d] = -c76[d];
      c72[d] = A[1][d];
    }
    tet(A, dot3(n2.e, A[0]), n2, n6, n7, n2, n6, 2, 6, 7);
  }
  FPB_KMOM_TETBAR();
  node(3, n3);  // reloaded (not held across the cell)
  {  // T5 (0, 2, 7, 3): E = (e2, e7, e3)
    double A[3][3];
    cross3(n7.e, n3.e, A[0]);
    cross3(n3.e, n2.e, A[1]);
#pragma unroll
    for (int d = 0; d < 3; ++d) A[2][d] = -c72[d];
    tet(A, dot3(n2.e, A[0]), n2, n7, n3, n2, n3, 2, 7, 3);
  }
}

// Register cap of the TET04 momentum kind: 184 leaves room next to the 8 momentum
// warps (47 K registers, 114 KB of shared memory) for two one-warp CTAs of
// the B_xyz lines kernel, so the two-stream NS step overlaps them from the
// start (C5 step 2.808 -> 2.786 ms; momentum alone unchanged: 1.56 ms, no
// spills; 176 measured 1.66 ms).  The other kinds keep 255 (the three-scalar
// tet kind would spill at 184).  One 8-warp CTA per SM either way (2 CTAs
// at 128 registers: spills, 13 % slower).
#ifndef FPB_KMOM_MAXNREG
#define FPB_KMOM_MAXNREG 184
#endif
template <int MAXT, int KIND>
__global__ void __maxnreg__(KIND == 0 ? FPB_KMOM_MAXNREG : 255)
k_kuhn_mom(KuhnGrid g, int kchunk, const double* __restrict__ xyz4, const double* __restrict__ vel,
           const double* __restrict__ phi, int64_t fstride, double rho, double mu, double kappa,
           double* __restrict__ part, double* __restrict__ out) {
  constexpr int NC = kmom_nc<KIND>(), kKmomStg = kmom_stg<KIND>(), kKmomWarpD = kmom_warp_d<KIND>();
  // output slot of (node, component): [n][3] (momentum) or [3][fstride] (scalars)
  auto oi = [&](int64_t nd, int d) -> int64_t { return (KIND & 1) ? d * fstride + nd : 3 * nd + d; };
  extern __shared__ __align__(16) double sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int a = blockIdx.x, b = blockIdx.y, c = blockIdx.z;
  const int i0 = 32 * a, j0 = kKmomTY * b;
  const int tyb = min(kKmomTY, ny - j0);  // cell rows of this CTA
  double* const stg = sm + (size_t)w * kKmomWarpD;
  volatile double* const ring = stg + kKmomStg;                                   // my top rows [slot][33][3]
  volatile double* const dring = sm + (size_t)(w - 1) * kKmomWarpD + kKmomStg;  // the warp below's
  double* const hold = stg + kKmomStg + kKmomRing * kKmomSlot;                   // lane-private
  volatile int* const yc = reinterpret_cast<volatile int*>(sm + (size_t)kKmomTY * kKmomWarpD);  // [TY][2]
  const double r = ((KIND & 1) ? 1.0 : rho) * c_ref[FPB_TET04].M[1];  // M[0][1] = W / 20
  const double muW = mu * c_ref[FPB_TET04].W;
  const double kW[3] = {rho * c_ref[FPB_TET04].W, muW, kappa * c_ref[FPB_TET04].W};  // scalars: kappa_f W
  if (threadIdx.x < 2 * kKmomTY) yc[threadIdx.x] = 0;
  __syncthreads();
  if (w >= tyb) return;  // no barrier below
  const int j = j0 + w;
  const int nchunk = (g.kc1 - g.kc0 + kchunk - 1) / kchunk;
  const int kb = g.kc0 + c * kchunk, ke = min(g.kc1, kb + kchunk);
  const int kfirst = c > 0 ? kb - 1 : kb;               // halo cell layer below the chunk
  const int klast = c == nchunk - 1 ? g.kc1 : ke - 1;   // last node layer written (kc1: the top face)
  const int64_t row = nx + 1, layer = (int64_t)(nx + 1) * (ny + 1);
  const bool cell = i0 + lane < nx;
  const bool last_x = i0 + 32 >= nx;
  const bool node = i0 + lane <= nx;                 // my node column i0 + lane is written here
  const bool xtra = i0 + 32 == nx && lane == 31;     // also owns node column nx
  const bool redge = lane == 31 && !last_x;          // right edge -> the next x-block (Px)
  const bool top_w = w == tyb - 1;                   // my top node row leaves the CTA
  const bool top_final = top_w && j + 1 == ny;

  auto stage = [&](int kl) {  // node layer kl, node rows j, j + 1, columns i0 .. i0 + 32
    double* s = stg + (kl % 3) * 2 * NC * 33;
    for (int q = lane; q < 33; q += 32) {
      const int ii = i0 + q;
      if (ii <= nx) {
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
          const int64_t nd = ii + (j + dj) * row + kl * layer;
          double* t = s + dj * NC * 33 + q;
          cp8(t, xyz4 + 4 * nd);
          cp8(t + 33, xyz4 + 4 * nd + 1);
          cp8(t + 66, xyz4 + 4 * nd + 2);
          cp8(t + 99, vel + 3 * nd);
          cp8(t + 132, vel + 3 * nd + 1);
          cp8(t + 165, vel + 3 * nd + 2);
          if constexpr (KIND & 1) {
#pragma unroll
            for (int f = 0; f < 3; ++f) cp8(t + (6 + f) * 33, phi + f * fstride + nd);
          }
        }
      }
    }
    cp_commit();
  };

  stage(kfirst);
  stage(kfirst + 1);
  double bot[4][3];  // corners dk = 0, index di + 2 dj
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int d = 0; d < 3; ++d) bot[q][d] = 0.0;
  for (int t = kfirst; t <= klast + 2; ++t) {
    // (C) node row j of layer t - 2 (held in smem since (B), so the warp
    // below had a whole iteration to forward it): add its top row, write out
    if (t - 2 >= kb) {
      const int kk = t - 2;
      double R[3], X[3];  // my column; column i0 + 32 (lane 31)
      const double* h = hold + (kk & 1) * 99;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        R[d] = h[d * 33 + lane];
        X[d] = h[d * 33 + 32];
      }
      if (w > 0) {
        // flag protocol (CTA scope, shared memory): the producer's slot
        // stores, __syncwarp, then lane 0's st.release of the full count; here
        // lane 0's ld.acquire of it, __syncwarp, then the slot loads; the
        // consumed count is released after them (and acquired by the
        // producer before it reuses the slot).  compute-sanitizer racecheck
        // does not model flag synchronisation and lists these slot accesses
        // as hazards (profiles/r02m_sanitizer).
        if (lane == 0)
          while (yc_acquire(yc + 2 * (w - 1)) < kk - kb + 1) __nanosleep(20);
        __syncwarp();
        const volatile double* e = dring + (kk % kKmomRing) * kKmomSlot;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          R[d] += e[lane * 3 + d];
          if (lane == 31) X[d] += e[32 * 3 + d];
        }
        __syncwarp();
        if (lane == 0) yc_release(yc + 2 * (w - 1) + 1, kk - kb + 1);  // consumed
      }
      const int64_t nd = i0 + lane + j * row + (int64_t)kk * layer;
      if (node) {
#pragma unroll
        for (int d = 0; d < 3; ++d) out[oi(nd, d)] = R[d];
      }
      if (xtra) {
#pragma unroll
        for (int d = 0; d < 3; ++d) out[oi(nd + 1, d)] = X[d];
      } else if (redge) {
#pragma unroll
        for (int d = 0; d < 3; ++d) part[g.px(a, b, kk, w) + d] = X[d];
      }
    }
    if (t > klast) continue;
    // (A) cell layer t
    __syncwarp();
    if (t + 2 <= ke) stage(t + 2);
    else cp_commit();
    cp_wait_1();
    __syncwarp();
    double top[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int d = 0; d < 3; ++d) top[q][d] = 0.0;
    if (cell && t < ke) {
      const double* s0 = stg + (t % 3) * 2 * NC * 33 + lane;
      const double* s1 = stg + ((t + 1) % 3) * 2 * NC * 33 + lane;
      if constexpr (KIND >= 2) {  // one Q1 hex per cell: local node b at corner c = {0,1,3,2,4,5,7,6}[b]
        constexpr int HK = KIND == 2 ? FPB_MOMENTUM_RHS : KIND_SCALAR3;
        double xe[8][3], ue[8][3], fe[Out<FPB_HEX08, HK>::NF], ae[Out<FPB_HEX08, HK>::NOUT];
#pragma unroll
        for (int bb = 0; bb < 8; ++bb) {
          const int cc = bb ^ ((bb >> 1) & 1);
          const double* sp = ((cc & 4) ? s1 : s0) + ((cc >> 1) & 1) * NC * 33 + (cc & 1);
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            xe[bb][d] = sp[d * 33];
            ue[bb][d] = sp[(3 + d) * 33];
            if constexpr (KIND == 3) fe[d * 8 + bb] = sp[(6 + d) * 33];
          }
        }
        if constexpr (KIND == 2) fe[0] = 0.0;
        hex_rhs_integrate<HK>(xe, ue, fe, rho, mu, kappa, ae);
#pragma unroll
        for (int bb = 0; bb < 8; ++bb) {
          const int cc = bb ^ ((bb >> 1) & 1);
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            if (cc & 4) top[cc & 3][d] += ae[bb * 3 + d];
            else bot[cc & 3][d] += ae[bb * 3 + d];
          }
        }
      } else if constexpr (KIND && FPB_KMOM_S3_SHARED) {  // three scalars, shared-node cell cycle
        kuhn_cell_shared<1>(s0, s1, r, muW, kW, bot, top);
      } else if constexpr (KIND) {  // three scalars: tet by tet
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) {
          asm volatile("" ::: "memory");  // one tet's node loads at a time (register pressure)
          double xe[4][3], ue[4][3], pe[3][4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int cc = kuhn_corner(tt, q);
            const double* sp = ((cc & 4) ? s1 : s0) + ((cc >> 1) & 1) * NC * 33 + (cc & 1);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              xe[q][d] = sp[d * 33];
              ue[q][d] = sp[(3 + d) * 33];
              pe[d][q] = sp[(6 + d) * 33];
            }
          }
          tet_s3_adj(xe, ue, pe, r, kW, [&](int q, int f, double v) {
            const int cc = kuhn_corner(tt, q);
            if (cc & 4) top[cc & 3][f] -= v;
            else bot[cc & 3][f] -= v;
          });
        }
      } else {
#if FPB_KMOM_SHARED
        kuhn_cell_shared<0>(s0, s1, r, muW, kW, bot, top);
#else
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) {
          asm volatile("" ::: "memory");  // one tet's node loads at a time (register pressure)
          double xe[4][3], ue[4][3];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int cc = kuhn_corner(tt, q);
            const double* sp = ((cc & 4) ? s1 : s0) + ((cc >> 1) & 1) * NC * 33 + (cc & 1);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              xe[q][d] = sp[d * 33];
              ue[q][d] = sp[(3 + d) * 33];
            }
          }
          tet_mom_adj_f(xe, ue, r, muW, [&](int q, int d, double v) {
            const int cc = kuhn_corner(tt, q);
            if (cc & 4) top[cc & 3][d] -= v;
            else bot[cc & 3][d] -= v;
          });
        }
#endif
      }
    }
    // (B) layer t's bottom face is complete in z: x-shuffle; the right edge
    // and the top node row leave the warp
    if (t >= kb) {
      double up[3], ex1[3];  // row j + 1 at my column; right edge of row j + 1 (lane 31)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double l0 = __shfl_up_sync(0xffffffffu, bot[1][d], 1);
        const double l1 = __shfl_up_sync(0xffffffffu, bot[3][d], 1);
        double* h = hold + (t & 1) * 99;
        h[d * 33 + lane] = lane > 0 ? bot[0][d] + l0 : bot[0][d];
        if (lane == 31) h[d * 33 + 32] = bot[1][d];
        up[d] = lane > 0 ? bot[2][d] + l1 : bot[2][d];
        ex1[d] = bot[3][d];
      }
      if (top_w) {  // row j + 1 leaves the CTA: final (top of the mesh) or Py / Px partials
        const int64_t nd1 = i0 + lane + (j + 1) * row + (int64_t)t * layer;
        if (top_final) {
          if (node) {
#pragma unroll
            for (int d = 0; d < 3; ++d) out[oi(nd1, d)] = up[d];
          }
          if (xtra) {
#pragma unroll
            for (int d = 0; d < 3; ++d) out[oi(nd1 + 1, d)] = ex1[d];
          }
        } else {
          if (node) {
#pragma unroll
            for (int d = 0; d < 3; ++d) part[g.py(a, b, t, lane) + d] = up[d];
          }
          if (xtra) {
#pragma unroll
            for (int d = 0; d < 3; ++d) part[g.py(a, b, t, 32) + d] = ex1[d];
          }
        }
        if (redge) {
#pragma unroll
          for (int d = 0; d < 3; ++d) part[g.px(a, b, t, tyb) + d] = ex1[d];
        }
      } else {  // to the warp above
        if (lane == 0)
          while (yc_acquire(yc + 2 * w + 1) < (t - kb + 1) - kKmomRing) __nanosleep(20);  // slot free
        __syncwarp();
        volatile double* slot = ring + (t % kKmomRing) * kKmomSlot;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          slot[lane * 3 + d] = up[d];
          if (lane == 31) slot[32 * 3 + d] = ex1[d];
        }
        __syncwarp();  // orders the warp's slot stores before lane 0's release
        if (lane == 0) yc_release(yc + 2 * w, t - kb + 1);  // full
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int d = 0; d < 3; ++d) bot[q][d] = top[q][d];
  }
  cp_wait_all();
}

// Boundary nodes: x-block edges (columns 32 a, 0 < a < nxb) over every node
// row, then y-block edges (rows TY b, 0 < b < nyb) over the other columns.
// out += Px(a - 1, b)[lr] (+ Py(a, b - 1)[0] + Px(a - 1, b - 1)[TY] at a
// y-block edge), resp. out += Py(a, b - 1)[l] — a fixed order per node.
__global__ void k_kuhn_fixup(KuhnGrid g, const double* __restrict__ part, double* __restrict__ out, int64_t fstride) {
  auto oi = [&](int64_t nd, int d) -> int64_t { return fstride ? d * fstride + nd : 3 * nd + d; };
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int64_t row = nx + 1, layer = (int64_t)(nx + 1) * (ny + 1);
  const int64_t nxe = (int64_t)(g.nxb - 1) * (ny + 1);                // x-edge nodes per layer
  const int64_t cols = nx + 1 - (g.nxb - 1);                          // columns that are not x-edges
  const int64_t per = nxe + (int64_t)(g.nyb - 1) * cols;
  const int64_t total = per * (g.kc1 - g.kc0 + 1);  // node layers kc0 .. kc1
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kq = q / per;
    int64_t u = q - kq * per;
    const int k = g.kc0 + (int)kq;
    if (u < nxe) {
      const int a = 1 + (int)(u / (ny + 1));
      const int jn = (int)(u - (int64_t)(a - 1) * (ny + 1));
      const int b = min(jn / kKmomTY, g.nyb - 1);
      const int lr = jn - kKmomTY * b;
      const int64_t nd = 32 * a + jn * row + (int64_t)k * layer;
      double s[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) s[d] = out[oi(nd, d)] + part[g.px(a - 1, b, k, lr) + d];
      if (lr == 0 && b > 0) {
#pragma unroll
        for (int d = 0; d < 3; ++d)
          s[d] = (s[d] + part[g.py(a, b - 1, k, 0) + d]) + part[g.px(a - 1, b - 1, k, kKmomTY) + d];
      }
#pragma unroll
      for (int d = 0; d < 3; ++d) out[oi(nd, d)] = s[d];
    } else {
      u -= nxe;
      const int b = 1 + (int)(u / cols);
      const int m = (int)(u - (int64_t)(b - 1) * cols);  // m-th column that is not an x-edge
      const int i = m < 32 ? m : m + min((m - 32) / 31 + 1, g.nxb - 1);
      const int a = min(i / 32, g.nxb - 1);
      const int64_t nd = i + (int64_t)(kKmomTY * b) * row + (int64_t)k * layer;
#pragma unroll
      for (int d = 0; d < 3; ++d) out[oi(nd, d)] = out[oi(nd, d)] + part[g.py(a, b - 1, k, i - 32 * a) + d];
    }
  }
}

int g_tuning_kmom_smem_kb = 0;  // fpb_set_tuning("kmom_smem_kb", KB): pad the CTA's shared memory (co-residency A/B)

template <int KIND>
inline size_t kmom_smem() { return (size_t)kKmomTY * kmom_warp_d<KIND>() * sizeof(double) + 2 * kKmomTY * sizeof(int); }

inline KuhnGrid kuhn_grid(int nx, int ny, int nz, int kc0 = 0, int kc1 = -1) {
  KuhnGrid g;
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  g.kc0 = kc0;
  g.kc1 = kc1 < 0 ? nz : kc1;
  g.nxb = (nx + 31) / 32;
  g.nyb = (ny + kKmomTY - 1) / kKmomTY;
  return g;
}

template <int KIND>
static int launch_kuhn(int nx, int ny, int nz, int kc0, int kc1, int kchunk, const double* xyz4, const double* vel,
                       const double* phi, int64_t fstride, double rho, double mu, double kappa, double* scratch,
                       double* out, cudaStream_t s) {
  const KuhnGrid g = kuhn_grid(nx, ny, nz, kc0, kc1);
  const int64_t plane = (int64_t)(nx + 1) * (ny + 1);
  // node planes no integrated cell touches (a slab's ghost planes) are zero
  const int64_t lo = plane * kc0, hi = plane * (kc1 + 1), n = plane * (nz + 1);
  if (KIND & 1) {
    for (int f = 0; f < 3; ++f) {
      if (lo > 0) FPB_CUDA(cudaMemsetAsync(out + f * fstride, 0, sizeof(double) * lo, s));
      if (hi < n) FPB_CUDA(cudaMemsetAsync(out + f * fstride + hi, 0, sizeof(double) * (n - hi), s));
    }
  } else {
    if (lo > 0) FPB_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 3 * lo, s));
    if (hi < n) FPB_CUDA(cudaMemsetAsync(out + 3 * hi, 0, sizeof(double) * 3 * (n - hi), s));
  }
  const int nchunk = (kc1 - kc0 + kchunk - 1) / kchunk;
  FPB_REQUIRE(g.nyb <= 65535 && nchunk <= 65535, "grid too large");
  const size_t smem = std::max(kmom_smem<KIND>(), (size_t)g_tuning_kmom_smem_kb * 1024);
  auto kern = k_kuhn_mom<32 * kKmomTY, KIND>;
  FPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<dim3(g.nxb, g.nyb, nchunk), 32 * kKmomTY, smem, s>>>(g, kchunk, xyz4, vel, phi, fstride, rho, mu, kappa,
                                                               scratch, out);
  FPB_LAUNCH_CHECK();
  const int64_t nb = ((int64_t)(g.nxb - 1) * (ny + 1) + (int64_t)(g.nyb - 1) * (nx + 1 - (g.nxb - 1))) * (kc1 - kc0 + 1);
  if (nb > 0) {
    k_kuhn_fixup<<<grid_for(nb, 256), 256, 0, s>>>(g, scratch, out, (KIND & 1) ? fstride : 0);
    FPB_LAUNCH_CHECK();
  }
  return FPB_OK;
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int64_t fpb_kuhn_mom_scratch_len(int nx, int ny, int nz) {
  if (nx < 1 || ny < 1 || nz < 1) return 0;
  return kuhn_grid(nx, ny, nz).scratch();
}

int fpb_assemble_momentum_kuhn(int nx, int ny, int nz, int kc0, int kc1, int kchunk, const double* xyz4,
                               const double* vel, double rho, double mu, double* scratch, double* out,
                               void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  FPB_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "Kuhn box %d x %d x %d", nx, ny, nz);
  FPB_REQUIRE(0 <= kc0 && kc0 < kc1 && kc1 <= nz, "cell layers [%d, %d) outside [0, %d)", kc0, kc1, nz);
  FPB_REQUIRE(kchunk >= 1, "bad z chunk %d", kchunk);
  FPB_REQUIRE(xyz4 && vel && scratch && out, "null argument");
  return launch_kuhn<0>(nx, ny, nz, kc0, kc1, kchunk, xyz4, vel, nullptr, 0, rho, mu, 0.0, scratch, out,
                        as_stream(stream));
}

int fpb_assemble_scalar3_kuhn(int nx, int ny, int nz, int kc0, int kc1, int kchunk, const double* xyz4,
                              const double* vel, const double* phi3, int64_t fstride, double kappa0, double kappa1,
                              double kappa2, double* scratch, double* out3, void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_TET04], "reference tables for TET04 not uploaded");
  FPB_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "Kuhn box %d x %d x %d", nx, ny, nz);
  FPB_REQUIRE(0 <= kc0 && kc0 < kc1 && kc1 <= nz, "cell layers [%d, %d) outside [0, %d)", kc0, kc1, nz);
  FPB_REQUIRE(kchunk >= 1, "bad z chunk %d", kchunk);
  FPB_REQUIRE(xyz4 && vel && phi3 && scratch && out3, "null argument");
  FPB_REQUIRE(fstride >= (int64_t)(nx + 1) * (ny + 1) * (nz + 1), "field stride %lld below the node count",
              (long long)fstride);
  return launch_kuhn<1>(nx, ny, nz, kc0, kc1, kchunk, xyz4, vel, phi3, fstride, kappa0, kappa1, kappa2, scratch,
                        out3, as_stream(stream));
}

int fpb_assemble_rhs_hexbox(int kind, int nx, int ny, int nz, int kc0, int kc1, int kchunk, const double* xyz4,
                            const double* vel, const double* phi3, int64_t fstride, double rho, double mu,
                            double kappa, double* scratch, double* out, void* stream) {
  FPB_REQUIRE(g_ref_loaded[FPB_HEX08], "reference tables for HEX08 not uploaded");
  FPB_REQUIRE(kind == FPB_MOMENTUM_RHS || kind == KIND_SCALAR3, "hex box RHS: MOMENTUM_RHS or the three scalars");
  FPB_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "hex box %d x %d x %d", nx, ny, nz);
  FPB_REQUIRE(0 <= kc0 && kc0 < kc1 && kc1 <= nz, "cell layers [%d, %d) outside [0, %d)", kc0, kc1, nz);
  FPB_REQUIRE(kchunk >= 1, "bad z chunk %d", kchunk);
  FPB_REQUIRE(xyz4 && vel && scratch && out && (kind == FPB_MOMENTUM_RHS || phi3), "null argument");
  if (kind == FPB_MOMENTUM_RHS)
    return launch_kuhn<2>(nx, ny, nz, kc0, kc1, kchunk, xyz4, vel, nullptr, 0, rho, mu, 0.0, scratch, out,
                          as_stream(stream));
  FPB_REQUIRE(fstride >= (int64_t)(nx + 1) * (ny + 1) * (nz + 1), "field stride below the node count");
  return launch_kuhn<3>(nx, ny, nz, kc0, kc1, kchunk, xyz4, vel, phi3, fstride, rho, mu, kappa, scratch, out,
                        as_stream(stream));
}

}  // extern "C"
