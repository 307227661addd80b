// Setup path: reference tables, synthetic box meshes, lane packs, the CSR
// node graph, the element->CSR map and packed geometry.  Every routine is
// bit-exact with the reference routine it cites (checked by
// tests/test_gpu_setup.py against tests/golden and the oracle).
#include <cub/device/device_scan.cuh>

#include <climits>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace fpb {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

__constant__ RefTables c_ref[5];
bool g_ref_loaded[5] = {false, false, false, false, false};

// ---------------------------------------------------------------------------
// grid coordinates: np.linspace(0, L, n+1)[i] == i * (L / n), last == L
// (numpy linspace: y = arange * step + start; y[-1] = stop), i fastest
// (mesh.py:158-187).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double lin(int i, int n, double L) {
  if (i == n) return L;
  double step = L / (double)n;
  return (double)i * step + 0.0;
}

// nz: global cell count along z; planes k0 .. k0 + nplanes - 1 are generated
// (slab of a larger grid, for z-slab domain decomposition)
__global__ void k_grid3(int nx, int ny, int nz, int k0, int nplanes, double lx, double ly, double lz,
                        double* coords) {
  int64_t total = (int64_t)(nx + 1) * (ny + 1) * nplanes;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t % (nx + 1));
    int64_t r = t / (nx + 1);
    int j = (int)(r % (ny + 1));
    int k = (int)(r / (ny + 1)) + k0;
    coords[3 * t + 0] = lin(i, nx, lx);
    coords[3 * t + 1] = lin(j, ny, ly);
    coords[3 * t + 2] = lin(k, nz, lz);
  }
}

__global__ void k_grid2(int nx, int ny, double lx, double ly, double* coords) {
  int64_t total = (int64_t)(nx + 1) * (ny + 1);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t % (nx + 1));
    int j = (int)(t / (nx + 1));
    coords[2 * t + 0] = lin(i, nx, lx);
    coords[2 * t + 1] = lin(j, ny, ly);
  }
}

// hex corner offsets (mesh.py:190-199)
__constant__ int c_hex_corner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                       {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
// pyramid bases seen from the cell centre (mesh.py:202-209)
__constant__ int c_hex_inward[6][4] = {{0, 1, 2, 3}, {4, 7, 6, 5}, {0, 4, 5, 1},
                                       {2, 6, 7, 3}, {0, 3, 7, 4}, {1, 5, 6, 2}};
// Kuhn permutations; the odd ones swap the last two nodes (mesh.py:212-213, :268-282)
__constant__ int c_kuhn[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 2}, {2, 1}, {1, 0}};

__device__ __forceinline__ int nid3(int i, int j, int k, int nx, int ny) {
  return i + (nx + 1) * (j + (ny + 1) * k);
}

// one thread per cell, cells k-major / i fastest (mesh.py:220-224)
__global__ void k_box3(int etype, int nx, int ny, int nz, int32_t* conn) {
  int64_t ncell = (int64_t)nx * ny * nz;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
       c += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(c % nx);
    int64_t r = c / nx;
    int j = (int)(r % ny);
    int k = (int)(r / ny);
    if (etype == FPB_HEX08) {
#pragma unroll
      for (int a = 0; a < 8; ++a)
        conn[c * 8 + a] = nid3(i + c_hex_corner[a][0], j + c_hex_corner[a][1], k + c_hex_corner[a][2], nx, ny);
    } else {  // TET04
      int v7 = nid3(i + 1, j + 1, k + 1, nx, ny);
      int v0 = nid3(i, j, k, nx, ny);
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        int p[3] = {i, j, k};
        p[c_kuhn[t][0]] += 1;
        int v1 = nid3(p[0], p[1], p[2], nx, ny);
        p[c_kuhn[t][1]] += 1;
        int v2 = nid3(p[0], p[1], p[2], nx, ny);
        int32_t* o = conn + (c * 6 + t) * 4;
        o[0] = v0;
        o[1] = v1;
        if (t >= 3) {
          o[2] = v7;
          o[3] = v2;
        } else {
          o[2] = v2;
          o[3] = v7;
        }
      }
    }
  }
}

__global__ void k_box2(int etype, int nx, int ny, int32_t* conn) {
  int64_t ncell = (int64_t)nx * ny;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
       c += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(c % nx), j = (int)(c / nx);
    int v0 = i + (nx + 1) * j, v1 = i + 1 + (nx + 1) * j;
    int v2 = i + 1 + (nx + 1) * (j + 1), v3 = i + (nx + 1) * (j + 1);
    if (etype == FPB_QUAD04) {
      conn[c * 4 + 0] = v0; conn[c * 4 + 1] = v1; conn[c * 4 + 2] = v2; conn[c * 4 + 3] = v3;
    } else {  // TRI03, mesh.py:252-254
      conn[c * 6 + 0] = v0; conn[c * 6 + 1] = v1; conn[c * 6 + 2] = v2;
      conn[c * 6 + 3] = v0; conn[c * 6 + 4] = v2; conn[c * 6 + 5] = v3;
    }
  }
}

// mixed mesh (mesh.py:292-336); pyramid cells are i < nlayers, numbered in
// cell order; centre = sequential sum of the 8 corners / 8 (ndarray.mean).
__global__ void k_mixed(int nx, int ny, int nz, int nlayers, double* coords, int32_t* pyr,
                        int32_t* hex) {
  int64_t ncell = (int64_t)nx * ny * nz;
  int64_t ngrid = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
       c += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(c % nx);
    int64_t r = c / nx;  // = k*ny + j
    int cell[8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
      cell[a] = nid3(i + c_hex_corner[a][0], (int)(r % ny) + c_hex_corner[a][1],
                     (int)(r / ny) + c_hex_corner[a][2], nx, ny);
    if (i < nlayers) {
      int64_t pc = r * nlayers + i;
      int64_t cid = ngrid + pc;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double s = coords[3 * (int64_t)cell[0] + d];
#pragma unroll
        for (int a = 1; a < 8; ++a) s += coords[3 * (int64_t)cell[a] + d];
        coords[3 * cid + d] = s / 8.0;
      }
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        int32_t* o = pyr + (pc * 6 + f) * 5;
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = cell[c_hex_inward[f][q]];
        o[4] = (int32_t)cid;
      }
    } else {
      int64_t hc = r * (nx - nlayers) + (i - nlayers);
#pragma unroll
      for (int a = 0; a < 8; ++a) hex[hc * 8 + a] = cell[a];
    }
  }
}

// lane packs (packing.py:104-115)
__global__ void k_packs(int64_t nelem, int nn, int vs, const int32_t* conn, int32_t* lane_conn) {
  int64_t npacks = (nelem + vs - 1) / vs;
  int64_t total = npacks * nn * vs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int v = (int)(t % vs);
    int64_t r = t / vs;
    int a = (int)(r % nn);
    int64_t p = r / nn;
    int64_t e = p * vs + v;
    if (e >= nelem) e = nelem - 1;
    lane_conn[t] = conn[e * nn + a];
  }
}

// ---------------------------------------------------------------------------
// CSR node graph.  The reference forms np.unique over all element node-pair
// keys plus the diagonal (sparse.py:59-75); the resulting sorted set is
// unique, so any exact algorithm reproduces it bit for bit.  Here: a node ->
// element incidence list (counting sort), then one warp per row selects the
// ascending distinct neighbours with warp-wide min reductions.
// ---------------------------------------------------------------------------
struct Groups {
  const int32_t* conn[8];
  int64_t start[9];  // global element offset of each group; start[ng] = total
  int nn[8];
  int ng;
};

__global__ void k_incidence_count(Groups G, int32_t* cnt) {
  for (int g = 0; g < G.ng; ++g) {
    int64_t total = (G.start[g + 1] - G.start[g]) * G.nn[g];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x)
      atomicAdd(&cnt[G.conn[g][t]], 1);
  }
}

__global__ void k_incidence_fill(Groups G, const int64_t* ptr, int32_t* cursor, int32_t* inc) {
  for (int g = 0; g < G.ng; ++g) {
    int nn = G.nn[g];
    int64_t total = (G.start[g + 1] - G.start[g]) * nn;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
      int node = G.conn[g][t];
      int slot = atomicAdd(&cursor[node], 1);
      inc[ptr[node] + slot] = (int32_t)(G.start[g] + t / nn);
    }
  }
}

__device__ __forceinline__ void elem_lookup(const Groups& G, int32_t geid, const int32_t*& c, int& nn) {
  int g = 0;
  while (g + 1 < G.ng && geid >= G.start[g + 1]) ++g;
  nn = G.nn[g];
  c = G.conn[g] + (int64_t)(geid - G.start[g]) * nn;
}

// pass 0: rowlen[i]; pass 1: colind[rowptr[i] ...]
__global__ void k_pattern_rows(Groups G, int32_t n, const int64_t* ptr, const int32_t* inc,
                               int pass, int32_t* rowlen, const int32_t* rowptr, int32_t* colind) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
    const int64_t lo = ptr[row], hi = ptr[row + 1];
    int last = -1, count = 0;
    while (true) {
      int mine = INT_MAX;
      if (lane == 0 && (int)row > last) mine = (int)row;  // the diagonal is always present
      for (int64_t k = lo + lane; k < hi; k += 32) {
        const int32_t* c;
        int nn;
        elem_lookup(G, inc[k], c, nn);
        for (int a = 0; a < nn; ++a) {
          int v = c[a];
          if (v > last && v < mine) mine = v;
        }
      }
      int m = __reduce_min_sync(0xffffffffu, mine);
      if (m == INT_MAX) break;
      if (pass == 1 && lane == 0) colind[rowptr[row] + count] = m;
      ++count;
      last = m;
    }
    if (pass == 0 && lane == 0) rowlen[row] = count;
  }
}

// element->CSR position: binary search of conn[e][j] in row conn[e][i]
__global__ void k_positions(int64_t nelem, int nn, const int32_t* conn, int32_t n, const int32_t* rowptr,
                            const int32_t* colind, int layout, int vs, int32_t* pos, int* missing) {
  int64_t npacks = (nelem + vs - 1) / vs;
  int64_t total = layout == 0 ? nelem * nn * nn : npacks * nn * nn * vs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t e;
    int i, j;
    if (layout == 0) {
      j = (int)(t % nn);
      i = (int)((t / nn) % nn);
      e = t / ((int64_t)nn * nn);
    } else {
      int v = (int)(t % vs);
      int64_t r = t / vs;
      j = (int)(r % nn);
      r /= nn;
      i = (int)(r % nn);
      int64_t p = r / nn;
      e = p * vs + v;
      if (e >= nelem) e = nelem - 1;
    }
    int row = conn[e * nn + i], col = conn[e * nn + j];
    if (row < 0 || row >= n || col < 0 || col >= n) {  // node outside the pattern: a missing pair
      pos[t] = -1;
      atomicExch(missing, 1);
      continue;
    }
    int lo = rowptr[row], hi = rowptr[row + 1];
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (colind[mid] < col) lo = mid + 1; else hi = mid;
    }
    if (lo < rowptr[row + 1] && colind[lo] == col) {
      pos[t] = lo;
    } else {
      pos[t] = -1;
      atomicExch(missing, 1);
    }
  }
}

// packed geometry at pack width vs (_kernels.py:78-147)
template <int ET>
__global__ void k_geometry(int64_t nelem, int vs, const int32_t* conn, const double* coords,
                           double* detjw, double* gradn, unsigned long long* bad) {
  constexpr int NN = Elem<ET>::NN, NG = Elem<ET>::NG, DIM = Elem<ET>::DIM;
  int64_t npacks = (nelem + vs - 1) / vs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < npacks * vs;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = t / vs;
    int v = (int)(t % vs);
    bool active = t < nelem;
    int64_t e = active ? t : nelem - 1;
    double xe[NN][DIM];
#pragma unroll
    for (int a = 0; a < NN; ++a) {
      int node = conn[e * NN + a];
#pragma unroll
      for (int d = 0; d < DIM; ++d) xe[a][d] = coords[(int64_t)node * DIM + d];
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      double J[DIM][DIM];
      double det = jacobian<ET>(xe, g, J);
      if (active && det <= 0.0)
        atomicMin(bad, (unsigned long long)((p * NG + g) * vs + v));
      detjw[(p * NG + g) * vs + v] = active ? det * refW<ET>(g) : 0.0;
      if (gradn) {
        double gN[DIM][NN];
        grad_shape<ET>(J, det, g, gN);
#pragma unroll
        for (int d = 0; d < DIM; ++d)
#pragma unroll
          for (int a = 0; a < NN; ++a) gradn[(((p * DIM + d) * NN + a) * NG + g) * vs + v] = gN[d][a];
      }
    }
  }
}

}  // namespace fpb

using namespace fpb;

extern "C" {

const char* fpb_last_error(void) { return g_last_error.c_str(); }
int fpb_version(void) { return 1; }

int fpb_set_reference_element(int etype, int nn, int ng, int dim, const double* N_h,
                              const double* dN_h, const double* w_h) {
  FPB_REQUIRE(etype >= 0 && etype < 5, "bad element type %d", etype);
  FPB_REQUIRE(nn == etype_nn(etype) && ng == etype_ng(etype) && dim == etype_dim(etype),
              "table shape mismatch for element type %d", etype);
  RefTables t;
  memset(&t, 0, sizeof(t));
  memcpy(t.N, N_h, sizeof(double) * nn * ng);
  memcpy(t.dN, dN_h, sizeof(double) * dim * nn * ng);
  memcpy(t.w, w_h, sizeof(double) * ng);
  // derived tables, summed over Gauss points in the reference's order
  for (int a = 0; a < nn; ++a) {
    double m1 = 0.0;
    for (int b = 0; b < nn; ++b) {
      double acc = 0.0;
      for (int g = 0; g < ng; ++g) acc += w_h[g] * N_h[b * ng + g] * N_h[a * ng + g];
      t.M[a * nn + b] = acc;
    }
    for (int g = 0; g < ng; ++g) {
      double sN = 0.0;
      for (int c = 0; c < nn; ++c) sN += N_h[c * ng + g];
      m1 += w_h[g] * (sN * N_h[a * ng + g]);
    }
    t.mN[a] = m1;
  }
  t.W = 0.0;
  for (int g = 0; g < ng; ++g) t.W += w_h[g];
  FPB_CUDA(cudaMemcpyToSymbol(c_ref, &t, sizeof(t), sizeof(RefTables) * etype));
  g_ref_loaded[etype] = true;
  return FPB_OK;
}

int fpb_grid_coords(int dim, int nx, int ny, int nz, double lx, double ly, double lz,
                    double* coords, void* stream) {
  FPB_REQUIRE(nx >= 1 && ny >= 1 && (dim == 2 || nz >= 1), "cell counts must be at least 1");
  if (dim == 2) {
    int64_t total = (int64_t)(nx + 1) * (ny + 1);
    k_grid2<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(nx, ny, lx, ly, coords);
  } else {
    int64_t total = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
    FPB_REQUIRE(total < INT_MAX, "mesh too large for int32 node ids");
    k_grid3<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(nx, ny, nz, 0, nz + 1, lx, ly, lz, coords);
  }
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_grid_coords_slab(int nx, int ny, int nz, int k0, int nplanes, double lx, double ly, double lz,
                         double* coords, void* stream) {
  FPB_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "cell counts must be at least 1");
  FPB_REQUIRE(k0 >= 0 && nplanes >= 1 && k0 + nplanes <= nz + 1, "slab planes outside the grid");
  int64_t total = (int64_t)(nx + 1) * (ny + 1) * nplanes;
  FPB_REQUIRE(total < INT_MAX, "slab too large for int32 node ids");
  k_grid3<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(nx, ny, nz, k0, nplanes, lx, ly, lz, coords);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_box_conn(int etype, int nx, int ny, int nz, int32_t* conn, void* stream) {
  FPB_REQUIRE(nx >= 1 && ny >= 1, "cell counts must be at least 1");
  if (etype == FPB_TET04 || etype == FPB_HEX08) {
    FPB_REQUIRE(nz >= 1, "cell counts must be at least 1");
    int64_t ncell = (int64_t)nx * ny * nz;
    k_box3<<<grid_for(ncell, 256), 256, 0, as_stream(stream)>>>(etype, nx, ny, nz, conn);
  } else if (etype == FPB_TRI03 || etype == FPB_QUAD04) {
    int64_t ncell = (int64_t)nx * ny;
    k_box2<<<grid_for(ncell, 256), 256, 0, as_stream(stream)>>>(etype, nx, ny, conn);
  } else {
    FPB_REQUIRE(false, "no box generator for element type %d", etype);
  }
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_mixed_conn(int nx, int ny, int nz, int nlayers, double* coords, int32_t* pyr_conn,
                   int32_t* hex_conn, void* stream) {
  FPB_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "cell counts must be at least 1");
  FPB_REQUIRE(nlayers >= 0 && nlayers <= nx, "bad pyramid layer count");
  int64_t ncell = (int64_t)nx * ny * nz;
  k_mixed<<<grid_for(ncell, 256), 256, 0, as_stream(stream)>>>(nx, ny, nz, nlayers, coords,
                                                                pyr_conn, hex_conn);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_build_packs(int64_t nelem, int nn, int vs, const int32_t* conn, int32_t* lane_conn,
                    void* stream) {
  FPB_REQUIRE(vs == 1 || vs == 2 || vs == 4 || vs == 8 || vs == 16 || vs == 32,
              "vector_size must be one of (1, 2, 4, 8, 16, 32), got %d", vs);
  if (nelem == 0) return FPB_OK;
  int64_t total = (nelem + vs - 1) / vs * nn * vs;
  k_packs<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(nelem, nn, vs, conn, lane_conn);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_build_pattern(int32_t n, int ngroups, const int32_t* const* conns_h,
                      const int64_t* nelem_h, const int* nn_h, int32_t* rowptr, int32_t* colind,
                      int64_t* nnz_h, void* stream) {
  FPB_REQUIRE(ngroups >= 0 && ngroups <= 8, "too many element groups");
  FPB_REQUIRE(n >= 0, "bad node count");
  cudaStream_t s = as_stream(stream);
  Groups G;
  memset(&G, 0, sizeof(G));
  G.ng = ngroups;
  G.start[0] = 0;
  for (int g = 0; g < ngroups; ++g) {
    G.conn[g] = conns_h[g];
    G.nn[g] = nn_h[g];
    G.start[g + 1] = G.start[g] + nelem_h[g];
  }
  FPB_REQUIRE(G.start[ngroups] < INT_MAX, "too many elements for int32 ids");
  int64_t ninc = 0;
  for (int g = 0; g < ngroups; ++g) ninc += nelem_h[g] * nn_h[g];

  int32_t *cnt = nullptr, *inc = nullptr, *rowlen = nullptr;
  int64_t* ptr = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, tb2 = 0;
  FPB_CUDA(cudaMallocAsync(&cnt, sizeof(int32_t) * (n + 1), s));
  FPB_CUDA(cudaMallocAsync(&ptr, sizeof(int64_t) * (n + 1), s));
  FPB_CUDA(cudaMallocAsync(&inc, sizeof(int32_t) * (ninc > 0 ? ninc : 1), s));
  FPB_CUDA(cudaMallocAsync(&rowlen, sizeof(int32_t) * (n + 1), s));
  FPB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), s));
  FPB_CUDA(cudaMemsetAsync(rowlen, 0, sizeof(int32_t) * (n + 1), s));
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, ptr, n + 1, s);
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, rowlen, rowptr, n + 1, s);
  if (tb2 > tmp_bytes) tmp_bytes = tb2;
  FPB_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));

  if (ninc > 0) k_incidence_count<<<grid_for(ninc, 256), 256, 0, s>>>(G, cnt);
  FPB_LAUNCH_CHECK();
  FPB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, ptr, n + 1, s));
  FPB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), s));
  if (ninc > 0) k_incidence_fill<<<grid_for(ninc, 256), 256, 0, s>>>(G, ptr, cnt, inc);
  FPB_LAUNCH_CHECK();
  int rows_grid = grid_for((int64_t)n * 32, 256, 32);
  k_pattern_rows<<<rows_grid, 256, 0, s>>>(G, n, ptr, inc, 0, rowlen, nullptr, nullptr);
  FPB_LAUNCH_CHECK();
  // rowlen has n+1 entries with rowlen[n] = 0, so the exclusive scan's last
  // entry is the total: rowptr[n] = nnz.  nnz < 2^31 is checked below.
  FPB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, rowlen, rowptr, n + 1, s));
  int32_t nnz32 = 0;
  FPB_CUDA(cudaMemcpyAsync(&nnz32, rowptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FPB_CUDA(cudaStreamSynchronize(s));
  if (nnz32 < 0) {
    set_error("CSR pattern exceeds 2^31 entries");
    cudaFreeAsync(cnt, s); cudaFreeAsync(ptr, s); cudaFreeAsync(inc, s);
    cudaFreeAsync(rowlen, s); cudaFreeAsync(tmp, s);
    return FPB_ECONFIG;
  }
  *nnz_h = nnz32;
  if (colind) {
    k_pattern_rows<<<rows_grid, 256, 0, s>>>(G, n, ptr, inc, 1, nullptr, rowptr, colind);
    FPB_LAUNCH_CHECK();
  }
  FPB_CUDA(cudaFreeAsync(cnt, s));
  FPB_CUDA(cudaFreeAsync(ptr, s));
  FPB_CUDA(cudaFreeAsync(inc, s));
  FPB_CUDA(cudaFreeAsync(rowlen, s));
  FPB_CUDA(cudaFreeAsync(tmp, s));
  return FPB_OK;
}

int fpb_matrix_positions(int64_t nelem, int nn, const int32_t* conn, int32_t n,
                         const int32_t* rowptr, const int32_t* colind, int layout, int vs,
                         int32_t* pos, void* stream) {
  FPB_REQUIRE(layout == 0 || layout == 1, "layout must be 0 (scalar) or 1 (packed)");
  if (nelem == 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  int* missing = nullptr;
  FPB_CUDA(cudaMallocAsync(&missing, sizeof(int), s));
  FPB_CUDA(cudaMemsetAsync(missing, 0, sizeof(int), s));
  int64_t npacks = (nelem + vs - 1) / vs;
  int64_t total = layout == 0 ? nelem * nn * nn : npacks * nn * nn * vs;
  k_positions<<<grid_for(total, 256), 256, 0, s>>>(nelem, nn, conn, n, rowptr, colind, layout, vs,
                                                   pos, missing);
  FPB_LAUNCH_CHECK();
  int h = 0;
  FPB_CUDA(cudaMemcpyAsync(&h, missing, sizeof(int), cudaMemcpyDeviceToHost, s));
  FPB_CUDA(cudaFreeAsync(missing, s));
  FPB_CUDA(cudaStreamSynchronize(s));
  if (h) {
    set_error("element node pair missing from CSR pattern");
    return FPB_EPATTERN;
  }
  return FPB_OK;
}

int fpb_geometry(int etype, int64_t nelem, int vs, const int32_t* conn, const double* coords,
                 double* detjw, double* gradn, int64_t* bad_elem_h, int* bad_gauss_h,
                 void* stream) {
  FPB_REQUIRE(etype >= 0 && etype < 5 && g_ref_loaded[etype],
              "reference tables for element type %d not uploaded", etype);
  *bad_elem_h = -1;
  *bad_gauss_h = -1;
  if (nelem == 0) return FPB_OK;
  cudaStream_t s = as_stream(stream);
  unsigned long long* bad = nullptr;
  FPB_CUDA(cudaMallocAsync(&bad, sizeof(unsigned long long), s));
  FPB_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
  int64_t total = (nelem + vs - 1) / vs * vs;
  int grid = grid_for(total, 128);
  switch (etype) {
    case FPB_TRI03: k_geometry<FPB_TRI03><<<grid, 128, 0, s>>>(nelem, vs, conn, coords, detjw, gradn, bad); break;
    case FPB_QUAD04: k_geometry<FPB_QUAD04><<<grid, 128, 0, s>>>(nelem, vs, conn, coords, detjw, gradn, bad); break;
    case FPB_TET04: k_geometry<FPB_TET04><<<grid, 128, 0, s>>>(nelem, vs, conn, coords, detjw, gradn, bad); break;
    case FPB_PYR05: k_geometry<FPB_PYR05><<<grid, 128, 0, s>>>(nelem, vs, conn, coords, detjw, gradn, bad); break;
    case FPB_HEX08: k_geometry<FPB_HEX08><<<grid, 128, 0, s>>>(nelem, vs, conn, coords, detjw, gradn, bad); break;
  }
  FPB_LAUNCH_CHECK();
  unsigned long long h = 0;
  FPB_CUDA(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, s));
  FPB_CUDA(cudaFreeAsync(bad, s));
  FPB_CUDA(cudaStreamSynchronize(s));
  if (h != ~0ull) {
    int ng = etype_ng(etype);
    int64_t v = (int64_t)(h % vs);
    int64_t pg = (int64_t)(h / vs);
    int64_t p = pg / ng;
    *bad_gauss_h = (int)(pg % ng);
    *bad_elem_h = p * vs + v;
    set_error("non-positive Jacobian in element %lld at Gauss point %d", (long long)*bad_elem_h,
              *bad_gauss_h);
    return FPB_EINVERTED;
  }
  return FPB_OK;
}

}  // extern "C"
