// Time-loop support on the device:
//   * sparse setup of the pressure operator — transpose_csr, spgemm
//     (normal_product = A^T diag(d) A), csr_add, apply_dirichlet
//     (sparse.py:133-254, timeloop.py:184-231);
//   * Robin boundary assembly: alpha * face mass, beta * face load
//     (assembly.py:383-411);
//   * the fused elementwise stages of FlowSolver.step (timeloop.py:336-440):
//     SSP-RK3 momentum / scalar stage updates, pressure right-hand side,
//     velocity correction — each with the reference's numpy rounding
//     sequence, so they are bitwise equal to it given equal inputs.
// Setup kernels favour simplicity (one thread per row, local scratch); the
// per-step kernels are bandwidth-bound streams.
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "common.cuh"

namespace fpb {

// ---- transpose_csr (sparse.py:133-138) ---------------------------------------
// rows of A^T = columns of A; within a row, entries in ascending original row
// (lexsort((rows, colind))).  Counting sort by column, then each output row
// is ordered by its (original row) keys — deterministic.
__global__ void k_col_count(int64_t nnz, const int32_t* colind, int32_t* cnt) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[colind[k]], 1);
}

__global__ void k_transpose_fill(int32_t n, const int32_t* rowptr, const int32_t* colind, const int32_t* tptr,
                                 int32_t* cursor, int32_t* trow, int64_t* tsrc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int c = colind[k];
      const int at = tptr[c] + atomicAdd(&cursor[c], 1);
      trow[at] = (int32_t)i;
      tsrc[at] = k;
    }
}

__global__ void k_transpose_sort(int32_t n, const int32_t* tptr, int32_t* trow, int64_t* tsrc,
                                 const double* vals, double* tvals) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    const int lo = tptr[c], hi = tptr[c + 1];
    for (int x = lo + 1; x < hi; ++x) {  // insertion sort by original row
      const int r = trow[x];
      const int64_t s = tsrc[x];
      int y = x - 1;
      while (y >= lo && trow[y] > r) {
        trow[y + 1] = trow[y];
        tsrc[y + 1] = tsrc[y];
        --y;
      }
      trow[y + 1] = r;
      tsrc[y + 1] = s;
    }
    for (int x = lo; x < hi; ++x) tvals[x] = vals[tsrc[x]];
  }
}

// ---- spgemm (sparse.py:141-188) ------------------------------------------------
// One thread per output row i: products a_ij * b_jc are visited in the
// reference order (A's row ascending, then B's row ascending); a column's
// first product initialises its entry and later ones add to it, exactly as
// _spgemm_fill, so every value is bitwise the reference's.  Distinct columns
// live in per-thread scratch (first-occurrence order), sorted at the end.
constexpr int kSpgemmCap = 256;

template <bool FILL>
__global__ void __launch_bounds__(128)
k_spgemm(int32_t n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci, const double* __restrict__ av,
         const int32_t* __restrict__ brp, const int32_t* __restrict__ bci, const double* __restrict__ bv,
         const int32_t* __restrict__ rowptr, int32_t* __restrict__ counts, int32_t* __restrict__ colind,
         double* __restrict__ vals, int32_t* col_scratch, double* val_scratch, int* err) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  int32_t* cs = col_scratch + tid * kSpgemmCap;
  double* vs = val_scratch ? val_scratch + tid * kSpgemmCap : nullptr;
  for (int64_t i = tid; i < n; i += nthr) {
    int m = 0;
    for (int ka = arp[i]; ka < arp[i + 1]; ++ka) {
      const int j = aci[ka];
      const double va = FILL ? av[ka] : 0.0;
      for (int kb = brp[j]; kb < brp[j + 1]; ++kb) {
        const int c = bci[kb];
        int q = 0;
        while (q < m && cs[q] != c) ++q;
        if (q == m) {
          if (m == kSpgemmCap) {
            atomicExch(err, 1);
            break;
          }
          cs[m++] = c;
          if (FILL) vs[q] = __dmul_rn(va, bv[kb]);
        } else if (FILL) {
          vs[q] = __dadd_rn(vs[q], __dmul_rn(va, bv[kb]));  // no contraction: numba's a += b * c
        }
      }
    }
    if (!FILL) {
      counts[i] = m;
      continue;
    }
    // sort (column, value) pairs by column and write the row
    for (int x = 1; x < m; ++x) {
      const int c = cs[x];
      const double v = vs[x];
      int y = x - 1;
      while (y >= 0 && cs[y] > c) {
        cs[y + 1] = cs[y];
        vs[y + 1] = vs[y];
        --y;
      }
      cs[y + 1] = c;
      vs[y + 1] = v;
    }
    const int base = rowptr[i];
    for (int x = 0; x < m; ++x) {
      colind[base + x] = cs[x];
      vals[base + x] = vs[x];
    }
  }
}

// row scaling: out[k] = vals[k] * d[row(k)]  (normal_product's A.vals * d[rows])
__global__ void k_scale_rows(int32_t n, const int32_t* rowptr, const double* vals, const double* d, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double di = d[i];
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) out[k] = vals[k] * di;
  }
}

// ---- csr_add (sparse.py:197-214): union of sorted rows, a + b where both ----
template <bool FILL>
__global__ void k_csr_add(int32_t n, const int32_t* arp, const int32_t* aci, const double* av, const int32_t* brp,
                          const int32_t* bci, const double* bv, const int32_t* rowptr, int32_t* counts,
                          int32_t* colind, double* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int ka = arp[i], kb = brp[i];
    const int ea = arp[i + 1], eb = brp[i + 1];
    int m = 0, o = FILL ? rowptr[i] : 0;
    while (ka < ea || kb < eb) {
      const int ca = ka < ea ? aci[ka] : INT32_MAX, cb = kb < eb ? bci[kb] : INT32_MAX;
      const int c = ca < cb ? ca : cb;
      if (FILL) {
        // np.add.at into zeros in [A, B] order: (0 + a) + b
        double v = 0.0;
        if (ca == c) v = v + av[ka];
        if (cb == c) v = v + bv[kb];
        colind[o + m] = c;
        vals[o + m] = v;
      }
      if (ca == c) ++ka;
      if (cb == c) ++kb;
      ++m;
    }
    if (!FILL) counts[i] = m;
  }
}

// ---- apply_dirichlet (sparse.py:219-254) ----------------------------------------
// b -= A[:, nodes] @ values on unflagged rows (in ascending entry order, like
// np.subtract.at), b[nodes] = values; rows and columns zeroed, diagonal one.
__global__ void k_dirichlet(int32_t n, const int32_t* rowptr, const int32_t* colind, const double* vals,
                            const uint8_t* flag, const double* lift, double* out, double* b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool ri = flag[i] != 0;
    double bi = b ? b[i] : 0.0;
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int c = colind[k];
      const bool ci = flag[c] != 0;
      if (b && ci && !ri) bi = __dsub_rn(bi, __dmul_rn(vals[k], lift[c]));
      out[k] = (ri || ci) ? (c == i && ri ? 1.0 : 0.0) : vals[k];
    }
    if (b) b[i] = ri ? lift[i] : bi;
  }
}

// ---- Robin boundary (assembly.py:383-411) ---------------------------------------
// One thread per face: surface element dA = |J| (2D: |dx/ds|; 3D:
// |dx/ds x dx/dt|), w_g = dA wts_g; Me = alpha w N_i N_j -> vals[pos], re =
// beta w N_i -> rhs[node] (FP64 reductions; 0.09 % of the paper's step).
__global__ void k_robin(int64_t nf, int nnf, int ng, int dim, const int32_t* conn, const double* coords,
                        const double* N, const double* dN, const double* wts, const int32_t* pos, double alpha,
                        double beta, double* vals, double* rhs) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    double x[4][3];
    for (int a = 0; a < nnf; ++a)
      for (int d = 0; d < dim; ++d) x[a][d] = coords[(int64_t)conn[f * nnf + a] * dim + d];
    double Me[16], re[4];
    for (int q = 0; q < 16; ++q) Me[q] = 0.0;
    for (int q = 0; q < 4; ++q) re[q] = 0.0;
    for (int g = 0; g < ng; ++g) {
      double t[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};  // J[.][d][l]
      for (int l = 0; l < dim - 1; ++l)
        for (int d = 0; d < dim; ++d) {
          double s = 0.0;
          for (int a = 0; a < nnf; ++a) s += x[a][d] * dN[(l * nnf + a) * ng + g];
          t[l][d] = s;
        }
      double dA;
      if (dim == 2) {
        dA = sqrt(__dadd_rn(__dmul_rn(t[0][0], t[0][0]), __dmul_rn(t[0][1], t[0][1])));
      } else {
        const double c0 = t[0][1] * t[1][2] - t[0][2] * t[1][1];
        const double c1 = t[0][2] * t[1][0] - t[0][0] * t[1][2];
        const double c2 = t[0][0] * t[1][1] - t[0][1] * t[1][0];
        dA = sqrt(c0 * c0 + c1 * c1 + c2 * c2);
      }
      const double w = dA * wts[g];
      for (int i = 0; i < nnf; ++i) {
        const double Ni = N[i * ng + g];
        re[i] += w * Ni;
        for (int j = 0; j < nnf; ++j) Me[i * nnf + j] += w * Ni * N[j * ng + g];
      }
    }
    if (alpha != 0.0)
      for (int q = 0; q < nnf * nnf; ++q) atomicAdd(&vals[pos[f * nnf * nnf + q]], alpha * Me[q]);
    if (beta != 0.0)
      for (int i = 0; i < nnf; ++i) atomicAdd(&rhs[conn[f * nnf + i]], beta * re[i]);
  }
}

// ---- FlowSolver.step stages (timeloop.py:367-440) -------------------------------
// momentum stage, per node i and component k (numpy evaluation order):
//   r = r + (load - Ru_k)   [Robin, when load != NULL]
//   r = r - grad_p
//   un = a * u0 + b * (uc + dt_rho * (r / lumped))
__global__ void k_stage_momentum(int64_t n, int dim, double a, double b, double dt_rho, const double* u0,
                                 const double* uc, const double* r, const double* grad_p, const double* lumped,
                                 const double* load, const double* Ru, double* un) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * dim; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / dim;
    const int k = (int)(t - i * dim);
    double rr = r[t];
    if (load) rr = __dadd_rn(rr, __dsub_rn(load[i], Ru[(int64_t)k * n + i]));
    rr = __dsub_rn(rr, grad_p[t]);
    const double inc = __dmul_rn(dt_rho, __ddiv_rn(rr, lumped[i]));
    un[t] = __dadd_rn(__dmul_rn(a, u0[t]), __dmul_rn(b, __dadd_rn(uc[t], inc)));
  }
}

// scalar stage: sn = a * phi0 + b * (phi + dt * (rs / lumped))
__global__ void k_stage_scalar(int64_t n, double a, double b, double dt, const double* phi0, const double* phi,
                               const double* rs, const double* lumped, double* sn) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double inc = __dmul_rn(dt, __ddiv_rn(rs[i], lumped[i]));
    sn[i] = __dadd_rn(__dmul_rn(a, phi0[i]), __dmul_rn(b, __dadd_rn(phi[i], inc)));
  }
}

// masked copy: u[nodes[q]] = values[q] (row of dim values)
__global__ void k_set_rows(int64_t m, int dim, const int64_t* nodes, const double* values, double* u) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * dim; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = t / dim;
    u[nodes[q] * dim + (t - q * dim)] = values ? values[t] : 0.0;
  }
}

// divergence accumulation: div = div - s   (out -= spmv(div_mats[k], u_k))
// and the pressure right-hand side after the last component:
//   g = (-rho / dt) * div
__global__ void k_axpy_sub(int64_t n, const double* s, double* div, double scale, double* g) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = __dsub_rn(div[i], s[i]);
    div[i] = d;
    if (g) g[i] = __dmul_rn(scale, d);
  }
}

// correction: corr_k = s_k / lumped (0 on Dirichlet rows); u_new = uc - dt_rho * corr
__global__ void k_correct(int64_t n, int dim, int k, double dt_rho, const double* s, const double* lumped,
                          const uint8_t* dflag, const double* uc, double* un) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double corr = __ddiv_rn(s[i], lumped[i]);
    if (dflag && dflag[i]) corr = 0.0;
    un[i * dim + k] = __dsub_rn(uc[i * dim + k], __dmul_rn(dt_rho, corr));
  }
}

}  // namespace fpb

using namespace fpb;

extern "C" {

int fpb_csr_transpose(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind, const double* vals,
                      int32_t* trowptr, int32_t* tcolind, double* tvals, void* stream) {
  cudaStream_t s = as_stream(stream);
  int32_t *cnt = nullptr, *cursor = nullptr;
  int64_t* src = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  FPB_CUDA(cudaMallocAsync(&cnt, sizeof(int32_t) * (n + 1), s));
  FPB_CUDA(cudaMallocAsync(&cursor, sizeof(int32_t) * (n + 1), s));
  FPB_CUDA(cudaMallocAsync(&src, sizeof(int64_t) * (nnz > 0 ? nnz : 1), s));
  FPB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), s));
  FPB_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (n + 1), s));
  if (nnz > 0) k_col_count<<<grid_for(nnz, 256), 256, 0, s>>>(nnz, colind, cnt);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, trowptr, n + 1, s);
  FPB_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
  FPB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, trowptr, n + 1, s));
  if (n > 0) {
    k_transpose_fill<<<grid_for(n, 256), 256, 0, s>>>(n, rowptr, colind, trowptr, cursor, tcolind, src);
    k_transpose_sort<<<grid_for(n, 256), 256, 0, s>>>(n, trowptr, tcolind, src, vals, tvals);
  }
  FPB_LAUNCH_CHECK();
  FPB_CUDA(cudaFreeAsync(tmp, s));
  FPB_CUDA(cudaFreeAsync(src, s));
  FPB_CUDA(cudaFreeAsync(cursor, s));
  FPB_CUDA(cudaFreeAsync(cnt, s));
  return FPB_OK;
}

static int spgemm_threads(int32_t n) { return (int)std::min<int64_t>(std::max<int32_t>(n, 1), 148 * 256); }

int fpb_spgemm_count(int32_t n, const int32_t* arp, const int32_t* aci, const int32_t* brp, const int32_t* bci,
                     int32_t* counts, void* stream) {
  cudaStream_t s = as_stream(stream);
  const int nt = spgemm_threads(n);
  int32_t* cs = nullptr;
  int* err = nullptr;
  FPB_CUDA(cudaMallocAsync(&cs, sizeof(int32_t) * (size_t)nt * kSpgemmCap, s));
  FPB_CUDA(cudaMallocAsync(&err, sizeof(int), s));
  FPB_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
  if (n > 0)
    k_spgemm<false><<<(nt + 127) / 128, 128, 0, s>>>(n, arp, aci, nullptr, brp, bci, nullptr, nullptr, counts,
                                                     nullptr, nullptr, cs, nullptr, err);
  FPB_LAUNCH_CHECK();
  int h = 0;
  FPB_CUDA(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  FPB_CUDA(cudaFreeAsync(cs, s));
  FPB_CUDA(cudaFreeAsync(err, s));
  FPB_CUDA(cudaStreamSynchronize(s));
  if (h) {
    set_error("spgemm row has more than %d distinct columns", kSpgemmCap);
    return FPB_ECONFIG;
  }
  return FPB_OK;
}

int fpb_spgemm_fill(int32_t n, const int32_t* arp, const int32_t* aci, const double* av, const int32_t* brp,
                    const int32_t* bci, const double* bv, const int32_t* rowptr, int32_t* colind, double* vals,
                    void* stream) {
  cudaStream_t s = as_stream(stream);
  const int nt = spgemm_threads(n);
  int32_t* cs = nullptr;
  double* vs = nullptr;
  int* err = nullptr;
  FPB_CUDA(cudaMallocAsync(&cs, sizeof(int32_t) * (size_t)nt * kSpgemmCap, s));
  FPB_CUDA(cudaMallocAsync(&vs, sizeof(double) * (size_t)nt * kSpgemmCap, s));
  FPB_CUDA(cudaMallocAsync(&err, sizeof(int), s));
  FPB_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
  if (n > 0)
    k_spgemm<true><<<(nt + 127) / 128, 128, 0, s>>>(n, arp, aci, av, brp, bci, bv, rowptr, nullptr, colind, vals,
                                                    cs, vs, err);
  FPB_LAUNCH_CHECK();
  FPB_CUDA(cudaFreeAsync(cs, s));
  FPB_CUDA(cudaFreeAsync(vs, s));
  FPB_CUDA(cudaFreeAsync(err, s));
  return FPB_OK;
}

int fpb_scale_rows(int32_t n, const int32_t* rowptr, const double* vals, const double* d, double* out,
                   void* stream) {
  if (n > 0) k_scale_rows<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, rowptr, vals, d, out);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_csr_add_count(int32_t n, const int32_t* arp, const int32_t* aci, const int32_t* brp, const int32_t* bci,
                      int32_t* counts, void* stream) {
  if (n > 0)
    k_csr_add<false><<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, arp, aci, nullptr, brp, bci, nullptr,
                                                                      nullptr, counts, nullptr, nullptr);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_csr_add_fill(int32_t n, const int32_t* arp, const int32_t* aci, const double* av, const int32_t* brp,
                     const int32_t* bci, const double* bv, const int32_t* rowptr, int32_t* colind, double* vals,
                     void* stream) {
  if (n > 0)
    k_csr_add<true><<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, arp, aci, av, brp, bci, bv, rowptr,
                                                                     nullptr, colind, vals);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_apply_dirichlet(int32_t n, const int32_t* rowptr, const int32_t* colind, const double* vals,
                        const uint8_t* flag, const double* lift, double* out, double* b, void* stream) {
  FPB_REQUIRE(!b || lift, "a right-hand side needs the lifted Dirichlet values");
  if (n > 0) k_dirichlet<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, rowptr, colind, vals, flag, lift, out, b);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_robin(int64_t nf, int nnf, int ng, int dim, const int32_t* conn, const double* coords, const double* N,
              const double* dN, const double* wts, const int32_t* pos, double alpha, double beta, double* vals,
              double* rhs, void* stream) {
  FPB_REQUIRE(nnf >= 2 && nnf <= 4 && ng >= 1 && ng <= 16 && (dim == 2 || dim == 3), "bad face rule");
  FPB_REQUIRE(alpha == 0.0 || pos, "alpha != 0 needs the face->CSR map");
  if (nf > 0)
    k_robin<<<grid_for(nf, 128), 128, 0, as_stream(stream)>>>(nf, nnf, ng, dim, conn, coords, N, dN, wts, pos, alpha,
                                                             beta, vals, rhs);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_stage_momentum(int64_t n, int dim, double a, double b, double dt_rho, const double* u0, const double* uc,
                       const double* r, const double* grad_p, const double* lumped, const double* load,
                       const double* Ru, double* un, void* stream) {
  FPB_REQUIRE(!load || Ru, "Robin load needs R u");
  if (n > 0)
    k_stage_momentum<<<grid_for(n * dim, 256, 8), 256, 0, as_stream(stream)>>>(n, dim, a, b, dt_rho, u0, uc, r,
                                                                             grad_p, lumped, load, Ru, un);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_stage_scalar(int64_t n, double a, double b, double dt, const double* phi0, const double* phi,
                     const double* rs, const double* lumped, double* sn, void* stream) {
  if (n > 0)
    k_stage_scalar<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(n, a, b, dt, phi0, phi, rs, lumped, sn);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_set_rows(int64_t m, int dim, const int64_t* nodes, const double* values, double* u, void* stream) {
  if (m > 0) k_set_rows<<<grid_for(m * dim, 256), 256, 0, as_stream(stream)>>>(m, dim, nodes, values, u);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_sub_into(int64_t n, const double* s, double* div, double scale, double* g, void* stream) {
  if (n > 0) k_axpy_sub<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(n, s, div, scale, g);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

int fpb_correct(int64_t n, int dim, int k, double dt_rho, const double* s, const double* lumped,
                const uint8_t* dflag, const double* uc, double* un, void* stream) {
  if (n > 0)
    k_correct<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(n, dim, k, dt_rho, s, lumped, dflag, uc, un);
  FPB_LAUNCH_CHECK();
  return FPB_OK;
}

}  // extern "C"
