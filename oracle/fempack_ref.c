/*
 * CPU oracle (TEST/BASELINE INFRASTRUCTURE ONLY) — C restatement of the
 * reference's packed assembly kernels and CSR vector kernels
 * (/root/reference/pkg/src/fempack/_kernels.py, sparse.py), used as the
 * `cpu_baseline` / `--impl reference` arm of bench.py ("kind": "port") and as
 * a fast checker at sizes the NumPy oracle handles slowly.
 *
 * Loop nests, lane-last layouts and the order of every floating-point
 * operation follow the reference kernels line by line (cited per function);
 * compiled with -ffp-contract=off, like Numba without fastmath, so results are
 * plain IEEE mul/add.  OpenMP splits packs across threads; the scatter uses
 * atomic adds (the reference's scatter is sequential, so summation order — and
 * only that — differs when nthreads > 1).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library.  Never part of the product path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXNN 8
#define MAXNG 8
#define MAXVS 32

/* geometry_packed (_kernels.py:78-147) for one pack; returns 0 or 1 + (v * MAXNG + ig) */
static int geometry_pack(int64_t p, int nn, int ng, int dim, int vs, int64_t nelem,
                         const int64_t* lane_conn, const double* coords, const double* dN,
                         const double* wg, double* detjw, double* gradn) {
  double xe[MAXNN][3][MAXVS], J[3][3][MAXVS], Ji[3][3][MAXVS], det[MAXVS];
  int64_t nact = nelem - p * vs;
  if (nact > vs) nact = vs;
  for (int a = 0; a < nn; ++a)
    for (int d = 0; d < dim; ++d)
      for (int v = 0; v < vs; ++v) xe[a][d][v] = coords[lane_conn[((int64_t)p * nn + a) * vs + v] * dim + d];
  for (int ig = 0; ig < ng; ++ig) {
    for (int d = 0; d < dim; ++d)
      for (int l = 0; l < dim; ++l) {
        for (int v = 0; v < vs; ++v) J[d][l][v] = 0.0;
        for (int a = 0; a < nn; ++a)
          for (int v = 0; v < vs; ++v) J[d][l][v] += xe[a][d][v] * dN[(l * nn + a) * ng + ig];
      }
    if (dim == 2) {
      for (int v = 0; v < vs; ++v) det[v] = J[0][0][v] * J[1][1][v] - J[0][1][v] * J[1][0][v];
    } else {
      for (int v = 0; v < vs; ++v)
        det[v] = J[0][0][v] * (J[1][1][v] * J[2][2][v] - J[1][2][v] * J[2][1][v]) -
                 J[0][1][v] * (J[1][0][v] * J[2][2][v] - J[1][2][v] * J[2][0][v]) +
                 J[0][2][v] * (J[1][0][v] * J[2][1][v] - J[1][1][v] * J[2][0][v]);
    }
    for (int v = 0; v < nact; ++v)
      if (det[v] <= 0.0) return 1 + v * MAXNG + ig;
    for (int v = 0; v < vs; ++v) detjw[ig * vs + v] = det[v] * wg[ig];
    for (int v = (int)nact; v < vs; ++v) detjw[ig * vs + v] = 0.0;
    if (dim == 2) {
      for (int v = 0; v < vs; ++v) {
        double inv = 1.0 / det[v];
        Ji[0][0][v] = J[1][1][v] * inv;
        Ji[0][1][v] = -J[0][1][v] * inv;
        Ji[1][0][v] = -J[1][0][v] * inv;
        Ji[1][1][v] = J[0][0][v] * inv;
      }
    } else {
      for (int v = 0; v < vs; ++v) {
        double inv = 1.0 / det[v];
        Ji[0][0][v] = (J[1][1][v] * J[2][2][v] - J[1][2][v] * J[2][1][v]) * inv;
        Ji[0][1][v] = (J[0][2][v] * J[2][1][v] - J[0][1][v] * J[2][2][v]) * inv;
        Ji[0][2][v] = (J[0][1][v] * J[1][2][v] - J[0][2][v] * J[1][1][v]) * inv;
        Ji[1][0][v] = (J[1][2][v] * J[2][0][v] - J[1][0][v] * J[2][2][v]) * inv;
        Ji[1][1][v] = (J[0][0][v] * J[2][2][v] - J[0][2][v] * J[2][0][v]) * inv;
        Ji[1][2][v] = (J[0][2][v] * J[1][0][v] - J[0][0][v] * J[1][2][v]) * inv;
        Ji[2][0][v] = (J[1][0][v] * J[2][1][v] - J[1][1][v] * J[2][0][v]) * inv;
        Ji[2][1][v] = (J[0][1][v] * J[2][0][v] - J[0][0][v] * J[2][1][v]) * inv;
        Ji[2][2][v] = (J[0][0][v] * J[1][1][v] - J[0][1][v] * J[1][0][v]) * inv;
      }
    }
    for (int a = 0; a < nn; ++a)
      for (int d = 0; d < dim; ++d)
        for (int v = 0; v < vs; ++v) {
          double acc = 0.0;
          for (int l = 0; l < dim; ++l) acc += Ji[l][d][v] * dN[(l * nn + a) * ng + ig];
          gradn[((d * nn + a) * ng + ig) * vs + v] = acc;
        }
  }
  return 0;
}

/* Geometry for all packs: detjw[npacks][ng][vs], gradn[npacks][dim][nn][ng][vs].
 * Returns -1 or the first bad p*vs+v (gauss in *bad_gauss). */
int64_t orc_geometry(int64_t npacks, int nn, int ng, int dim, int vs, int64_t nelem,
                     const int64_t* lane_conn, const double* coords, const double* dN,
                     const double* wg, double* detjw, double* gradn, int* bad_gauss, int nthreads) {
  int64_t bad = -1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t p = 0; p < npacks; ++p) {
    int rc = geometry_pack(p, nn, ng, dim, vs, nelem, lane_conn, coords, dN, wg,
                           detjw + p * ng * vs, gradn + p * dim * nn * ng * vs);
    if (rc) {
#pragma omp critical
      {
        int64_t e = p * vs + (rc - 1) / MAXNG;
        if (bad < 0 || e < bad) { bad = e; *bad_gauss = (rc - 1) % MAXNG; }
      }
    }
  }
  return bad;
}

static inline void atomic_add(double* p, double v) {
#pragma omp atomic
  *p += v;
}

/* momentum_rhs_packed (_kernels.py:320-382) + scatter_vector_dim_packed
 * (_kernels.py:511-519), one pack at a time, reading cached geometry. */
void orc_momentum_rhs(int64_t npacks, int nn, int ng, int dim, int vs, const int64_t* lane_conn,
                      const double* N, const double* detjw, const double* gradn,
                      const double* vel, double rho, double mu, double* rhs, int nthreads) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t p = 0; p < npacks; ++p) {
    double ue[MAXNN][3][MAXVS], ug[3][MAXVS], G[3][3][MAXVS], S[3][3][MAXVS], c[3][MAXVS];
    double divu[MAXVS], visc[MAXVS], us[MAXVS], gk[MAXVS], out[MAXNN][3][MAXVS];
    const int64_t* lc = lane_conn + p * nn * vs;
    const double* dj = detjw + p * ng * vs;
    const double* gr = gradn + p * dim * nn * ng * vs;
    memset(out, 0, sizeof(out));
    for (int a = 0; a < nn; ++a)
      for (int d = 0; d < dim; ++d)
        for (int v = 0; v < vs; ++v) ue[a][d][v] = vel[lc[a * vs + v] * dim + d];
    for (int ig = 0; ig < ng; ++ig) {
      for (int d = 0; d < dim; ++d) {
        for (int v = 0; v < vs; ++v) ug[d][v] = 0.0;
        for (int a = 0; a < nn; ++a)
          for (int v = 0; v < vs; ++v) ug[d][v] += ue[a][d][v] * N[a * ng + ig];
      }
      for (int l = 0; l < dim; ++l)
        for (int k = 0; k < dim; ++k) {
          for (int v = 0; v < vs; ++v) G[l][k][v] = 0.0;
          for (int a = 0; a < nn; ++a)
            for (int v = 0; v < vs; ++v) G[l][k][v] += ue[a][k][v] * gr[((l * nn + a) * ng + ig) * vs + v];
        }
      for (int v = 0; v < vs; ++v) divu[v] = 0.0;
      for (int d = 0; d < dim; ++d)
        for (int v = 0; v < vs; ++v) divu[v] += G[d][d][v];
      for (int l = 0; l < dim; ++l)
        for (int k = 0; k < dim; ++k)
          for (int v = 0; v < vs; ++v) S[l][k][v] = 0.5 * (G[l][k][v] + G[k][l][v]);
      for (int k = 0; k < dim; ++k) {
        for (int v = 0; v < vs; ++v) { us[v] = 0.0; gk[v] = 0.0; }
        for (int l = 0; l < dim; ++l)
          for (int v = 0; v < vs; ++v) {
            us[v] += ug[l][v] * S[l][k][v];
            gk[v] += ug[l][v] * G[k][l][v];
          }
        for (int v = 0; v < vs; ++v) c[k][v] = 2.0 * us[v] + divu[v] * ug[k][v] - gk[v];
      }
      for (int i = 0; i < nn; ++i)
        for (int k = 0; k < dim; ++k) {
          for (int v = 0; v < vs; ++v) visc[v] = 0.0;
          for (int l = 0; l < dim; ++l)
            for (int v = 0; v < vs; ++v) visc[v] += S[k][l][v] * gr[((l * nn + i) * ng + ig) * vs + v];
          for (int v = 0; v < vs; ++v)
            out[i][k][v] -= dj[ig * vs + v] * (rho * N[i * ng + ig] * c[k][v] + 2.0 * mu * visc[v]);
        }
    }
    for (int i = 0; i < nn; ++i)
      for (int v = 0; v < vs; ++v) {
        int64_t node = lc[i * vs + v];
        for (int d = 0; d < dim; ++d) {
          if (nthreads > 1) atomic_add(&rhs[node * dim + d], out[i][d][v]);
          else rhs[node * dim + d] += out[i][d][v];
        }
      }
  }
}

/* convection_packed (_kernels.py:238-266) + scatter_matrix_packed
 * (_kernels.py:473-481); vel may be a unit field e_k (continuity B_k). */
void orc_convection(int64_t npacks, int nn, int ng, int dim, int vs, const int64_t* lane_conn,
                    const double* N, const double* detjw, const double* gradn, const double* vel,
                    const int64_t* pos, double* vals, int nthreads) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t p = 0; p < npacks; ++p) {
    double ue[MAXNN][3][MAXVS], ug[3][MAXVS], adv[MAXVS], out[MAXNN][MAXNN][MAXVS];
    const int64_t* lc = lane_conn + p * nn * vs;
    const double* dj = detjw + p * ng * vs;
    const double* gr = gradn + p * dim * nn * ng * vs;
    memset(out, 0, sizeof(out));
    for (int a = 0; a < nn; ++a)
      for (int d = 0; d < dim; ++d)
        for (int v = 0; v < vs; ++v) ue[a][d][v] = vel[lc[a * vs + v] * dim + d];
    for (int ig = 0; ig < ng; ++ig) {
      for (int d = 0; d < dim; ++d) {
        for (int v = 0; v < vs; ++v) ug[d][v] = 0.0;
        for (int a = 0; a < nn; ++a)
          for (int v = 0; v < vs; ++v) ug[d][v] += ue[a][d][v] * N[a * ng + ig];
      }
      for (int j = 0; j < nn; ++j) {
        for (int v = 0; v < vs; ++v) adv[v] = 0.0;
        for (int d = 0; d < dim; ++d)
          for (int v = 0; v < vs; ++v) adv[v] += ug[d][v] * gr[((d * nn + j) * ng + ig) * vs + v];
        for (int i = 0; i < nn; ++i)
          for (int v = 0; v < vs; ++v) out[i][j][v] += dj[ig * vs + v] * adv[v] * N[i * ng + ig];
      }
    }
    const int64_t* pp = pos + p * nn * nn * vs;
    for (int i = 0; i < nn; ++i)
      for (int j = 0; j < nn; ++j)
        for (int v = 0; v < vs; ++v) {
          if (nthreads > 1) atomic_add(&vals[pp[(i * nn + j) * vs + v]], out[i][j][v]);
          else vals[pp[(i * nn + j) * vs + v]] += out[i][j][v];
        }
  }
}

/* scalar_rhs_packed (_kernels.py:420-461) + scatter_vector_packed
 * (_kernels.py:492-498). */
void orc_scalar_rhs(int64_t npacks, int nn, int ng, int dim, int vs, const int64_t* lane_conn,
                    const double* N, const double* detjw, const double* gradn, const double* vel,
                    const double* phi, double kappa, double* rhs, int nthreads) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t p = 0; p < npacks; ++p) {
    double ue[MAXNN][3][MAXVS], fe[MAXNN][MAXVS], ug[3][MAXVS], gphi[3][MAXVS];
    double adv[MAXVS], diff[MAXVS], out[MAXNN][MAXVS];
    const int64_t* lc = lane_conn + p * nn * vs;
    const double* dj = detjw + p * ng * vs;
    const double* gr = gradn + p * dim * nn * ng * vs;
    memset(out, 0, sizeof(out));
    for (int a = 0; a < nn; ++a)
      for (int v = 0; v < vs; ++v) {
        int64_t node = lc[a * vs + v];
        fe[a][v] = phi[node];
        for (int d = 0; d < dim; ++d) ue[a][d][v] = vel[node * dim + d];
      }
    for (int ig = 0; ig < ng; ++ig) {
      for (int d = 0; d < dim; ++d) {
        for (int v = 0; v < vs; ++v) { ug[d][v] = 0.0; gphi[d][v] = 0.0; }
        for (int a = 0; a < nn; ++a)
          for (int v = 0; v < vs; ++v) {
            ug[d][v] += ue[a][d][v] * N[a * ng + ig];
            gphi[d][v] += fe[a][v] * gr[((d * nn + a) * ng + ig) * vs + v];
          }
      }
      for (int v = 0; v < vs; ++v) adv[v] = 0.0;
      for (int d = 0; d < dim; ++d)
        for (int v = 0; v < vs; ++v) adv[v] += ug[d][v] * gphi[d][v];
      for (int i = 0; i < nn; ++i) {
        for (int v = 0; v < vs; ++v) diff[v] = 0.0;
        for (int d = 0; d < dim; ++d)
          for (int v = 0; v < vs; ++v) diff[v] += gphi[d][v] * gr[((d * nn + i) * ng + ig) * vs + v];
        for (int v = 0; v < vs; ++v)
          out[i][v] -= dj[ig * vs + v] * (N[i * ng + ig] * adv[v] + kappa * diff[v]);
      }
    }
    for (int i = 0; i < nn; ++i)
      for (int v = 0; v < vs; ++v) {
        int64_t node = lc[i * vs + v];
        if (nthreads > 1) atomic_add(&rhs[node], out[i][v]);
        else rhs[node] += out[i][v];
      }
  }
}

/* _spmv (sparse.py:78-84) */
void orc_spmv(int64_t n, const int64_t* rowptr, const int64_t* colind, const double* vals,
              const double* x, double* y, int nthreads) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) acc += vals[k] * x[colind[k]];
    y[i] = acc;
  }
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
