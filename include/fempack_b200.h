/*
 * fempack_b200 — C ABI of the B200-native FE assembly + solver-vector path.
 *
 * Drop-in boundary for the reference mini-app `fempack`
 * (/root/reference/pkg/src/fempack).  The reference is Python/Numba and binds
 * no FFI; each entry point below replaces one reference kernel or setup
 * routine (cited per function).  The Python host package
 * `paper_2107_11541_b200` binds these through ctypes.
 *
 * Conventions (mirroring the reference kernel contract, _kernels.py:1-15):
 *  - every pointer argument is a DEVICE pointer unless the name ends in _h;
 *  - outputs are caller-allocated; assembly kernels ACCUMULATE into them
 *    (callers zero them, as assembly.py:167/:206 do);
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *  - calls are stream-ordered and asynchronous unless documented otherwise;
 *  - return FPB_OK (0) or an error code; fpb_last_error() describes it.
 *
 * Index types: node ids, connectivity, CSR column indices, row pointers and
 * element->CSR positions are int32 on the device (every BASELINE config has
 * nnz < 2^31; larger meshes are rejected with FPB_ECONFIG).
 */
#ifndef FEMPACK_B200_H
#define FEMPACK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define FPB_OK 0
#define FPB_ECONFIG 1   /* ConfigurationError (errors.py:4-5) */
#define FPB_EINVERTED 2 /* InvertedElementError (errors.py:8-22) */
#define FPB_EPATTERN 3  /* ScatterPatternError (errors.py:33-34) */
#define FPB_ECUDA 4     /* CUDA runtime failure */

/* element types, ElementType (elements.py:28-33) */
typedef enum { FPB_TRI03 = 0, FPB_QUAD04 = 1, FPB_TET04 = 2, FPB_PYR05 = 3, FPB_HEX08 = 4 } fpb_etype;

/* kernel kinds, KernelKind (assembly.py:32-41), plus the fused continuity
 * kind FPB_GRADIENT_XYZ (= CONVECTION with unit e_k for k < dim in one pass,
 * timeloop.py:159-171) */
typedef enum {
  FPB_MASS = 0,
  FPB_LAPLACIAN = 1,
  FPB_CONVECTION = 2,
  FPB_MOMENTUM_RHS = 3,
  FPB_SCALAR_RHS = 4,
  FPB_GRADIENT_XYZ = 5
} fpb_kind;

const char* fpb_last_error(void);
int fpb_version(void);
/* Performance knobs with no effect beyond rounding (for measured design
 * choices, profiles/): "rows_nb" = 0 assembles simplex matrices with the
 * incidence-walking row kernel instead of the neighbour-staged one;
 * "blk_pipe" element-block pipelining; "kgrad_march" = 0 runs Kuhn-box B_xyz
 * interior rows by the row kernel instead of the z-marching lines;
 * "kgrad_kchunk" planes per z-chunk of the lines (0 = from the grid);
 * "kgrad_bthreads" threads per CTA of the Kuhn boundary rows (32/64/128);
 * "kmom_smem_kb" pads the Kuhn momentum CTA's shared memory (co-residency
 * experiments); "hex_canon_rows" rows per CTA of the hex row pass (32/64).
 * Python presets any of them from FPB_TUNE_<NAME>=<int> at library load. */
int fpb_set_tuning(const char* name, int value);

/* Upload one reference element's tables (host pointers) to device constant
 * memory: N[nn][ng], dN[dim][nn][ng], w[ng] — the constant inputs of every
 * reference kernel (elements.py:258-274). */
int fpb_set_reference_element(int etype, int nn, int ng, int dim, const double* N_h,
                              const double* dN_h, const double* w_h);

/* ---- setup (mesh.py, packing.py, sparse.py, assembly.py) -------------- */

/* Structured-grid node coordinates, i fastest, np.linspace-exact
 * (mesh.py:158-187).  coords[(nx+1)(ny+1)(nz+1)][3] (2-D: [(nx+1)(ny+1)][2],
 * nz ignored). */
int fpb_grid_coords(int dim, int nx, int ny, int nz, double lx, double ly, double lz,
                    double* coords, void* stream);

/* Planes k0 .. k0+nplanes-1 of the (nx, ny, nz) grid (z-slab of a larger
 * mesh for domain decomposition); coords[(nx+1)(ny+1) nplanes][3], values
 * identical to the corresponding rows of fpb_grid_coords on the full grid. */
int fpb_grid_coords_slab(int nx, int ny, int nz, int k0, int nplanes, double lx, double ly, double lz,
                         double* coords, void* stream);

/* Single-type box connectivity, cells k-major (mesh.py:227-289):
 * TET04 = 6 Kuhn tets/cell, HEX08 = 1/cell, QUAD04 = 1/cell, TRI03 = 2/cell.
 * conn[nelem][nn] int32. */
int fpb_box_conn(int etype, int nx, int ny, int nz, int32_t* conn, void* stream);

/* Mixed pyramid/hex box (mesh.py:292-336): cells with i < nlayers become 6
 * pyramids around an appended centre node.  Writes pyramid connectivity
 * pyr_conn[6*npyrcells][5], hex_conn[nhexcells][8] and the centre
 * coordinates into coords[ngrid + c][3] (coords[0:ngrid] must already hold
 * the grid from fpb_grid_coords). */
int fpb_mixed_conn(int nx, int ny, int nz, int nlayers, double* coords, int32_t* pyr_conn,
                   int32_t* hex_conn, void* stream);

/* Lane packs (packing.py:85-127): lane_conn[npacks][nn][vs] with the tail
 * replicating the last element.  npacks = ceil(nelem/vs). */
int fpb_build_packs(int64_t nelem, int nn, int vs, const int32_t* conn, int32_t* lane_conn,
                    void* stream);

/* Node-adjacency CSR graph (sparse.py:59-75).  Two calls: with colind==NULL
 * it fills rowptr[n+1] and returns nnz through nnz_h (synchronous); with
 * colind!=NULL it fills colind[nnz] (ascending within rows, diagonal always
 * present).  groups: ngroups connectivity arrays conns[g][nelem[g]][nn[g]]
 * given as host arrays of device pointers. */
int fpb_build_pattern(int32_t n, int ngroups, const int32_t* const* conns_h,
                      const int64_t* nelem_h, const int* nn_h, int32_t* rowptr, int32_t* colind,
                      int64_t* nnz_h, void* stream);

/* Element->CSR value index (assembly.py:44-52, :89-93).  layout 0 = scalar
 * pos[e][i][j]; layout 1 = packed pos[p][i][j][vs] (padded lanes replicate
 * the last element).  Returns FPB_EPATTERN (synchronously) if a node pair is
 * missing from the pattern. */
int fpb_matrix_positions(int64_t nelem, int nn, const int32_t* conn, int32_t n,
                         const int32_t* rowptr, const int32_t* colind, int layout, int vs,
                         int32_t* pos, void* stream);

/* Geometry (_kernels.py:78-147) in the reference packed layout at pack width
 * vs: detjw[npacks][ng][vs], gradn[npacks][dim][nn][ng][vs] (gradn may be
 * NULL).  Padded lanes get detjw = 0.  Returns FPB_EINVERTED (synchronously)
 * with *bad_elem_h / *bad_gauss_h set to the first non-positive determinant
 * in the reference's (pack, gauss, lane) scan order. */
int fpb_geometry(int etype, int64_t nelem, int vs, const int32_t* conn, const double* coords,
                 double* detjw, double* gradn, int64_t* bad_elem_h, int* bad_gauss_h,
                 void* stream);

/* ---- assembly (assembly.py:209-270, _kernels.py:150-519) -------------- */

/* One element group, packed at 32 lanes (one warp per pack).
 *  lane_conn[npacks][nn][32]   (fpb_build_packs with vs = 32)
 *  coords[nnode][dim], vel[nnode][dim] (CONVECTION / *_RHS), phi[nnode]
 *  pos[npacks][nn][nn][32]     (matrix kinds; fpb_matrix_positions layout 1, vs 32)
 *  out: matrix kinds -> vals[nnz]; FPB_GRADIENT_XYZ -> dim arrays vals[k*nnz]
 *       MOMENTUM_RHS -> rhs[nnode][dim]; SCALAR_RHS -> rhs[nnode]
 * Contributions are added with FP64 reductions (scatter). */
int fpb_assemble(int kind, int etype, int64_t nelem, const int32_t* lane_conn,
                 const double* coords, const double* vel, const double* phi, double rho,
                 double mu, double kappa, const int32_t* pos, int64_t nnz, double* out,
                 void* stream);

/* HEX08 continuity matrices B_x, B_y, B_z with each element's geometry
 * evaluated once (hexblock.cu), replacing the reference's 3 x CONVECTION(e_k)
 * of gradient_matrices (timeloop.py:159-171, _kernels.py:238-266).
 * fpb_hex_gradient_h: H[72][nelem] (plane q = 24 k + 8 l + 4 s + U': the
 *   Walsh-transformed adjugate columns, see hexblock.cu); conn[nelem][8]
 *   16-byte aligned, xyz4 = fpb_pack4 records.
 * fpb_hex_gradient_rows: out[k * nnz + j] = B_k (overwritten, or added when
 *   accumulate) for the rows listed —
 *   canonical rows (interior box pattern, fpb_hex_canon_slots[m][d] = CSR
 *   offset of relative corner d of incidence m): canon_rows[ncanon],
 *   canon_inc8[8][ncanon] element ids in incidence order;
 *   generic rows in blocks of 32: gblk_rows[ngblocks][32] (row or -1),
 *   ginc[ngblocks][maxinc][32] (element id or -1), gslot[ngblocks][maxinc][32]
 *   (uint2 relative-corner slot bytes: byte 0 = corner sign bits p of the
 *   row's node, byte d = off-diagonal slot of corner p ^ d).
 *   box_nx, box_ny > 0: the mesh is the generator's hex box with nx x ny
 *   cells per layer and every canonical row's canon_inc8 equals
 *   (i-1+mx) + nx ((j-1+my) + ny (k-1+mz)) (the caller verified it): the
 *   kernel computes the element ids instead of reading canon_inc8. */
int fpb_hex_canon_slots(int32_t* slots_h /* [8][8] */);
int fpb_hex_gradient_h(int64_t nelem, const int32_t* conn, const double* xyz4, double* H, void* stream);
int fpb_hex_gradient_rows(int32_t ncanon, const int32_t* canon_rows, const int32_t* canon_inc8, int32_t ngblocks,
                          int maxinc, int rowcap, const int32_t* gblk_rows, const int32_t* ginc,
                          const uint32_t* gslot, const double* H, int64_t nelem, const int32_t* rowptr,
                          const int32_t* colind, int64_t nnz, int accumulate, double* out, int box_nx, int box_ny,
                          void* stream);

/* ---- multi-GPU: NCCL halo sum and allreduce (halo.cu) ----
 * The compiled entry points of the z-slab decomposition.  NCCL is loaded at
 * run time (libnccl.so.2).  A caller creates one communicator per rank:
 * rank 0 calls fpb_nccl_unique_id, broadcasts the 128 bytes out of band,
 * every rank calls fpb_nccl_comm_init (device = its CUDA device).
 * fpb_halo_sum: for each segment i, x[offsets[i] .. + counts[i]) is sent to
 *   peers[i] and the peer's matching segment (same order on both sides) is
 *   received and ADDED (scratch: sum(counts) doubles); nseg <= 16.  Replaces
 *   distributed.halo_sum_nodes / halo_sum_rows's torch.distributed exchange.
 * fpb_halo_exchange: general form — segment i sends x[send_off[i] ..) and
 *   receives the peer's into x[recv_off[i] ..), added (add = 1, through
 *   scratch) or copied in place (add = 0: distributed.refresh_ghosts).
 * fpb_allreduce_sum: in-place SUM of count doubles across the ranks (dots).
 * All stream-ordered and CUDA-graph capturable. */
int fpb_nccl_unique_id(unsigned char* id128);
int fpb_nccl_comm_init(int nranks, int rank, const unsigned char* id128, int device, void** comm);
int fpb_nccl_comm_destroy(void* comm);
int fpb_halo_sum(void* comm, int nseg, const int32_t* peers, const int64_t* offsets, const int64_t* counts,
                 double* x, double* scratch, void* stream);
int fpb_halo_exchange(void* comm, int nseg, const int32_t* peers, const int64_t* send_off, const int64_t* recv_off,
                      const int64_t* counts, int add, double* x, double* scratch, void* stream);
int fpb_allreduce_sum(void* comm, double* x, int64_t count, void* stream);

/* Element-local contributions without a scatter, replacing the reference's
 * assemble_element_scalar / assemble_element_packed (assembly.py:296-380).
 * lane_conn[npacks][nn][vs] (vs = 1: conn[nelem][nn]); out in the reference's
 * layout at the same vs — matrix kinds [p][i][j][v], MOMENTUM_RHS [p][a][k][v],
 * SCALAR_RHS [p][a][v]; padded lanes are not written (caller zero-fills).
 * Kinds: FPB_MASS .. FPB_SCALAR_RHS. */
int fpb_assemble_elements(int kind, int etype, int64_t nelem, int vs, const int32_t* lane_conn,
                          const double* coords, const double* vel, const double* phi, double rho,
                          double mu, double kappa, double* out, void* stream);

/* 32-byte node records for 256-bit loads: rec[i] = (a[i][0..dim), 0.., extra[i]
 * or 0); rec must be 32-byte aligned.  Coordinates are packed once per mesh,
 * velocity (+ the transported scalar in the 4th slot) once per call. */
int fpb_pack4(int64_t n, int dim, const double* a, const double* extra, double* rec, void* stream);

/* ---- row-owned assembly for affine simplices (TRI03, TET04) -------------
 * Each CSR row / node is owned by one thread that walks its incident
 * elements in ascending order and writes its outputs once: no atomics, no
 * zero fill, bitwise reproducible (see rows.cu).  Incidence lists are SELL-32:
 * slice s = rows [32s, 32s+32) holds columns [slice_ptr[s], slice_ptr[s+1]),
 * entry (m, lane) at inc[32 m + lane] (element id, -1 padding).
 *
 * fpb_incidence_build: slice_ptr[ceil(n/32)+1]; with inc == NULL only sizes
 * (returns the column count through ncols_h, synchronous); otherwise also
 * fills inc[32 * ncols].
 * fpb_incidence_nodes: incn[32 * ncols][4] = node ids of each entry's element,
 * rotated by an even permutation so the row's own node is first (XOR with
 * its local index for tets, rotation for triangles; orientation and det
 * are unchanged), -1 padding.  The hot loop reads these instead of inc.
 * fpb_incidence_slots: for matrices, slots[32 * ncols] packs one byte per
 * node of the rotated record: byte 0 = offset of the diagonal in the row's
 * column list, bytes 1.. = offsets with the diagonal skipped (the kernel
 * keeps the diagonal in registers); returns the longest row through
 * rowcap_h (synchronous).
 * Row windows: only rows [row0, row1) are assembled (row0 a multiple of 32,
 * row1 <= n; 0, n = all) — e.g. interface rows first so a halo exchange
 * can overlap the interior (distributed.py).
 * fpb_assemble_rows: element nodes come from incn (required; inc and conn
 * are accepted for ABI stability and unused); node data come as 32-byte
 * records (fpb_pack4): xyz4[n] = (x, y, z|0, 0), uvw4[n] = (u, v, w|0,
 * phi|0); out is overwritten (accumulate = 0) or added to (accumulate = 1);
 * layouts of out
 * as in fpb_assemble. */
int fpb_incidence_build(int32_t n, int64_t nelem, int nn, const int32_t* conn, int32_t* slice_ptr,
                        int32_t* inc, int64_t* ncols_h, void* stream);
int fpb_incidence_slots(int32_t n, int nn, int64_t ncols, const int32_t* slice_ptr,
                        const int32_t* inc, const int32_t* conn, const int32_t* rowptr,
                        const int32_t* colind, uint32_t* slots, int* rowcap_h, void* stream);
int fpb_incidence_nodes(int32_t n, int64_t ncols, int nn, const int32_t* slice_ptr, const int32_t* inc,
                        const int32_t* conn, int32_t* incn, void* stream);
int fpb_assemble_rows(int kind, int etype, int32_t n, int32_t row0, int32_t row1, const int32_t* slice_ptr,
                      const int32_t* inc,
                      const int32_t* conn, const int32_t* incn, const uint32_t* slots, const double* xyz4,
                      const double* uvw4, double rho, double mu, double kappa, const int32_t* rowptr,
                      const int32_t* colind, int64_t nnz, int rowcap, int accumulate, double* out, void* stream);

/* ---- TET04 continuity matrices by column pairs (pairs.cu) --------------
 * B_x, B_y, B_z (FPB_GRADIENT_XYZ) with one register sum per CSR column:
 * every row walks a stream of (q, r) edge-vector slot pairs sorted by
 * target column (det grad N_j = e_q x e_r for the tets on edge ij) instead
 * of accumulating each incidence into three columns in shared memory.
 * fpb_pair_stream_build from the incidence slices and slot words
 * (fpb_incidence_slots): call 1 (words = NULL) fills pair_ptr[nslices + 1]
 * (stream words per row of each 32-row slice, prefix-summed) and *total_h;
 * call 2 fills words[total * 32] (uint16).  FPB_ECONFIG for rows over 128
 * entries or 64 incidences — callers then use fpb_assemble_rows. */
int fpb_pair_stream_build(int32_t n, const int32_t* slice_ptr, const uint32_t* slots, const int32_t* rowptr,
                          int64_t* pair_ptr, uint16_t* words, int64_t* total_h, void* stream);
int fpb_assemble_gradient_pairs(int32_t n, int32_t row0, int32_t row1, const int64_t* pair_ptr,
                                const uint16_t* words, const double* xyz4, const int32_t* rowptr,
                                const int32_t* colind, int64_t nnz, int rowcap, int accumulate, double* out,
                                void* stream);

/* Slice-list form of the pair-stream kernel: rows of the 32-row slices
 * slist[nslices].  canon_len > 0:
 * every row of those slices has the same stream, uploaded once with
 * fpb_pair_canon_set (even length <= 512) and read from constant memory
 * (pair_ptr / words unused); canon_len = 0: the per-slice stream as in
 * fpb_assemble_gradient_pairs. */
int fpb_pair_canon_set(const uint16_t* words_h, int len);
int fpb_assemble_gradient_pairs_slices(int32_t n, int32_t nslices, const int32_t* slist, int canon_len,
                                       const int64_t* pair_ptr, const uint16_t* words,
                                       const double* xyz4, const int32_t* rowptr, const int32_t* colind, int64_t nnz,
                                       int rowcap, int accumulate, double* out, void* stream);
/* The compile-time stream of an interior Kuhn-box row (72 words; returns the
 * count) and the kernel that uses it on the listed rows rows[nrows] (any
 * order; 32 per warp): every listed row must have that stream and 15 entries
 * with the diagonal at CSR offset 7 (the caller verifies both).  rlos[nrows]
 * (row starts) and nbr[14][nrows] (off-diagonal columns in CSR order) are
 * optional precomputed copies that shorten the load chain (NULL: read
 * through rowptr / colind). */
int fpb_pair_kuhn_table(uint16_t* words_h);
/* The per-row stream for an arbitrary row list rows[nrows] (the rows the
 * Kuhn kernel does not take): each row reads its own slice's stream. */
int fpb_assemble_gradient_pairs_rows(int32_t n, int32_t nrows, const int32_t* rows, const int64_t* pair_ptr,
                                     const uint16_t* words, const double* xyz4, const int32_t* rowptr,
                                     const int32_t* colind, int64_t nnz, int rowcap, int accumulate, double* out,
                                     void* stream);
int fpb_assemble_gradient_pairs_kuhn(int32_t nrows, const int32_t* rows, const int32_t* rlos, const int32_t* nbr,
                                     const double* xyz4, const int32_t* rowptr, const int32_t* colind, int64_t nnz,
                                     int accumulate, double* out, void* stream);
/* Same rows on the generator's Kuhn box (nx x ny cells per layer; the
 * connectivity checked equal to generate_box_mesh's, assembly.py KuhnBox):
 * the canonical rows are exactly the interior nodes (nrows = (nx-1)(ny-1)
 * (nz-1), the caller checks the count), so row ids and the 14 neighbours'
 * ids are computed — neither rows nor colind is read (rows may be NULL). */
int fpb_assemble_gradient_pairs_kuhn_box(int32_t nrows, const int32_t* rows, int nx, int ny, const double* xyz4,
                                         const int32_t* rowptr, int64_t nnz, int accumulate, double* out,
                                         void* stream);
/* The boundary (non-canonical) rows of the same Kuhn box (nx x ny x nz
 * cells): each row keeps the interior stream's words whose tet lies in a
 * cell inside the box; CSR slots by popcount of the present neighbours.
 * Only cells of layers [vk0, vk1) contribute values (a z-slab's own layers;
 * 0, nz for the whole box).  rows: the node ids (any order). */
int fpb_assemble_gradient_kuhn_boundary(int32_t nrows, const int32_t* rows, int nx, int ny, int nz, int vk0,
                                        int vk1, const double* xyz4, const int32_t* rowptr, int64_t nnz,
                                        int accumulate, double* out, void* stream);
/* Interior node lines (i in 1..nx-1, j in 1..ny-1) of node planes [kz0, kz1]
 * (1 <= kz0, kz1 <= nz-1) of the Kuhn box: every incident tet is integrated
 * (z-marching, staged coordinates); fpb_assemble_gradient_pairs_kuhn_box is
 * this with planes [1, nz-1]. */
int fpb_assemble_gradient_kuhn_lines(int nx, int ny, int nz, int kz0, int kz1, const double* xyz4,
                                     const int32_t* rowptr, int64_t nnz, int accumulate, double* out, void* stream);

/* ---- row-owned assembly for Gauss-loop elements (QUAD04, PYR05, HEX08) --
 * Matrix kinds only (rowsq.cu).  Incidence lists as for the simplices
 * (fpb_incidence_build, element ids); fpb_incidence_slots8 fills
 * slots[2 * 32 * ncols] (one uint2 per entry): byte b = 0xff for the row's
 * own node, else node b's offset in the row's column list with the diagonal
 * skipped; missing pairs -> FPB_EPATTERN; longest row through rowcap_h
 * (synchronous).  fpb_assemble_rows_gl overwrites (accumulate = 0) or adds
 * to (1) out (FPB_GRADIENT_XYZ: dim arrays of nnz); each row thread
 * evaluates its incident elements' Gauss loops itself — no atomics, bitwise
 * reproducible. */
int fpb_incidence_slots8(int32_t n, int nn, int64_t ncols, const int32_t* slice_ptr, const int32_t* inc,
                         const int32_t* conn, const int32_t* rowptr, const int32_t* colind, uint32_t* slots,
                         int* rowcap_h, void* stream);
int fpb_assemble_rows_gl(int kind, int etype, int32_t n, int32_t row0, int32_t row1, const int32_t* slice_ptr,
                         const int32_t* inc,
                         const int32_t* conn, const uint32_t* slots, const double* xyz4, const double* uvw4,
                         const int32_t* rowptr, const int32_t* colind, int64_t nnz, int rowcap, int accumulate,
                         double* out, void* stream);

/* ---- element-block RHS assembly (deterministic, atomic-free) ------------
 * Blocks of fpb_block_elems(etype) consecutive elements (256 for the affine
 * simplices, integrated two per thread; 128 for Gauss-loop types); phase 1
 * integrates each
 * element once and reduces inside the block (sorted gather lists), phase 2
 * sums the per-(block, node) partials per node in ascending block order.
 * fpb_blocks_build: with blk_nodes == NULL fills blk_ptr[nblocks+1] and
 * returns the partial count P through npartial_h (synchronous); otherwise
 * and the largest block's distinct-node count through maxnu_h; otherwise
 * (npartial_h holding P) fills blk_nodes[P], blk_gptr[P + nblocks],
 * blk_gslot and blk_lidx [nblocks * block_elems * nn], node_pptr[n+1],
 * node_plist[P].  Phase 1 stages each block's distinct nodes through shared
 * memory (blk_lidx = local node of every element slot).
 * fpb_assemble_blocks: kind MOMENTUM_RHS or SCALAR_RHS; coordinates as
 * 32-byte records (fpb_pack4); velocity (+ scalar) either as records uvw4
 * or, with uvw4 = NULL, straight from the caller's vel[n][dim] (+ phi[n]) —
 * no packing pass; partial[P * nv] is scratch; out overwritten
 * (accumulate = 0) or added to.  Windows: phase 1 integrates blocks
 * [blk0, blk1), phase 2 sums the partials of nodes [node0, node1) — the
 * full call is (0, nblocks) and (0, n); a node's partials must all have
 * been integrated before its phase 2 (interface-first schedules,
 * distributed.py). */
int fpb_block_elems(int etype);
int fpb_blocks_build(int etype, int64_t nelem, const int32_t* conn, int32_t n, int32_t* blk_ptr,
                     int32_t* blk_nodes, uint16_t* blk_gptr, uint16_t* blk_gslot, uint16_t* blk_lidx,
                     int32_t* node_pptr, int32_t* node_plist, int64_t* npartial_h, int* maxnu_h,
                     void* stream);
int fpb_assemble_blocks(int kind, int etype, int64_t nelem, int64_t blk0, int64_t blk1, const double* xyz4,
                        const double* uvw4, const double* vel, const double* phi, double rho, double mu, double kappa,
                        const int32_t* blk_ptr, const int32_t* blk_nodes, const uint16_t* blk_gptr,
                        const uint16_t* blk_gslot, const uint16_t* blk_lidx, int maxnu, double* partial, int32_t n,
                        int32_t node0, int32_t node1, const int32_t* node_pptr, const int32_t* node_plist,
                        int accumulate, double* out, void* stream);

/* Three scalar-transport RHS sharing one velocity in one element-block pass
 * (enthalpy + two species, timeloop.py:76-79, :361-363; BASELINE config 3):
 * phi3 / out3 are [3][n] (field-major), kappa_f the diffusivity of field f;
 * each field's RHS equals fpb_assemble_blocks(FPB_SCALAR_RHS, ..., kappa_f)
 * to rounding.  Staging, geometry and the velocity moments are shared;
 * partial holds 3 doubles per (block, node). */
int fpb_assemble_blocks_scalar3(int etype, int64_t nelem, int64_t blk0, int64_t blk1, const double* xyz4,
                                const double* vel, const double* phi3, double kappa0, double kappa1, double kappa2,
                                const int32_t* blk_ptr, const int32_t* blk_nodes, const uint16_t* blk_gptr,
                                const uint16_t* blk_gslot, const uint16_t* blk_lidx, int maxnu, double* partial,
                                int32_t n, int32_t node0, int32_t node1, const int32_t* node_pptr,
                                const int32_t* node_plist, int accumulate, double* out3, void* stream);

/* Momentum RHS of a Kuhn box mesh (reference momentum_rhs_packed,
 * _kernels.py:320-382, + scatter_vector_dim_packed :511-519, as driven by
 * AssemblyContext.assemble_rhs, assembly.py:235-270) when the TET04
 * connectivity is exactly generate_box_mesh(TET04, nx, ny, nz)'s
 * (mesh.py:258-282; the caller checks it, e.g. against fpb_box_conn).
 * Coordinates (32-byte records, fpb_pack4) and vel[n][3] are read as given.
 * 32 x 8 cell pencils march z-chunks of kchunk cell layers; out[n][3] is
 * overwritten in a fixed summation order (bitwise reproducible).  Only the
 * cell layers [kc0, kc1) are integrated (a z-slab's own layers; 0, nz for
 * the whole box); node planes outside [kc0, kc1] are zeroed.  scratch:
 * fpb_kuhn_mom_scratch_len(nx, ny, nz) doubles (CTA boundary partials). */
int64_t fpb_kuhn_mom_scratch_len(int nx, int ny, int nz);
int fpb_assemble_momentum_kuhn(int nx, int ny, int nz, int kc0, int kc1, int kchunk, const double* xyz4,
                               const double* vel, double rho, double mu, double* scratch, double* out,
                               void* stream);
/* The three scalar-transport RHS of config 3 (enthalpy + two species,
 * scalar_rhs_packed, _kernels.py:420-461, one velocity) on the same Kuhn box
 * in one pass: phi3 / out3 are [3][fstride] (field-major), kappa_f the
 * diffusivity of field f; same pencils, layer range and scratch. */
int fpb_assemble_scalar3_kuhn(int nx, int ny, int nz, int kc0, int kc1, int kchunk, const double* xyz4,
                              const double* vel, const double* phi3, int64_t fstride, double kappa0, double kappa1,
                              double kappa2, double* scratch, double* out3, void* stream);
/* The same pencils on the generator's HEX08 box (one Q1 hex per cell,
 * generate_box_mesh(HEX08, nx, ny, nz), mesh.py:265-267; the caller checks
 * the connectivity against fpb_box_conn): kind FPB_MOMENTUM_RHS (out[n][3],
 * rho, mu; phi3 NULL) or 101 = the three scalars (phi3 / out[3][fstride],
 * diffusivities rho, mu, kappa), momentum_rhs_packed / scalar_rhs_packed
 * (_kernels.py:320-382, :420-461) through the Walsh forms of elemcore.cuh. */
int fpb_assemble_rhs_hexbox(int kind, int nx, int ny, int nz, int kc0, int kc1, int kchunk, const double* xyz4,
                            const double* vel, const double* phi3, int64_t fstride, double rho, double mu,
                            double kappa, double* scratch, double* out, void* stream);

/* ---- solver vector kernels (sparse.py:78-130, krylov.py) -------------- */

/* y = A x (sparse.py:78-84).  nnz = rowptr[n] sizes the lanes per row. */
int fpb_spmv(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
             const double* vals, const double* x, double* y, void* stream);
/* SELL-32 copy of a CSR matrix for the solver kernels (one thread per row,
 * coalesced loads, the reference's summation order and rounding).  Call 1
 * (scol = sval = NULL): sell_ptr[nslices + 1] slice offsets, *total_h =
 * sell_ptr[nslices] (entries incl. padding) and, if maxoff_h, the largest
 * |col - row| (needs colind).  Call 2: fills scol and / or sval [total]
 * (either may be NULL: pattern and values are separable); scol holds int32
 * columns, or with idx16 int16 offsets col - row (requires maxoff < 32768;
 * 10 instead of 12 bytes per entry). */
int fpb_sell_build(int32_t n, const int32_t* rowptr, const int32_t* colind, const double* vals, int64_t* sell_ptr,
                   void* scol, int idx16, double* sval, int64_t* total_h, int32_t* maxoff_h, void* stream);
/* y = A x on the SELL-32 copy; bit-identical to sparse.py:80-84 */
int fpb_spmv_sell(int32_t n, const int64_t* sell_ptr, const void* scol, int idx16, const double* sval,
                  const double* x, double* y, void* stream);
/* out = alpha*x + y (sparse.py:96-99) */
int fpb_axpy(int64_t n, double alpha, const double* x, const double* y, double* out,
             void* stream);
/* result[0] = sum x_i y_i, deterministic fixed-order two-level reduction.
 * work must hold fpb_dot_work_size() doubles. */
int64_t fpb_dot_work_size(void);
int fpb_dot(int64_t n, const double* x, const double* y, double* result, double* work,
            void* stream);
/* d[i] = stored diagonal of row i or 0 (sparse.py:48-56) */
int fpb_diagonal(int32_t n, const int32_t* rowptr, const int32_t* colind, const double* vals,
                 double* d, void* stream);
/* row sums: lumped[i] = sum_k vals[k], k in row i (timeloop.py:174-181) */
int fpb_row_sums(int32_t n, const int32_t* rowptr, const double* vals, double* out, void* stream);

/* ---- device-resident Jacobi-PCG (krylov.py:27-89) ----------------------
 * One call runs up to `iters` iterations of the reference recurrence with
 * every scalar kept on the device.  state[] (device, 8 doubles) carries
 * {rz, bnorm, tol, status, iterations, relres, pq, spare}; status 0 =
 * running, 1 = converged, 2 = breakdown (pq <= 0).  hist[] receives relres
 * per completed iteration at hist[iterations % hist_cap] (fpb_pcg_init
 * writes hist[0]); launch arguments are the same for every batch, so a
 * batch can be captured once in a CUDA graph and replayed.  Once status != 0 the
 * remaining iterations are no-ops, so batches can be launched without a host
 * round trip per iteration.  vectors: x, r, p, q, z and the Jacobi diagonal d
 * (z = r / d, krylov.py:65,84), all of length n; nnz picks the lanes per
 * row of the fused CSR SpMV.  sell_ptr / scol / sval / sell_idx16
 * (fpb_sell_build; sell_ptr NULL = CSR): the fused SpMVs run on the SELL-32
 * copy instead (one thread per row, the reference's per-row summation
 * order). */
int fpb_pcg_init(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind, const double* vals,
                 const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16, const double* b, const double* x0, double* x, double* r, double* p,
                 double* z, const double* d, double* state, double* hist, double tol,
                 double* work, void* stream);
int fpb_pcg_iterate(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
                    const double* vals, const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16, double* x, double* r, double* p, double* q, double* z,
                    const double* d, double* state, double* hist, int64_t hist_cap, int iters,
                    double* work, void* stream);

/* ---- device-resident Jacobi-BiCGSTAB (BASELINE config 5) ----------------
 * Not in the reference: the van der Vorst
 * recurrence as scipy.sparse.linalg.bicgstab states it, operation for
 * operation (rtilde = r0; p = r + beta (p - omega v); phat = p / d;
 * v = A phat; alpha = rho / (rtilde, v); s = r - alpha v; shat = s / d;
 * t = A shat; omega = (t, s) / (t, t); x += alpha phat; x += omega shat;
 * r = s - omega t; stop when ||r|| < tol ||b||, or ||s|| < tol ||b|| after
 * the half step).  d = NULL runs unpreconditioned.  state[] holds
 * fpb_bicgstab_state_size() doubles: [0] rho, [1] rho_prev, [2] alpha,
 * [3] omega, [4] ||b||, [5] tol ||b||, [6] status (0 running, 1 converged,
 * 2 rho breakdown, 3 (rtilde, v) = 0, 4 omega breakdown), [7] iterations,
 * [8] ||r|| / ||b||.  Five fused kernels per iteration; iterations after
 * status != 0 are no-ops, so batches need no host round trip and replay
 * from a CUDA graph like the PCG's.  sell_ptr / scol / sval / sell_idx16 as
 * for the PCG. */
int fpb_bicgstab_state_size(void);
/* x = x0 | 0, r = rtilde = b - A x0 | b, p = v = 0; reductions over the
 * owned rows [own_lo, own_hi) (0, n on one GPU).  defer = 0 finishes the
 * scalars on the device; defer = 1 leaves {||b||^2, ||r||^2} (partial, this
 * rank) in state[16..17] for an allreduce followed by fpb_bicgstab_finish(0). */
int fpb_bicgstab_init(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind, const double* vals,
                      const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16, const double* b, const double* x0, double* x, double* r, double* rt, double* p, double* v,
                      double* state, double* hist, double tol, int64_t own_lo, int64_t own_hi, int defer,
                      double* work, void* stream);
/* `iters` whole iterations on one GPU (all rows owned, scalars on device). */
int fpb_bicgstab_iterate(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
                         const double* vals, const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16,
                         const double* d, double* x, double* r, const double* rt, double* p,
                         double* ph, double* v, double* sv, double* sh, double* t, double* state, double* hist,
                         int64_t hist_cap, int iters, double* work, void* stream);
/* One reduction step of an iteration, for domain decomposition: step 1 =
 * direction + v = A phat with (rtilde, v); 2 = s, shat with ||s||^2; 3 =
 * t = A shat with (t, s), (t, t); 4 = x, r update with ||r||^2, (rtilde, r).
 * With defer = 1 the partial sums land in state[16..17] (step 2's ||s||^2
 * in state[18], so it can ride on step 3's reduction); the caller allreduces
 * them (and refreshes ghost entries of v / t after steps 1 / 3) before
 * fpb_bicgstab_finish(step) — finish(2) then finish(3) after step 3. */
int fpb_bicgstab_step(int step, int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
                      const double* vals, const int64_t* sell_ptr, const void* scol, const double* sval, int sell_idx16,
                      const double* d, double* x, double* r, const double* rt, double* p,
                      double* ph, double* v, double* sv, double* sh, double* t, double* state, double* hist,
                      int64_t hist_cap, int64_t own_lo, int64_t own_hi, int defer, double* work, void* stream);
int fpb_bicgstab_finish(int step, double* state, double* hist, int64_t hist_cap, double tol, void* stream);

/* ---- time-loop support (flow.cu) --------------
 * Pressure-operator setup on the device, each mirroring a reference routine:
 *   fpb_csr_transpose      transpose_csr (sparse.py:133-138); trowptr[n+1]
 *   fpb_spgemm_count/fill  spgemm (sparse.py:141-188): counts[n] per row,
 *                          then colind/vals at the caller's rowptr (exclusive
 *                          scan of counts); values summed in the reference's
 *                          product order (bitwise equal)
 *   fpb_scale_rows         A.vals * d[rows] (normal_product, sparse.py:191-194)
 *   fpb_csr_add_count/fill csr_add (sparse.py:197-214), union of patterns
 *   fpb_apply_dirichlet    apply_dirichlet (sparse.py:219-254): flag[n] (1 =
 *                          constrained), lift[n] = values on constrained
 *                          nodes; b (nullable) updated in place
 *   fpb_robin              assemble_boundary (assembly.py:383-411) for one
 *                          face group: face rule N[nnf][ng], dN[dim-1][nnf][ng],
 *                          wts[ng]; vals (via the face->CSR map pos) and rhs
 *                          accumulated
 * FlowSolver.step stages (timeloop.py:367-440), numpy rounding order:
 *   fpb_stage_momentum  un = a u0 + b (uc + dt_rho ((r [+ load - Ru_k] - grad_p) / lumped))
 *                       (u0, uc, r, grad_p, un: [n][dim]; Ru: [dim][n])
 *   fpb_stage_scalar    sn = a phi0 + b (phi + dt (rs / lumped))
 *   fpb_set_rows        u[nodes[q]][:] = values[q][:] (values NULL -> 0)
 *   fpb_sub_into        div -= s; g = scale * div when g != NULL
 *   fpb_correct         un[:, k] = uc[:, k] - dt_rho * (dflag ? 0 : s / lumped) */
int fpb_csr_transpose(int32_t n, int64_t nnz, const int32_t* rowptr, const int32_t* colind, const double* vals,
                      int32_t* trowptr, int32_t* tcolind, double* tvals, void* stream);
int fpb_spgemm_count(int32_t n, const int32_t* arp, const int32_t* aci, const int32_t* brp, const int32_t* bci,
                     int32_t* counts, void* stream);
int fpb_spgemm_fill(int32_t n, const int32_t* arp, const int32_t* aci, const double* av, const int32_t* brp,
                    const int32_t* bci, const double* bv, const int32_t* rowptr, int32_t* colind, double* vals,
                    void* stream);
int fpb_scale_rows(int32_t n, const int32_t* rowptr, const double* vals, const double* d, double* out,
                   void* stream);
int fpb_csr_add_count(int32_t n, const int32_t* arp, const int32_t* aci, const int32_t* brp, const int32_t* bci,
                      int32_t* counts, void* stream);
int fpb_csr_add_fill(int32_t n, const int32_t* arp, const int32_t* aci, const double* av, const int32_t* brp,
                     const int32_t* bci, const double* bv, const int32_t* rowptr, int32_t* colind, double* vals,
                     void* stream);
int fpb_apply_dirichlet(int32_t n, const int32_t* rowptr, const int32_t* colind, const double* vals,
                        const uint8_t* flag, const double* lift, double* out, double* b, void* stream);
int fpb_robin(int64_t nf, int nnf, int ng, int dim, const int32_t* conn, const double* coords, const double* N,
              const double* dN, const double* wts, const int32_t* pos, double alpha, double beta, double* vals,
              double* rhs, void* stream);
int fpb_stage_momentum(int64_t n, int dim, double a, double b, double dt_rho, const double* u0, const double* uc,
                       const double* r, const double* grad_p, const double* lumped, const double* load,
                       const double* Ru, double* un, void* stream);
int fpb_stage_scalar(int64_t n, double a, double b, double dt, const double* phi0, const double* phi,
                     const double* rs, const double* lumped, double* sn, void* stream);
int fpb_set_rows(int64_t m, int dim, const int64_t* nodes, const double* values, double* u, void* stream);
int fpb_sub_into(int64_t n, const double* s, double* div, double scale, double* g, void* stream);
int fpb_correct(int64_t n, int dim, int k, double dt_rho, const double* s, const double* lumped,
                const uint8_t* dflag, const double* uc, double* un, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FEMPACK_B200_H */
