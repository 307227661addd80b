"""Generate golden fixtures from the UNMODIFIED reference (build container only).

    NUMBA_CACHE_DIR=/tmp/nc python tools/make_golden.py

Imports `fempack` from /root/reference/pkg/src (read-only; numba caches go to
NUMBA_CACHE_DIR) and writes `tests/golden/<case>.npz`.  The fixtures pin both
the CPU oracle (`oracle/fempack_np.py`) and the CUDA path; nothing on the GPU
box reads /root/reference.

Every fixture is produced through the reference's public API exactly as its
bench/tests call it: `generate_box_mesh` / `generate_mixed_mesh` /
`renumber_by_type` (mesh.py), `build_packs` (packing.py),
`build_node_pattern` (sparse.py:59-75), `AssemblyContext.build` +
`assemble_matrix` / `assemble_rhs` (assembly.py:83-270), `spmv/axpy/dot`
(sparse.py:110-130), `apply_dirichlet` + `pcg_solve` (krylov.py:27-89), and
`gradient_matrices` / `lumped_mass` (timeloop.py:159-181).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
sys.path.insert(0, "/root/reference/pkg/src")

from fempack.assembly import AssemblyContext, KernelKind  # noqa: E402
from fempack.elements import ElementType, reference_element  # noqa: E402
from fempack.krylov import pcg_solve  # noqa: E402
from fempack.mesh import generate_box_mesh, generate_mixed_mesh, renumber_by_type  # noqa: E402
from fempack.packing import PackConfig, build_packs  # noqa: E402
from fempack.sparse import apply_dirichlet, axpy, build_node_pattern, dot, norm2, spmv  # noqa: E402
from fempack.timeloop import gradient_matrices, lumped_mass  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a.astype(np.int64)).tobytes()).hexdigest()


def smooth_fields(mesh):  # test_assembly.py:199-213
    x = mesh.coords
    if mesh.dim == 2:
        vel = np.stack([np.sin(x[:, 0]) + 0.2 * x[:, 1], np.cos(x[:, 1])], axis=1)
    else:
        vel = np.stack([np.sin(x[:, 0]) + 0.2 * x[:, 1], np.cos(x[:, 1]) * x[:, 2],
                        x[:, 0] * x[:, 1] + 0.5], axis=1)
    phi = np.cos(x[:, 0]) * np.sin(x[:, 1]) + x[:, -1]
    return np.ascontiguousarray(vel), np.ascontiguousarray(phi)


CASES = {
    # name: (builder, full_int_arrays, full_matrix_kinds)
    "tri_4x3": (lambda: generate_box_mesh(ElementType.TRI03, 4, 3), True, True),
    "quad_4x3": (lambda: generate_box_mesh(ElementType.QUAD04, 4, 3), True, True),
    "tet_6": (lambda: generate_box_mesh(ElementType.TET04, 6, 6, 6), True, True),
    "pyr_6": (lambda: generate_box_mesh(ElementType.PYR05, 6, 6, 6), True, True),
    "hex_8": (lambda: generate_box_mesh(ElementType.HEX08, 8, 8, 8), True, True),
    "mixed_8": (lambda: renumber_by_type(generate_mixed_mesh(8, 8, 8, fraction=0.5))[0], True, True),
    "mixed_3x2x2": (lambda: generate_mixed_mesh(3, 2, 2, fraction=0.5), True, True),
    # config 1 of BASELINE.json: 50,400 tets
    "tet_c1": (lambda: generate_box_mesh(ElementType.TET04, 20, 20, 21), False, False),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    # reference element tables (elements.py:258-274)
    tabs = {}
    for et in ElementType:
        r = reference_element(et)
        tabs[f"{et.value}_N"] = r.N
        tabs[f"{et.value}_dN"] = r.dN
        tabs[f"{et.value}_w"] = r.weights
    np.savez_compressed(os.path.join(OUT, "elements.npz"), **tabs)

    for name, (builder, full_int, full_mat) in CASES.items():
        mesh = builder()
        d = {"dim": mesh.dim, "coords": mesh.coords,
             "etypes": np.array([g.etype.value for g in mesh.groups])}
        for gi, g in enumerate(mesh.groups):
            d[f"conn{gi}"] = g.conn.astype(np.int32)
        pat = build_node_pattern(mesh)
        d["rowptr"] = pat.rowptr
        if full_int:
            d["colind"] = pat.colind.astype(np.int32)
        d["colind_sha"] = sha(pat.colind)
        for vs in (8, 32):
            ctx = AssemblyContext.build(mesh, vector_size=vs)
            for gi, gd in enumerate(ctx.groups):
                if full_int:
                    d[f"lane_conn{gi}_vs{vs}"] = gd.packset.lane_conn.astype(np.int32)
                    d[f"pos_packed{gi}_vs{vs}"] = gd.pos_packed.astype(np.int32)
                d[f"lane_conn{gi}_vs{vs}_sha"] = sha(gd.packset.lane_conn)
                d[f"pos_packed{gi}_vs{vs}_sha"] = sha(gd.pos_packed)
                d[f"pos_scalar{gi}_sha"] = sha(gd.pos_scalar)
        ctx = AssemblyContext.build(mesh, vector_size=8)
        rng = np.random.default_rng(0)  # bench.py:196-197
        vel = rng.standard_normal((mesh.nnode, mesh.dim))
        scal = [rng.standard_normal(mesh.nnode) for _ in range(3)]
        d["bench_vel"] = vel
        for s in range(3):
            d[f"bench_scalar{s}"] = scal[s]
        svel, sphi = smooth_fields(mesh)
        d["smooth_vel"], d["smooth_phi"] = svel, sphi
        # matrices, packed layout (the reference bench default)
        kinds = [("mass", KernelKind.MASS, None), ("laplacian", KernelKind.LAPLACIAN, None),
                 ("convection", KernelKind.CONVECTION, vel)]
        if not full_mat:
            kinds = [kinds[0], kinds[2]]
        for key, kind, v in kinds:
            d[f"mat_{key}"] = ctx.assemble_matrix(kind, "packed", velocity=v).vals.copy()
        d["mat_convection_smooth"] = ctx.assemble_matrix(
            KernelKind.CONVECTION, "packed", velocity=svel).vals.copy()
        d["rhs_momentum"] = ctx.assemble_rhs(KernelKind.MOMENTUM_RHS, "packed", vel, None, 1.0, 1e-2, 0.0)
        d["rhs_momentum_smooth"] = ctx.assemble_rhs(KernelKind.MOMENTUM_RHS, "packed", svel, None, 1.2, 1e-2, 0.0)
        for s in range(3):
            d[f"rhs_scalar{s}"] = ctx.assemble_rhs(KernelKind.SCALAR_RHS, "packed", vel, scal[s], 1.0, 0.0, 1e-2)
        d["rhs_scalar_smooth"] = ctx.assemble_rhs(KernelKind.SCALAR_RHS, "packed", svel, sphi, 1.0, 0.0, 0.3)
        # scalar layout too (layout equivalence is part of the contract)
        d["rhs_momentum_scalar_layout"] = ctx.assemble_rhs(
            KernelKind.MOMENTUM_RHS, "scalar", vel, None, 1.0, 1e-2, 0.0)
        # continuity: gradient matrices B_k and lumped mass (timeloop.py:159-181)
        grads = gradient_matrices(ctx, "packed")
        for k, B in enumerate(grads):
            if full_mat or k == mesh.dim - 1:
                d[f"mat_grad{k}"] = B.vals.copy()
        d["lumped_mass"] = lumped_mass(ctx, "packed")
        # vector kernels on the MASS matrix (bench.py:228-237) and bench vectors
        M = ctx.assemble_matrix(KernelKind.MASS, "packed")
        x = np.random.default_rng(1).standard_normal(mesh.nnode)
        d["spmv_x"] = x
        d["spmv_y"] = spmv(M, x)
        d["axpy_out"] = axpy(2.5, scal[0], scal[1])
        d["dot"] = np.array(dot(scal[0], scal[1]))
        d["norm2"] = np.array(norm2(scal[0]))
        # PCG on the pinned LAPLACIAN (bench.py:240-256)
        if full_mat or name == "tet_c1":
            lap = ctx.assemble_matrix(KernelKind.LAPLACIAN, "packed")
            pinned, _ = apply_dirichlet(lap, np.array([0]))
            b = np.random.default_rng(0).standard_normal(mesh.nnode)
            b[0] = 0.0
            xs, st = pcg_solve(pinned, b, tol=1e-8)
            d["cg_b"] = b
            d["cg_vals"] = pinned.vals
            d["cg_x"] = xs
            d["cg_iterations"] = np.array(st.iterations)
            d["cg_history"] = np.array(st.residual_history)
            d["cg_true_residual"] = np.array(st.true_residual)
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **d)
        print(f"{name}: nnode={mesh.nnode} nelem={mesh.nelem} nnz={pat.nnz} -> "
              f"{os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
