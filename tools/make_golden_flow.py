"""Golden fixtures for the device time loop from the
UNMODIFIED reference (build container only).

    NUMBA_CACHE_DIR=/tmp/nc python tools/make_golden_flow.py

Writes tests/golden/flow_<case>.npz with, per case: the mesh arguments, the
boundary nodes and Robin structures (assembly.py:383-411), the lumped mass
and pinned pressure operator (timeloop.py:174-231: gradient_matrices ->
transpose_csr / normal_product / csr_add / apply_dirichlet, sparse.py:133-254),
and the state after each of two FlowSolver.step calls (timeloop.py:336-440)
with their diagnostics.  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
sys.path.insert(0, "/root/reference/pkg/src")

from fempack.assembly import assemble_boundary  # noqa: E402
from fempack.elements import ElementType  # noqa: E402
from fempack.mesh import generate_box_mesh, generate_mixed_mesh, renumber_by_type  # noqa: E402
from fempack.timeloop import FlowSolver, FlowState, TimeConfig, preset_state  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def mixed_initial(mesh):  # test_timeloop.py:318-328
    x, y, z = mesh.coords.T
    st = FlowState.zeros(mesh)
    st.velocity[:, 0] = np.sin(np.pi * x) * np.cos(np.pi * y)
    st.velocity[:, 1] = -np.cos(np.pi * x) * np.sin(np.pi * y)
    st.velocity[:, 2] = 0.1 * np.sin(np.pi * z)
    st.heat[:] = np.cos(np.pi * x) * np.cos(np.pi * z)
    st.species[0] = x * y
    st.species[1] = z * (1.0 - z)
    return st


def smooth_initial(mesh):
    st = FlowState.zeros(mesh)
    x = mesh.coords
    st.velocity[:, 0] = 0.3 * np.sin(np.pi * x[:, 1])
    st.velocity[:, 1] = 0.2 * np.cos(np.pi * x[:, 0])
    if mesh.dim == 3:
        st.velocity[:, 2] = 0.1 * x[:, 0] * x[:, 1]
    st.heat[:] = np.cos(np.pi * x[:, 0])
    st.species[0] = x[:, 0] * x[:, 1]
    st.species[1] = x[:, -1]
    return st


CASES = {
    # name: (mesh builder args, initial-state builder, solver kwargs, TimeConfig)
    "mixed": (("mixed", 4, 4, 4), "mixed", dict(robin_alpha=10.0, robin_beta=1.0), dict(dt=1e-2, tol=1e-13)),
    "tet_rest": (("box", "TET04", 3, 3, 3), "rest", {}, dict(dt=1e-2, tol=1e-12)),
    "tet_smooth": (("box", "TET04", 4, 3, 3), "smooth", dict(robin_alpha=5.0, robin_beta=0.5), dict(dt=5e-3, tol=1e-12)),
    "quad_tg": (("box", "QUAD04", 8, 8), "taylor-green-2d", {}, dict(dt=1e-2, tol=1e-12)),
    "hex_uniform": (("box", "HEX08", 3, 3, 2), "uniform", {}, dict(dt=1e-2, tol=1e-12)),
    "tri_smooth": (("box", "TRI03", 6, 5), "smooth", dict(robin_alpha=2.0), dict(dt=1e-2, tol=1e-12)),
    # interior nodes moved by up to 0.2 h (tests/test_flow.py applies the same jitter)
    "tet_jitter": (("jitter", "TET04", 5, 4, 4), "smooth", dict(robin_alpha=3.0, robin_beta=0.2), dict(dt=5e-3, tol=1e-12)),
    "hex_jitter": (("jitter", "HEX08", 4, 4, 3), "smooth", dict(robin_alpha=1.0), dict(dt=5e-3, tol=1e-12)),
}


def jitter(coords, dims, seed=3):
    """Move interior nodes by up to 0.2 h per axis (boundary nodes stay)."""
    rng = np.random.default_rng(seed)
    x = coords.copy()
    h = np.array([1.0 / d for d in dims])
    lo, hi = x.min(axis=0), x.max(axis=0)
    interior = np.all((x > lo + 1e-12) & (x < hi - 1e-12), axis=1)
    x[interior] += 0.2 * h * rng.uniform(-1.0, 1.0, size=(int(interior.sum()), x.shape[1]))
    return x


def build_mesh(spec):
    if spec[0] == "mixed":
        mesh, _ = renumber_by_type(generate_mixed_mesh(*spec[1:], fraction=0.5))
        return mesh
    mesh = generate_box_mesh(ElementType[spec[1]], *spec[2:])
    if spec[0] == "jitter":
        mesh.coords = jitter(mesh.coords, spec[2:])
    return mesh


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, (spec, init, kw, tc) in CASES.items():
        mesh = build_mesh(spec)
        if init == "mixed":
            state, extra = mixed_initial(mesh), {}
        elif init == "smooth":
            state, extra = smooth_initial(mesh), {}
        else:
            state, extra = preset_state(init, mesh)
        kw = dict(kw, **extra)
        solver = FlowSolver(mesh, TimeConfig(nsteps=2, **tc), layout="packed", **kw)
        d = {"spec": np.array([str(s) for s in spec]), "dt": tc["dt"], "tol": tc["tol"],
             "robin_alpha": kw.get("robin_alpha", 0.0), "robin_beta": kw.get("robin_beta", 0.0),
             "boundary_nodes": mesh.boundary_nodes(),
             "lumped": solver.lumped,
             "lap_rowptr": solver.laplacian.rowptr, "lap_colind": solver.laplacian.colind,
             "lap_vals": solver.laplacian.vals,
             "div0_rowptr": solver.div_mats[0].rowptr, "div0_colind": solver.div_mats[0].colind,
             "div0_vals": solver.div_mats[0].vals}
        if "dirichlet_nodes" in kw:
            d["dirichlet_nodes"] = np.asarray(kw["dirichlet_nodes"])
            d["dirichlet_values"] = np.asarray(kw["dirichlet_values"])
        a, b = kw.get("robin_alpha", 0.0), kw.get("robin_beta", 0.0)
        if a or b:
            R, load = assemble_boundary(mesh, solver.ctx.pattern, a, b)
            d["robin_vals"], d["robin_load"] = R.vals, load
        for f in ("velocity", "pressure", "heat", "species"):
            d[f"s0_{f}"] = getattr(state, f).copy()
        st = state
        for k in (1, 2):
            st, diag = solver.step(st)
            for f in ("velocity", "pressure", "heat", "species"):
                d[f"s{k}_{f}"] = getattr(st, f).copy()
            d[f"s{k}_iterations"] = diag.solver.iterations
            d[f"s{k}_div_star"] = diag.div_star
            d[f"s{k}_div_after"] = diag.div_after
            d[f"s{k}_history"] = np.asarray(diag.solver.residual_history)
        path = os.path.join(OUT, f"flow_{name}.npz")
        np.savez_compressed(path, **d)
        print(name, mesh.nnode, [d[f"s{k}_iterations"] for k in (1, 2)], os.path.getsize(path))


if __name__ == "__main__":
    main()
