"""Config-2 setup hashes from the UNMODIFIED reference (build container only).

    NUMBA_CACHE_DIR=/tmp/nc python tools/make_c2_hashes.py

Builds the 94x94x95 TET04 box (5,036,520 tets) with the reference's own
`generate_box_mesh` and `AssemblyContext.build(mesh, vector_size=8)`
(mesh.py:227-289, assembly.py:83-96; ~2 min, ~12 GB) and writes
tests/golden/c2_hashes.json: sha256 of coords (float64 bytes), conn,
lane_conn, CSR rowptr / colind and the element->CSR maps pos_scalar /
pos_packed (int64 bytes), plus their shapes.  tests/test_gpu_scale.py
checks the device setup against it bit for bit (SURVEY.md 8(a) a1-a4 at
full config-2 size).  Also records the reference's B_x/B_y/B_z and momentum
RHS checksums for the bench fields as a second, independent value pin.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
sys.path.insert(0, "/root/reference/pkg/src")

from fempack.assembly import AssemblyContext, KernelKind  # noqa: E402
from fempack.elements import ElementType  # noqa: E402
from fempack.mesh import generate_box_mesh  # noqa: E402
from fempack.timeloop import gradient_matrices  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c2_hashes.json")


def sha(a: np.ndarray, dtype=np.int64) -> str:
    return hashlib.sha256(np.ascontiguousarray(a.astype(dtype)).tobytes()).hexdigest()


def main():
    t0 = time.time()
    mesh = generate_box_mesh(ElementType.TET04, 94, 94, 95)
    t1 = time.time()
    ctx = AssemblyContext.build(mesh, vector_size=8)
    t2 = time.time()
    g = ctx.groups[0]
    rec = {
        "mesh": "TET04 94x94x95 unit cube (config 2)", "vector_size": 8,
        "seconds": {"generate_box_mesh": round(t1 - t0, 1), "AssemblyContext.build": round(t2 - t1, 1)},
        "shapes": {"coords": list(mesh.coords.shape), "conn": list(g.conn.shape),
                   "lane_conn": list(g.packset.lane_conn.shape), "rowptr": list(ctx.pattern.rowptr.shape),
                   "colind": list(ctx.pattern.colind.shape), "pos_scalar": list(g.pos_scalar.shape),
                   "pos_packed": list(g.pos_packed.shape)},
        "sha256": {"coords": sha(mesh.coords, np.float64), "conn": sha(g.conn),
                   "lane_conn": sha(g.packset.lane_conn), "rowptr": sha(ctx.pattern.rowptr),
                   "colind": sha(ctx.pattern.colind), "pos_scalar": sha(g.pos_scalar),
                   "pos_packed": sha(g.pos_packed)},
    }
    rng = np.random.default_rng(0)
    vel = rng.standard_normal((mesh.nnode, 3))
    r = ctx.assemble_rhs(KernelKind.MOMENTUM_RHS, "packed", velocity=vel, rho=1.0, mu=1e-2)
    grads = gradient_matrices(ctx, "packed")
    rec["values"] = {
        "momentum_rhs": {"sum_abs": float(np.abs(r).sum()), "max_abs": float(np.abs(r).max()),
                         "checksum_w": float((r * np.arange(1, r.size + 1).reshape(r.shape) / r.size).sum())},
    }
    for k, B in enumerate(grads):
        v = B.vals
        rec["values"][f"B_{'xyz'[k]}"] = {"sum_abs": float(np.abs(v).sum()), "max_abs": float(np.abs(v).max()),
                                          "checksum_w": float((v * np.arange(1, v.size + 1) / v.size).sum())}
    rec["seconds"]["total"] = round(time.time() - t0, 1)
    with open(OUT, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec["seconds"]))


if __name__ == "__main__":
    main()
