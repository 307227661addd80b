"""B200-native FE assembly + solver vector path of arXiv 2107.11541.

Drop-in for the reference mini-app `fempack`'s hot path: `AssemblyContext`
(assemble_matrix / assemble_rhs), `sparse.spmv/axpy/dot/norm2` and
`krylov.pcg_solve` / `bicgstab_solve`, plus the setup they need (box meshes,
packs, CSR graph, element->CSR map), the Robin boundary, the pressure-operator
setup and the `FlowSolver` time loop built on them, all running as
hand-written sm_100a kernels behind the C ABI in include/fempack_b200.h.
See DESIGN.md.
"""

__version__ = "0.1.0"

from .assembly import (AssemblyContext, KernelKind, assemble_boundary, assemble_element_packed,
                       assemble_element_scalar, gradient_matrices, lumped_mass, matrix_positions)
from .elements import (ElementGeometry, ElementType, FaceRule, ReferenceElement, compute_geometry, face_rule,
                       integrate_reference_monomial, reference_element)
from .errors import (ChecksumMismatchError, ConfigurationError, InvertedElementError,
                     ScatterPatternError, SolverBreakdownError, StepFailureError)
from .krylov import SolverStats, bicgstab_solve, pcg_solve
from .mesh import (ElementGroup, FaceGroup, Mesh, extract_boundary, generate_box_mesh, generate_mixed_mesh,
                   renumber_by_type)
from .packing import PackConfig, PackSet, build_packs, pack_array, unpack_array
from .sparse import (CsrMatrix, apply_dirichlet, axpy, build_node_pattern, csr_add, dot, norm2, normal_product,
                     spgemm, spmv, transpose_csr)
from .timeloop import (FlowSolver, FlowState, StepDiagnostics, TimeConfig, integrate_ode, preassemble_laplacian,
                       preset_state, pressure_poisson, ssp_rk3_step)

__all__ = [
    "AssemblyContext", "KernelKind", "assemble_boundary", "assemble_element_packed", "assemble_element_scalar",
    "gradient_matrices", "lumped_mass", "matrix_positions",
    "ElementGeometry", "ElementType", "FaceRule", "ReferenceElement", "compute_geometry", "face_rule",
    "integrate_reference_monomial", "reference_element",
    "ChecksumMismatchError", "ConfigurationError", "InvertedElementError", "ScatterPatternError",
    "SolverBreakdownError", "StepFailureError",
    "SolverStats", "pcg_solve", "bicgstab_solve",
    "ElementGroup", "FaceGroup", "Mesh", "extract_boundary", "generate_box_mesh", "generate_mixed_mesh",
    "renumber_by_type",
    "PackConfig", "PackSet", "build_packs", "pack_array", "unpack_array",
    "CsrMatrix", "axpy", "build_node_pattern", "dot", "norm2", "spmv",
    "apply_dirichlet", "csr_add", "normal_product", "spgemm", "transpose_csr",
    "FlowSolver", "FlowState", "StepDiagnostics", "TimeConfig", "preassemble_laplacian", "preset_state",
    "pressure_poisson", "integrate_ode", "ssp_rk3_step",
]
