"""B200-native FE assembly + solver vector path of arXiv 2107.11541.

Drop-in for the reference mini-app `fempack`'s hot path: `AssemblyContext`
(assemble_matrix / assemble_rhs), `sparse.spmv/axpy/dot/norm2` and
`krylov.pcg_solve`, plus the setup they need (box meshes, packs, CSR graph,
element->CSR map), all running as hand-written sm_100a kernels behind the C
ABI in include/fempack_b200.h.  See DESIGN.md.
"""

__version__ = "0.1.0"

from .assembly import AssemblyContext, KernelKind, gradient_matrices, lumped_mass, matrix_positions
from .elements import ElementType, ReferenceElement, reference_element
from .errors import (ChecksumMismatchError, ConfigurationError, InvertedElementError,
                     ScatterPatternError, SolverBreakdownError, StepFailureError)
from .krylov import SolverStats, bicgstab_solve, pcg_solve
from .mesh import ElementGroup, Mesh, generate_box_mesh, generate_mixed_mesh, renumber_by_type
from .packing import PackConfig, PackSet, build_packs
from .sparse import CsrMatrix, axpy, build_node_pattern, dot, norm2, spmv

__all__ = [
    "AssemblyContext", "KernelKind", "gradient_matrices", "lumped_mass", "matrix_positions",
    "ElementType", "ReferenceElement", "reference_element",
    "ChecksumMismatchError", "ConfigurationError", "InvertedElementError", "ScatterPatternError",
    "SolverBreakdownError", "StepFailureError",
    "SolverStats", "pcg_solve", "bicgstab_solve",
    "ElementGroup", "Mesh", "generate_box_mesh", "generate_mixed_mesh", "renumber_by_type",
    "PackConfig", "PackSet", "build_packs",
    "CsrMatrix", "axpy", "build_node_pattern", "dot", "norm2", "spmv",
]
