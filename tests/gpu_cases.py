"""Device-mesh builders matching the golden cases (tests/golden/*.npz)."""

import paper_2107_11541_b200 as P

E = P.ElementType

CASES = {
    "tri_4x3": lambda: P.generate_box_mesh(E.TRI03, 4, 3),
    "quad_4x3": lambda: P.generate_box_mesh(E.QUAD04, 4, 3),
    "tet_6": lambda: P.generate_box_mesh(E.TET04, 6, 6, 6),
    "pyr_6": lambda: P.generate_box_mesh(E.PYR05, 6, 6, 6),
    "hex_8": lambda: P.generate_box_mesh(E.HEX08, 8, 8, 8),
    "mixed_8": lambda: P.renumber_by_type(P.generate_mixed_mesh(8, 8, 8, fraction=0.5))[0],
    "mixed_3x2x2": lambda: P.generate_mixed_mesh(3, 2, 2, fraction=0.5),
    "tet_c1": lambda: P.generate_box_mesh(E.TET04, 20, 20, 21),
}
