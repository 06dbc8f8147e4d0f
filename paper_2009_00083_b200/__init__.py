"""B200-native (sm_100a) Localized Topological Simplification hot path.

Drop-in for the reference's LTS path (arXiv 2009.00083): the Python argument
surface of SPEC's engine (simplify_field / remove_extrema) and the reference's
order.py / critical.py / triangulation.py types, backed by hand-written CUDA in
liblts_sm100.so.  See DESIGN.md.
"""
from .errors import (ConstraintNotExtremum, FieldError, LocalizeError, LTSNativeError, MeshError,
                     NonManifoldEdge, NonTriangleFace, NoSaddleError, VerifyError)
from .triangulation import (Triangulation, build_explicit_triangulation, build_grid_triangulation,
                            grid_link_tables, link_adjacency, load_off, make_icosahedron, make_octahedron,
                            make_torus, write_off)
from .order import (OrderField, ScalarField, ZetaMode, ZetaPolicy, compute_order_field,
                    order_from_ranks, realize_numeric)
from .critical import (CriticalSet, Criticality, Kind, classify_all, classify_vertex,
                       extract_critical_points, extrema)
from .engine import (ConstraintSet, PassRegions, SimplifyOptions, SimplifyReport, discover_regions,
                     remove_extrema, remove_pass, simplify_field, simplify_field_host, simplify_raw,
                     verify_constraints)
from .persistence import (PersistencePairs, compute_extremum_saddle_pairs, persistence_curve,
                          persistence_simplify)

__all__ = [
    "ConstraintNotExtremum", "FieldError", "LocalizeError", "LTSNativeError", "MeshError",
    "NonManifoldEdge", "NonTriangleFace", "NoSaddleError", "VerifyError", "Triangulation",
    "build_explicit_triangulation", "build_grid_triangulation", "grid_link_tables", "link_adjacency",
    "load_off", "write_off", "make_octahedron", "make_icosahedron", "make_torus", "OrderField", "ScalarField", "ZetaMode", "ZetaPolicy", "compute_order_field",
    "order_from_ranks", "realize_numeric", "CriticalSet", "Criticality", "Kind", "classify_all", "classify_vertex",
    "extract_critical_points", "extrema", "ConstraintSet", "PassRegions", "SimplifyOptions",
    "SimplifyReport", "discover_regions", "remove_extrema", "remove_pass", "simplify_field", "simplify_field_host",
    "simplify_raw", "verify_constraints", "PersistencePairs", "compute_extremum_saddle_pairs",
    "persistence_curve", "persistence_simplify",
]
