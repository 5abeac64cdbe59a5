"""B200-native colored DG surface-integral hot path (arXiv 1601.07613).

Drop-in for the reference package ``meshchroma`` on the path the north star
names: mesh setup, fixed-palette surface coloring, color-major
renumbering, AMR split-edge colors, the Algorithm 1 sweeps — plus the DG
RHS / SSP-RK operator the reference leaves out of scope.  Names below
mirror /root/reference/pkg/src/meshchroma/__init__.py:11-99.

Host setup is numpy + native C++ (coloring); every sweep / DG evaluation
runs in hand-written sm_100a kernels through ``libmeshchroma_b200.so``
(C ABI in include/meshchroma_b200.h).  No CPU fallback exists.
"""

from .amr import (FamilyRecord, RefinedMesh, RefinementMap, child_color,
                  coarsen, max_refined_neighbors, reconstruct_refinement,
                  refine)
from .coloring import (ColoringConfig, ColoringReport, SurfaceColoring, color,
                       color_set_size, modified_greedy, naive_greedy,
                       resolve_conflicts, verify_coloring)
from .errors import (DanglingVertexError, LevelConstraintError,
                     MalformedSectionError, MeshChromaError,
                     NativeLibraryError, NonManifoldError, PartialFamilyError,
                     PlanMeshMismatchError, RestartsExhaustedError,
                     SwapBudgetExceededError, UnrefinableKindError,
                     UnsupportedVersionError, WriteConflictError)
from .generators import (FAMILIES, GeneratorSpec, gen_hybrid_rect, gen_quad_rect,
                         gen_tet_prism, gen_tri_rect, generate, shuffle_elements)
from .mesh import (ConnectivityGraph, Diagnostic, Element, ElementKind, Mesh,
                   Surface, assemble, build_surfaces, connectivity_graph,
                   validate, vizing_bound)
from .meshio import (NativeMesh, read_msh, read_native, write_native,
                     write_report)
from .reorder import (CoalescingReport, ReorderingPlan, apply_plan, build_plan,
                      coalescing_metric, invert_plan)
from .scaling import ScalingPoint, ScalingSeries, fit_loglog_slope, run_series
from .sweeps import (AccumulationState, MemoryEstimate, assert_race_free,
                     basis_count, default_payload, memory_saved,
                     surface_buffer, sweep_atomic, sweep_buffered,
                     sweep_colored, sweep_sequential)

__version__ = "0.1.0"
