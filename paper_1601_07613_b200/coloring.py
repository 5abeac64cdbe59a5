"""Fixed-palette surface coloring (drop-in for ``meshchroma.coloring``).

API, dataclasses and error behaviour follow
/root/reference/pkg/src/meshchroma/coloring.py; the greedy pass, the
conflict repair and the restart loop run in native C++
(``csrc/coloring.cpp``: ``mc_color``, ``mc_modified_greedy``,
``mc_resolve_conflicts``, ``mc_naive_greedy``) and reproduce the
reference's CPython ``random.Random`` stream exactly, so colorings are
bit-identical for the same seed.

``verify_coloring`` stays vectorised numpy (coloring.py:491-522 semantics).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .mesh import Diagnostic, ElementKind, Mesh, connectivity_graph, vizing_bound


def color_set_size(mesh: Mesh) -> int:
    """3 for pure triangle meshes, 4 once quads or tets are present
    (coloring.py:38-42)."""
    if mesh.element_kind_profile == frozenset({ElementKind.TRIANGLE}):
        return 3
    return 4


@dataclass(frozen=True)
class ColoringConfig:
    rng_seed: int = 0
    max_swaps_per_conflict: int | None = None   # None -> 10 * n_surfaces
    max_restarts: int = 5
    audit: bool = False


@dataclass(eq=False)
class SurfaceColoring:
    """Color per surface (-1 = uncolored) plus the palette size."""

    colors: np.ndarray  # (ns,) int32
    n_colors: int

    @property
    def is_complete(self) -> bool:
        return bool((self.colors >= 1).all())

    def conflict_ids(self) -> np.ndarray:
        return np.flatnonzero(self.colors < 0)

    def color_counts(self) -> tuple:
        counts = np.bincount(self.colors[self.colors >= 1],
                             minlength=self.n_colors + 1)
        return tuple(int(c) for c in counts[1: self.n_colors + 1])

    def copy(self) -> "SurfaceColoring":
        return SurfaceColoring(self.colors.copy(), self.n_colors)


@dataclass(frozen=True)
class ColoringReport:
    n_elements: int
    n_surfaces: int
    n_colors: int
    vizing_bound: int
    greedy_conflicts: int
    resolutions: int
    swaps: int
    loop_breaks: int
    no_swap_breaks: int
    forced_reswaps: int
    restarts: int
    color_counts: tuple
    greedy_seconds: float
    resolve_seconds: float
    total_seconds: float

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k in (
            "n_elements", "n_surfaces", "n_colors", "vizing_bound",
            "greedy_conflicts", "resolutions", "swaps", "loop_breaks",
            "no_swap_breaks", "forced_reswaps", "restarts")}
        for i, n in enumerate(self.color_counts, start=1):
            d[f"color_count_{i}"] = n
        for k in ("greedy_seconds", "resolve_seconds", "total_seconds"):
            d[k] = round(getattr(self, k), 6)
        return d


def _incidence_arrays(mesh: Mesh):
    se = np.ascontiguousarray(mesh.surf_elems, dtype=np.int64)
    es = np.ascontiguousarray(mesh.elem_surfs, dtype=np.int64)
    return se, es


def _budget(config: ColoringConfig, mesh: Mesh) -> int:
    b = config.max_swaps_per_conflict
    return 10 * mesh.n_surfaces if b is None else int(b)


def modified_greedy(mesh: Mesh, config: ColoringConfig | None = None
                    ) -> SurfaceColoring:
    """Greedy pass only; unresolvable surfaces stay -1 (coloring.py:351-362)."""
    config = config or ColoringConfig()
    if mesh.n_surfaces == 0:
        raise ValueError("mesh has no surfaces")
    n_colors = color_set_size(mesh)
    se, _ = _incidence_arrays(mesh)
    out = np.empty(mesh.n_surfaces, dtype=np.int32)
    nconf = np.zeros(1, dtype=np.int64)
    lib = _native.lib()
    _native.check(lib.mc_modified_greedy(
        mesh.n_surfaces, mesh.n_elements, _native.ptr(se), n_colors,
        int(config.rng_seed), _native.ptr(out), _native.ptr(nconf)))
    return SurfaceColoring(out, n_colors)


def resolve_conflicts(mesh: Mesh, coloring: SurfaceColoring,
                      config: ColoringConfig | None = None,
                      stats_out: dict | None = None) -> SurfaceColoring:
    """Repair a partial coloring with a fresh RNG stream
    (coloring.py:365-392)."""
    config = config or ColoringConfig()
    se, es = _incidence_arrays(mesh)
    colors = np.ascontiguousarray(coloring.colors, dtype=np.int32).copy()
    if len(colors) != mesh.n_surfaces:
        raise ValueError("coloring does not match the mesh")
    st = _native.ColoringStats()
    lib = _native.lib()
    _native.check(lib.mc_resolve_conflicts(
        mesh.n_surfaces, mesh.n_elements, _native.ptr(se), _native.ptr(es),
        int(coloring.n_colors), int(config.rng_seed), _budget(config, mesh),
        int(bool(config.audit)), _native.ptr(colors), st))
    if stats_out is not None:
        stats_out.update(resolutions=st.resolutions, swaps=st.swaps,
                         loop_breaks=st.loop_breaks,
                         no_swap_breaks=st.no_swap_breaks,
                         forced_reswaps=st.forced_reswaps)
    return SurfaceColoring(colors, coloring.n_colors)


def color(mesh: Mesh, config: ColoringConfig | None = None):
    """Complete valid coloring plus report (coloring.py:395-459).

    Greedy and repair share one RNG stream; a budget overrun restarts from
    ``rng_seed + attempt``; ``RestartsExhaustedError`` after
    ``max_restarts + 1`` attempts."""
    config = config or ColoringConfig()
    if mesh.n_surfaces == 0:
        raise ValueError("mesh has no surfaces")
    n_colors = color_set_size(mesh)
    se, es = _incidence_arrays(mesh)
    out = np.empty(mesh.n_surfaces, dtype=np.int32)
    st = _native.ColoringStats()
    lib = _native.lib()
    _native.check(lib.mc_color(
        mesh.n_surfaces, mesh.n_elements, _native.ptr(se), _native.ptr(es),
        n_colors, int(config.rng_seed), _budget(config, mesh),
        int(config.max_restarts), int(bool(config.audit)), _native.ptr(out),
        st))
    coloring = SurfaceColoring(out, n_colors)
    report = ColoringReport(
        n_elements=mesh.n_elements, n_surfaces=mesh.n_surfaces,
        n_colors=n_colors,
        vizing_bound=vizing_bound(connectivity_graph(mesh)),
        greedy_conflicts=st.greedy_conflicts, resolutions=st.resolutions,
        swaps=st.swaps, loop_breaks=st.loop_breaks,
        no_swap_breaks=st.no_swap_breaks, forced_reswaps=st.forced_reswaps,
        restarts=st.restarts, color_counts=coloring.color_counts(),
        greedy_seconds=st.greedy_seconds, resolve_seconds=st.resolve_seconds,
        total_seconds=st.total_seconds)
    return coloring, report


def naive_greedy(mesh: Mesh) -> SurfaceColoring:
    """First-fit baseline with an unbounded palette (coloring.py:462-488)."""
    if mesh.n_surfaces == 0:
        raise ValueError("mesh has no surfaces")
    se, _ = _incidence_arrays(mesh)
    out = np.empty(mesh.n_surfaces, dtype=np.int32)
    top = np.zeros(1, dtype=np.int32)
    _native.check(_native.lib().mc_naive_greedy(
        mesh.n_surfaces, mesh.n_elements, _native.ptr(se), _native.ptr(out),
        _native.ptr(top)))
    return SurfaceColoring(out, int(top[0]))


def verify_coloring(mesh: Mesh, coloring: SurfaceColoring) -> list:
    """Every element with a repeated color and every uncolored surface;
    empty means complete and valid (same diagnostics, in the same order and
    wording, as coloring.py:491-522).  A slot is in conflict when another
    slot of its element row carries the same color (>= 1); the slot-pair
    comparison over the <= 4 local sides is done for all elements at once."""
    colors = np.asarray(coloring.colors)
    es = mesh.elem_surfs
    slot_col = np.where(es >= 0, colors[np.maximum(es, 0)], 0).astype(np.int64)
    slot_col[slot_col < 1] = 0                       # uncolored / absent: never a repeat
    twin = (slot_col[:, :, None] == slot_col[:, None, :]) & (slot_col[:, :, None] > 0)
    in_conflict = twin.sum(axis=2) > 1               # (ne, sides)
    out: list = []
    for e in np.flatnonzero(in_conflict.any(axis=1)):
        hit = in_conflict[e]
        out.append(Diagnostic(
            "conflict",
            f"element {e} repeats color(s) {sorted(set(slot_col[e][hit].tolist()))} "
            f"on surfaces {es[e][hit].tolist()}",
            element_id=int(e)))
    out.extend(Diagnostic("uncolored", f"surface {k} has no color", surface_id=int(k))
               for k in np.flatnonzero(colors < 1))
    return out
