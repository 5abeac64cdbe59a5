"""Synthetic mesh generators (the inputs of every benchmark config).

Same vertex numbering, element order and local vertex order as the
reference generators (/root/reference/pkg/src/meshchroma/generators.py),
because surface ids, colors and permutations downstream must match the
reference bit for bit:

* ``gen_tri_rect`` — cell (i, j) gives elements 2(j*nx+i)+{0,1}; even cells
  (i+j even) split along a-c, odd cells along b-d (generators.py:96-105);
* ``gen_quad_rect`` — one quad per cell, (a, b, c, d) (generators.py:126-131);
* ``gen_tet_prism`` — cell (i*ny+j)*nz+k holds six tets around the v0-v7
  diagonal (generators.py:141-148, 166-179);
* ``shuffle_elements`` — ``np.random.default_rng(seed).permutation``
  (generators.py:194-197; numpy is the pinned third-party dependency).

Periodic wrap-around is topological only: wrapped cells reuse vertex ids
from the opposite side (generators.py:67-76); ``dg.geometry`` unwraps
coordinates for the DG operator.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import ElementKind, KIND_TO_CODE, MAX_ELEM_VERTS, Mesh, assemble

FAMILIES = ("tri_rect", "quad_rect", "tet_prism", "tri_closed")


@dataclass(frozen=True)
class GeneratorSpec:
    family: str
    nx: int
    ny: int
    nz: int = 1
    periodic_x: bool = False
    periodic_y: bool = False

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown family {self.family!r}")


def generate(spec: GeneratorSpec) -> Mesh:
    if spec.family == "tri_rect":
        return gen_tri_rect(spec.nx, spec.ny, (spec.periodic_x, spec.periodic_y))
    if spec.family == "tri_closed":
        return gen_tri_rect(spec.nx, spec.ny, (True, True))
    if spec.family == "quad_rect":
        return gen_quad_rect(spec.nx, spec.ny, (spec.periodic_x, spec.periodic_y))
    return gen_tet_prism(spec.nx, spec.ny, spec.nz)


def _check_axis(name: str, n: int, periodic: bool) -> None:
    if n < 1:
        raise ValueError(f"{name} must be >= 1, got {n}")
    if periodic and n < 3:
        raise ValueError(f"periodic {name} needs at least 3 cells, got {n}")


def _pair(periodic):
    if isinstance(periodic, (bool, np.bool_)):
        return bool(periodic), bool(periodic)
    px, py = periodic
    return bool(px), bool(py)


def _lattice(nx: int, ny: int, px: bool, py: bool):
    """Coordinates of the stored vertices and an (ny+1, nx+1) table of the
    vertex id at each lattice point, folded on periodic axes."""
    cols = nx if px else nx + 1
    rows = ny if py else ny + 1
    yy, xx = np.divmod(np.arange(rows * cols), cols)
    coords = np.stack([xx, yy], axis=1).astype(np.float64)
    ii = np.arange(nx + 1) % cols
    jj = np.arange(ny + 1) % rows
    table = jj[:, None] * cols + ii[None, :]
    return coords, table


def _cell_corners(table, nx, ny):
    j, i = np.divmod(np.arange(nx * ny), nx)          # cell order j-major
    a = table[j, i]
    b = table[j, i + 1]
    c = table[j + 1, i + 1]
    d = table[j + 1, i]
    return i, j, a, b, c, d


def gen_tri_rect(nx: int, ny: int, periodic=False, *, device=None) -> Mesh:
    """Two right triangles per unit cell, diagonal alternating with parity."""
    px, py = _pair(periodic)
    _check_axis("nx", nx, px)
    _check_axis("ny", ny, py)
    coords, table = _lattice(nx, ny, px, py)
    i, j, a, b, c, d = _cell_corners(table, nx, ny)
    even = (i + j) % 2 == 0
    ev = np.full((nx * ny, 2, MAX_ELEM_VERTS), -1, dtype=np.int64)
    ev[:, 0, 0] = a
    ev[:, 0, 1] = b
    ev[:, 0, 2] = np.where(even, c, d)
    ev[:, 1, 0] = np.where(even, a, b)
    ev[:, 1, 1] = c
    ev[:, 1, 2] = d
    ev = ev.reshape(-1, MAX_ELEM_VERTS)
    kinds = np.full(len(ev), KIND_TO_CODE[ElementKind.TRIANGLE], np.int8)
    return assemble(coords, kinds, ev, device=device)


def gen_quad_rect(nx: int, ny: int, periodic=False, *, device=None) -> Mesh:
    """One unit quad per cell, counter-clockwise (a, b, c, d)."""
    px, py = _pair(periodic)
    _check_axis("nx", nx, px)
    _check_axis("ny", ny, py)
    coords, table = _lattice(nx, ny, px, py)
    _, _, a, b, c, d = _cell_corners(table, nx, ny)
    ev = np.stack([a, b, c, d], axis=1).astype(np.int64)
    kinds = np.full(len(ev), KIND_TO_CODE[ElementKind.QUAD], np.int8)
    return assemble(coords, kinds, ev, device=device)


# six tetrahedra per hex cell sharing the v0-v7 diagonal; corner k of the
# cell is (i + (k & 1), j + ((k >> 1) & 1), kz + (k >> 2))
_HEX_SPLIT = np.array([(0, 1, 3, 7), (0, 1, 7, 5), (0, 5, 7, 4),
                       (0, 3, 2, 7), (0, 6, 4, 7), (0, 2, 6, 7)],
                      dtype=np.int64)


def gen_hybrid_rect(nx: int, ny: int, periodic=False, *, device=None) -> Mesh:
    """Conforming triangle + quad mix (not a reference generator: the
    reference's hybrid meshes are its test fixture ``conftest.hybrid_patch``,
    same layout): cells with i+j even are split along a-c into triangles
    (a, b, c), (a, c, d), the other cells stay quads (a, b, c, d); elements
    in cell order.  Colored with the 4-color palette (``coloring.py:38-42``);
    the DG operator runs it as ``MC_KIND_HYBRID``."""
    px, py = _pair(periodic)
    _check_axis("nx", nx, px)
    _check_axis("ny", ny, py)
    coords, table = _lattice(nx, ny, px, py)
    i, j, a, b, c, d = _cell_corners(table, nx, ny)
    even = (i + j) % 2 == 0
    # two slots per cell; odd cells use the first only
    ev = np.full((nx * ny, 2, MAX_ELEM_VERTS), -1, dtype=np.int64)
    ev[:, 0, 0], ev[:, 0, 1], ev[:, 0, 2] = a, b, c
    ev[:, 0, 3] = np.where(even, -1, d)
    ev[:, 1, 0], ev[:, 1, 1], ev[:, 1, 2] = a, c, d
    kinds = np.empty((nx * ny, 2), np.int8)
    kinds[:, 0] = np.where(even, KIND_TO_CODE[ElementKind.TRIANGLE], KIND_TO_CODE[ElementKind.QUAD])
    kinds[:, 1] = KIND_TO_CODE[ElementKind.TRIANGLE]
    keep = np.stack([np.ones(nx * ny, bool), even], axis=1)
    return assemble(coords, kinds[keep], ev[keep], device=device)


def gen_tet_prism(nx: int, ny: int, nz: int, *, device=None) -> Mesh:
    """Box of unit hex cells, each cut into six positively oriented tets."""
    for name, n in (("nx", nx), ("ny", ny), ("nz", nz)):
        _check_axis(name, n, False)
    npts = (nx + 1) * (ny + 1) * (nz + 1)
    rest, x = np.divmod(np.arange(npts), nx + 1)
    z, y = np.divmod(rest, ny + 1)
    coords = np.stack([x, y, z], axis=1).astype(np.float64)
    # cells ordered i-major, then j, then k (cell id = (i*ny+j)*nz+k)
    cid = np.arange(nx * ny * nz)
    ij, k = np.divmod(cid, nz)
    i, j = np.divmod(ij, ny)
    corner = np.empty((len(cid), 8), dtype=np.int64)
    for m in range(8):
        ci, cj, ck = i + (m & 1), j + ((m >> 1) & 1), k + (m >> 2)
        corner[:, m] = (ck * (ny + 1) + cj) * (nx + 1) + ci
    ev = np.full((len(cid), 6, MAX_ELEM_VERTS), -1, dtype=np.int64)
    ev[:, :, :] = corner[:, _HEX_SPLIT]
    ev = ev.reshape(-1, MAX_ELEM_VERTS)
    kinds = np.full(len(ev), KIND_TO_CODE[ElementKind.TET], np.int8)
    return assemble(coords, kinds, ev, device=device)


def shuffle_elements(mesh: Mesh, seed: int, *, device=None) -> Mesh:
    """Re-assemble with element ids permuted by numpy's PCG64 stream."""
    order = np.random.default_rng(seed).permutation(mesh.n_elements)
    return assemble(mesh.vertices, mesh.elem_kind[order],
                    mesh.elem_verts[order], device=device)
