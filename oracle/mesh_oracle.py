"""Synthetic meshes and surface extraction restated in numpy (oracle).

TEST INFRASTRUCTURE ONLY: used by tests/ and by bench.py's CPU legs (the
reference arm builds its sample mesh here so it never touches the product
library).  Restates /root/reference/pkg/src/meshchroma:

  generators.gen_tri_rect   :79-106   two triangles per cell, diagonal
                                      alternating with cell parity, CCW
  generators.gen_quad_rect  :109-131  one quad per cell
  generators.gen_tet_prism  :138-182  six tets per hex cell around v0-v7
  generators.shuffle_elements :185-197 default_rng(seed).permutation
  mesh.assemble             :207-300  surface ids by first encounter in
                                      element-major / side-minor order,
                                      left = smaller element id

Returns plain dicts of arrays (vertices, elem_kind, elem_verts, elem_surfs,
surf_verts, surf_elems), the reference's Mesh fields.  Pinned against the
reference-generated goldens in tests/test_oracle_golden.py.
"""

from __future__ import annotations

import numpy as np

TRI, QUAD, TET = 0, 1, 2
NVERT = {TRI: 3, QUAD: 4, TET: 4}
SIDES = {TRI: ((0, 1), (1, 2), (2, 0)),
         QUAD: ((0, 1), (1, 2), (2, 3), (3, 0)),
         TET: ((0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3))}


def assemble(vertices, kinds, elem_verts) -> dict:
    vertices = np.asarray(vertices, dtype=np.float64)
    kinds = np.asarray(kinds, dtype=np.int8)
    ev = np.asarray(elem_verts, dtype=np.int64)
    ne = len(kinds)
    width = 3 if (kinds == TET).any() else 2
    # every (element, local side) slot, element-major
    slots = np.full((ne, 4, width), -1, dtype=np.int64)
    for k in np.unique(kinds):
        rows = np.flatnonzero(kinds == k)
        for j, pos in enumerate(SIDES[int(k)]):
            slots[rows, j, :] = ev[rows][:, list(pos)]
    valid = slots[:, :, 0] >= 0
    slot_id = np.flatnonzero(valid.reshape(-1))          # ascending = encounter order
    tup = np.sort(slots.reshape(-1, width)[slot_id], axis=1)
    # group equal vertex tuples; a stable sort keeps the first encounter first
    order = np.lexsort(tup.T[::-1])
    st = tup[order]
    new = np.ones(len(st), dtype=bool)
    new[1:] = (st[1:] != st[:-1]).any(axis=1)
    grp = np.cumsum(new) - 1                             # tuple group per sorted slot
    first_pos = np.flatnonzero(new)                      # sorted position of each group head
    first_slot = order[first_pos]                        # its encounter index
    rank = np.empty(len(first_pos), dtype=np.int64)      # surface id = encounter rank
    rank[np.argsort(first_slot, kind="stable")] = np.arange(len(first_pos))
    sid_sorted = rank[grp]
    sid = np.empty(len(st), dtype=np.int64)
    sid[order] = sid_sorted
    ns = len(first_pos)
    count = np.bincount(sid, minlength=ns)
    if (count > 2).any():
        raise ValueError("non-manifold: a surface is shared by more than two elements")
    elem = slot_id // 4
    side = slot_id % 4
    surf_verts = np.empty((ns, width), dtype=np.int64)
    surf_verts[sid] = tup
    # the first slot of a surface is its smaller element (element-major)
    left = np.full(ns, -1, dtype=np.int64)
    right = np.full(ns, -1, dtype=np.int64)
    by = np.argsort(sid, kind="stable")
    head = np.ones(len(by), dtype=bool)
    head[1:] = sid[by][1:] != sid[by][:-1]
    left[sid[by][head]] = elem[by][head]
    right[sid[by][~head]] = elem[by][~head]
    elem_surfs = np.full((ne, 4), -1, dtype=np.int64)
    elem_surfs[elem, side] = sid
    return dict(vertices=vertices, elem_kind=kinds, elem_verts=ev, elem_surfs=elem_surfs,
                surf_verts=surf_verts, surf_elems=np.stack([left, right], axis=1))


def _pair(periodic):
    if isinstance(periodic, (bool, np.bool_)):
        return bool(periodic), bool(periodic)
    return bool(periodic[0]), bool(periodic[1])


def _grid(nx, ny, px, py):
    mx = nx if px else nx + 1
    my = ny if py else ny + 1
    jj, ii = np.divmod(np.arange(mx * my), mx)
    verts = np.stack([ii, jj], axis=1).astype(np.float64)
    ci = np.arange(nx + 1) % mx
    cj = np.arange(ny + 1) % my
    return verts, cj[:, None] * mx + ci[None, :]


def gen_tri_rect(nx, ny, periodic=False) -> dict:
    px, py = _pair(periodic)
    verts, vid = _grid(nx, ny, px, py)
    j, i = np.divmod(np.arange(nx * ny), nx)
    a, b = vid[j, i], vid[j, i + 1]
    c, d = vid[j + 1, i + 1], vid[j + 1, i]
    even = (i + j) % 2 == 0
    ev = np.full((nx * ny, 2, 4), -1, dtype=np.int64)
    ev[:, 0, :3] = np.stack([a, b, np.where(even, c, d)], axis=1)
    ev[:, 1, :3] = np.stack([np.where(even, a, b), c, d], axis=1)
    ev = ev.reshape(-1, 4)
    return assemble(verts, np.full(len(ev), TRI, np.int8), ev)


def gen_quad_rect(nx, ny, periodic=False) -> dict:
    px, py = _pair(periodic)
    verts, vid = _grid(nx, ny, px, py)
    j, i = np.divmod(np.arange(nx * ny), nx)
    ev = np.stack([vid[j, i], vid[j, i + 1], vid[j + 1, i + 1], vid[j + 1, i]], axis=1)
    return assemble(verts, np.full(len(ev), QUAD, np.int8), ev)


def gen_hybrid_rect(nx, ny, periodic=False) -> dict:
    """Triangle + quad mix: the reference tests' ``conftest.hybrid_patch``
    layout (cells with i+j even -> triangles (a,b,c), (a,c,d); others quads)."""
    px, py = _pair(periodic)
    verts, vid = _grid(nx, ny, px, py)
    rows, kinds = [], []
    for c in range(nx * ny):
        j, i = divmod(c, nx)
        a, b, cc, d = vid[j, i], vid[j, i + 1], vid[j + 1, i + 1], vid[j + 1, i]
        if (i + j) % 2 == 0:
            rows += [(a, b, cc, -1), (a, cc, d, -1)]
            kinds += [TRI, TRI]
        else:
            rows.append((a, b, cc, d))
            kinds.append(QUAD)
    return assemble(verts, np.asarray(kinds, np.int8), np.asarray(rows, np.int64))


# six tets per hex cell sharing the diagonal v0-v7 (corner bits: x, y, z)
_HEX = ((0, 1, 3, 7), (0, 1, 7, 5), (0, 5, 7, 4), (0, 3, 2, 7), (0, 6, 4, 7), (0, 2, 6, 7))


def gen_tet_prism(nx, ny, nz) -> dict:
    n = np.arange((nx + 1) * (ny + 1) * (nz + 1))
    kz, r = np.divmod(n, (nx + 1) * (ny + 1))
    jy, ix = np.divmod(r, nx + 1)
    verts = np.stack([ix, jy, kz], axis=1).astype(np.float64)
    # cells in (i, j, k) C order: cell id (i*ny + j)*nz + k
    c = np.arange(nx * ny * nz)
    i, rest = np.divmod(c, ny * nz)
    j, k = np.divmod(rest, nz)
    corner = [((k + (b >> 2)) * (ny + 1) + (j + ((b >> 1) & 1))) * (nx + 1) + (i + (b & 1))
              for b in range(8)]
    ev = np.stack([np.stack([corner[v] for v in t], axis=1) for t in _HEX], axis=1)
    ev = ev.reshape(-1, 4)
    return assemble(verts, np.full(len(ev), TET, np.int8), ev)


def shuffle_elements(mesh: dict, seed: int) -> dict:
    order = np.random.default_rng(seed).permutation(len(mesh["elem_kind"]))
    return assemble(mesh["vertices"], mesh["elem_kind"][order], mesh["elem_verts"][order])
