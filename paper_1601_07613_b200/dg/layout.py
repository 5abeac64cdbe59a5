"""Color-major DG surface list and element geometry (host, built once).

Input: a mesh already renumbered by ``reorder.apply_plan`` (so surfaces are
grouped by color and, in color 1, left/right are ``k`` / ``N1 + k``) and its
coloring.  Output: the arrays ``mc_dg_create`` uploads (DESIGN.md
§Surface record):

* ``left``/``right`` int32 (right = -1 physical boundary);
* ``code`` uint32: bits 0-5 left side code, 6-11 right side code, then the
  first/last-touch flags of each side; a side code is ``6*f + v`` where
  ``f`` is the element-local side and ``v`` the orientation variant (2D:
  which way the local edge runs w.r.t. the sorted surface vertices, or a
  mortar half; tet: the permutation mapping the sorted face vertices to
  the element's local face vertices);
* ``geom`` float64 (dim+2): unit normal pointing out of the left element,
  then ``s_L = |surface| / |det J_L|`` and ``s_R`` likewise;
* per element ``jinv`` (dim x dim, d xi_r / d x_d) and ``detj``.

First/last-touch flags mark, for every element, the side through which the
colored sweep first and last reaches it; the kernels fuse the volume
integral into the first touch and the RK update into the last.  Nothing
else in the accumulation order changes: per element it is volume, then
colors 1..n (Algorithm 1).

Nonconforming (AMR) meshes: each hanging (full, half1, half2) triple of a
``RefinedMesh`` becomes two mortar surfaces (fine child left, coarse
element right, the coarse side evaluated on the matching half of its
edge); the full coarse edge is dropped.  The mortar-inclusive race
certificate is checked here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ..errors import WriteConflictError
from ..mesh import ElementKind, Mesh, SIDE_POSITIONS, CODE_TO_KIND
from .basis import DIM, EDGE_VARIANTS, FACE_PERMS, HYBRID, HYBRID_TRI_CODE0

FLAG_L_FIRST = 1 << 12
FLAG_L_LAST = 1 << 13
FLAG_R_FIRST = 1 << 14
FLAG_R_LAST = 1 << 15
FLAG_R_GHOST = 1 << 16
FLAG_FLIPPED = 1 << 17


def mesh_kind(mesh: Mesh):
    """The DG element kind: a single ElementKind, or ``HYBRID`` for a
    conforming triangle + quad mix."""
    kinds = mesh.element_kind_profile
    if kinds == {ElementKind.TRIANGLE, ElementKind.QUAD}:
        return HYBRID
    if len(kinds) != 1:
        raise NotImplementedError("DG operator needs a single-kind or a triangle + quad mesh")
    return next(iter(kinds))


def element_kinds(mesh: Mesh) -> np.ndarray:
    """(ne,) uint8 element kind codes (0 triangle, 1 quad, 2 tet)."""
    return np.asarray(mesh.elem_kind, dtype=np.uint8)


def unwrapped_element_coords(mesh: Mesh, period=None) -> np.ndarray:
    """(ne, nvert, dim) vertex coordinates per element; periodic generator
    meshes are unwrapped relative to local vertex 0.  Hybrid meshes: 4
    slots, a triangle's fourth repeats its third vertex (``element_centroids``
    averages the real ones)."""
    kind = mesh_kind(mesh)
    nvert = kind.n_vertices
    ev = mesh.elem_verts[:, :nvert]
    if kind is HYBRID:
        ev = np.where(ev >= 0, ev, ev[:, 2:3])
    X = mesh.vertices[ev].copy()
    if period is not None:
        for d, L in enumerate(period):
            if not L:
                continue
            delta = X[:, :, d] - X[:, :1, d]
            X[:, :, d] -= L * np.round(delta / L)
    return X


def element_centroids(mesh: Mesh, X: np.ndarray) -> np.ndarray:
    """Vertex centroids from ``unwrapped_element_coords`` output."""
    if mesh_kind(mesh) is not HYBRID:
        return X.mean(axis=1)
    quad = element_kinds(mesh) == 1
    S = X[:, :3].sum(axis=1) + np.where(quad, 1.0, 0.0)[:, None] * X[:, 3]
    return S / np.where(quad, 4.0, 3.0)[:, None]


def element_geometry(kind, X: np.ndarray, ekind=None):
    """Affine map x = x0 + J xi per element: (detJ (ne,), Jinv (ne,d,d)).
    Hybrid: ``ekind`` (0 triangle, 1 quad) picks each element's map."""
    if kind is HYBRID:
        det = np.empty(len(X))
        inv = np.empty((len(X), 2, 2))
        for code, k in ((0, ElementKind.TRIANGLE), (1, ElementKind.QUAD)):
            m = ekind == code
            if m.any():
                det[m], inv[m] = element_geometry(k, X[m][:, :k.n_vertices])
        return det, inv
    if kind is ElementKind.QUAD:
        J = np.stack([X[:, 1] - X[:, 0], X[:, 3] - X[:, 0]], axis=2)
        skew = X[:, 2] - (X[:, 1] + X[:, 3] - X[:, 0])
        if np.abs(skew).max(initial=0.0) > 1e-9 * (np.abs(J).max() + 1.0):
            raise NotImplementedError("only affine (parallelogram) quads are supported")
    else:
        d = DIM[kind]
        J = np.stack([X[:, r + 1] - X[:, 0] for r in range(d)], axis=2)
    # closed-form determinant / inverse (batched LAPACK is slow at 10^7 elements)
    if J.shape[1] == 2:
        a, b, c, d = J[:, 0, 0], J[:, 0, 1], J[:, 1, 0], J[:, 1, 1]
        det = a * d - b * c
        inv = np.stack([np.stack([d, -b], 1), np.stack([-c, a], 1)], 1)
    else:
        c0 = np.cross(J[:, :, 1], J[:, :, 2])
        c1 = np.cross(J[:, :, 2], J[:, :, 0])
        c2 = np.cross(J[:, :, 0], J[:, :, 1])
        det = (J[:, :, 0] * c0).sum(1)
        inv = np.stack([c0, c1, c2], 1)          # rows of J^-1 * det
    if (np.abs(det) < 1e-300).any():
        raise ValueError("degenerate element")
    return det, inv / det[:, None, None]


def _side_codes_2d(kind, elem_verts, elems, local, surf_verts, mids=None):
    """Orientation variant for 2D sides (0/1 conforming, 2..5 mortar)."""
    a_idx = np.asarray([SIDE_POSITIONS[kind][f][0] for f in range(4 if kind is ElementKind.QUAD else 3)])
    b_idx = np.asarray([SIDE_POSITIONS[kind][f][1] for f in range(len(a_idx))])
    A = elem_verts[elems, a_idx[local]]
    B = elem_verts[elems, b_idx[local]]
    P0, P1 = surf_verts[:, 0], surf_verts[:, 1]
    if mids is None:
        v = np.where(A == P0, 0, 1)
        if not ((A == P0) & (B == P1) | (A == P1) & (B == P0)).all():
            raise AssertionError("side does not match its surface")
        return local * 6 + v

    def param(P):
        return np.where(P == A, 0.0, np.where(P == B, 1.0, np.where(P == mids, 0.5, np.nan)))

    s0, s1 = param(P0), param(P1)
    if np.isnan(s0).any() or np.isnan(s1).any():
        raise AssertionError("mortar half does not lie on the coarse edge")
    table = {v: i for i, v in enumerate(EDGE_VARIANTS)}
    v = np.array([table[(a, b)] for a, b in zip(s0.tolist(), s1.tolist())], dtype=np.int64)
    return local * 6 + v


def _side_codes_any(kind, ekind, elem_verts, elems, local, surf_verts, mids=None):
    """2D side codes; hybrid meshes per element kind, triangle codes after
    the quad's 24 (``HYBRID_TRI_CODE0``)."""
    if kind is not HYBRID:
        return _side_codes_2d(kind, elem_verts, elems, local, surf_verts, mids)
    out = np.zeros(len(elems), dtype=np.int64)
    for code, k, off in ((0, ElementKind.TRIANGLE, HYBRID_TRI_CODE0), (1, ElementKind.QUAD, 0)):
        m = ekind[elems] == code
        if m.any():
            out[m] = off + _side_codes_2d(k, elem_verts, elems[m], local[m], surf_verts[m],
                                          None if mids is None else mids[m])
    return out


def _side_codes_tet(elem_verts, elems, local, surf_verts):
    sides = np.asarray(SIDE_POSITIONS[ElementKind.TET])
    loc = sides[local]                                  # (n, 3) local vertex ids
    G = np.take_along_axis(elem_verts[elems], loc, axis=1)   # global ids
    codes = np.full(len(elems), -1, dtype=np.int64)
    for pi, perm in enumerate(FACE_PERMS):
        ok = (G[:, perm[0]] == surf_verts[:, 0]) & (G[:, perm[1]] == surf_verts[:, 1]) \
            & (G[:, perm[2]] == surf_verts[:, 2])
        codes[ok & (codes < 0)] = pi
    if (codes < 0).any():
        raise AssertionError("face does not match its surface")
    return local * 6 + codes


def _local_side(mesh: Mesh, elems, sids):
    es = mesh.elem_surfs[elems]
    hit = es == sids[:, None]
    if not hit.any(axis=1).all():
        raise AssertionError("element does not list the surface")
    return np.argmax(hit, axis=1)


@dataclass
class SurfaceList:
    kind: ElementKind
    n_elements: int
    n_ghosts: int
    bounds: np.ndarray        # n_colors + 1
    left: np.ndarray          # int32
    right: np.ndarray         # int32
    code: np.ndarray          # uint32
    geom: np.ndarray          # (ns, dim+2) float64
    jinv: np.ndarray          # (ne+ng, dim, dim)
    detj: np.ndarray          # (ne+ng,)
    slot_ptr: np.ndarray      # (ne+1,) CSR of (2*s+side) slots per element
    slots: np.ndarray         # int32
    mesh_surface: np.ndarray  # source surface id (in the layout mesh) per entry
    ekind: np.ndarray = None  # (ne+ng,) uint8 element kinds (0 tri, 1 quad, 2 tet)
    inner: np.ndarray | None = None   # per color: surfaces before the ghost-touching ones

    @property
    def n_surfaces(self) -> int:
        return len(self.left)

    @property
    def n_colors(self) -> int:
        return len(self.bounds) - 1


def _normals(kind, Xl, local_l, surf_pts_l, centroid):
    """Outward unit normal of the left element and the surface measure."""
    if kind is ElementKind.TET:
        A, B, C = surf_pts_l[:, 0], surf_pts_l[:, 1], surf_pts_l[:, 2]
        n = np.cross(B - A, C - A)
        meas = 0.5 * np.linalg.norm(n, axis=1)
        mid = (A + B + C) / 3.0
    else:
        A, B = surf_pts_l[:, 0], surf_pts_l[:, 1]
        t = B - A
        n = np.stack([t[:, 1], -t[:, 0]], axis=1)
        meas = np.linalg.norm(t, axis=1)
        mid = 0.5 * (A + B)
    n = n / np.linalg.norm(n, axis=1)[:, None]
    flip = ((mid - centroid) * n).sum(axis=1) < 0
    n[flip] *= -1.0
    return n, meas


def build_surface_list(mesh: Mesh, colors: np.ndarray, n_colors: int,
                       period=None, mortars=None, owned=None, flipped=None,
                       code_sort=False, code_sort_window: int = 0,
                       code_sort_skip_first: bool = False) -> SurfaceList:
    """Assemble the device surface list from a color-grouped mesh.

    ``colors`` must be non-decreasing over surface ids (a mesh produced by
    apply_plan).  ``mortars``: optional (n, 3) hanging triples
    (full, half_lo, half_hi) in this mesh's surface ids.  ``owned``:
    number of owned elements (elements >= owned are read-only ghosts).
    ``code_sort``: within each color, order surfaces by their (left, right)
    side codes (stable), so the lanes of a warp read the same reference-face
    table rows (shared-memory broadcasts).  Any order within a color is
    race free and leaves every element's accumulation order unchanged.
    ``code_sort_window`` > 0 sorts by code only inside consecutive windows of
    that many surfaces (keeps the element-ascending order at a coarse scale);
    ``code_sort_skip_first`` leaves color 1 (the coalesced color) unsorted.
    """
    kind = mesh_kind(mesh)
    dim = DIM[kind]
    ne_all = mesh.n_elements
    ne = ne_all if owned is None else int(owned)
    colors = np.asarray(colors)
    if (np.diff(colors) < 0).any():
        raise ValueError("surfaces must be grouped by color (apply a ReorderingPlan first)")
    X = unwrapped_element_coords(mesh, period)
    ekind = element_kinds(mesh)
    detj, jinv = element_geometry(kind, X, ekind)
    cen = element_centroids(mesh, X)

    ns = mesh.n_surfaces
    sid = np.arange(ns)
    L = mesh.surf_elems[:, 0].copy()
    R = mesh.surf_elems[:, 1].copy()
    coarse_local = None
    if mortars is not None and len(mortars):
        mortars = np.asarray(mortars, dtype=np.int64)
        full = mortars[:, 0]
        coarse = L[full]
        for k in (1, 2):
            if (R[mortars[:, k]] >= 0).any():
                raise AssertionError("mortar half is not one-sided")
            R[mortars[:, k]] = coarse
        keep = np.ones(ns, dtype=bool)
        keep[full] = False
        coarse_local_full = _local_side(mesh, coarse, full)
        coarse_local = np.full(ns, -1, dtype=np.int64)
        coarse_local[mortars[:, 1]] = coarse_local_full
        coarse_local[mortars[:, 2]] = coarse_local_full
        mid_of = np.full(ns, -1, dtype=np.int64)
        for k in (1, 2):
            hv = mesh.surf_verts[mortars[:, k]]
            fv = mesh.surf_verts[full]
            end0 = (hv[:, 0] == fv[:, 0]) | (hv[:, 0] == fv[:, 1])
            m = np.where(end0, hv[:, 1], hv[:, 0])
            mid_of[mortars[:, k]] = m
        sid = sid[keep]
    L, R, col = L[sid], R[sid], colors[sid]
    sv = mesh.surf_verts[sid]

    # race certificate including mortar coupling (O(n) counting per color)
    for c in range(1, n_colors + 1):
        m = col == c
        touched = np.concatenate([L[m], R[m & (R >= 0)]])
        cnt = np.bincount(touched, minlength=ne_all)
        if (cnt > 1).any():
            e = int(np.flatnonzero(cnt > 1)[0])
            raise WriteConflictError(f"color {c} writes element {e} {int(cnt[e])} times")

    loc_l = _local_side(mesh, L, sid)
    has_r = R >= 0
    mortar_r = np.zeros(len(sid), dtype=bool)
    if coarse_local is not None:
        mortar_r = coarse_local[sid] >= 0
    loc_r = np.zeros(len(sid), dtype=np.int64)
    conf_r = has_r & ~mortar_r
    loc_r[conf_r] = _local_side(mesh, R[conf_r], sid[conf_r])
    if mortar_r.any():
        loc_r[mortar_r] = coarse_local[sid[mortar_r]]

    if kind is ElementKind.TET:
        code_l = _side_codes_tet(mesh.elem_verts, L, loc_l, sv)
        code_r = np.zeros(len(sid), dtype=np.int64)
        code_r[has_r] = _side_codes_tet(mesh.elem_verts, R[has_r], loc_r[has_r], sv[has_r])
    else:
        code_l = _side_codes_any(kind, ekind, mesh.elem_verts, L, loc_l, sv)
        code_r = np.zeros(len(sid), dtype=np.int64)
        code_r[conf_r] = _side_codes_any(kind, ekind, mesh.elem_verts, R[conf_r], loc_r[conf_r],
                                         sv[conf_r])
        if mortar_r.any():
            code_r[mortar_r] = _side_codes_any(kind, ekind, mesh.elem_verts, R[mortar_r],
                                               loc_r[mortar_r],
                                              sv[mortar_r], mids=mid_of[sid[mortar_r]])

    # surface vertex coordinates as seen by the left element (unwrapped)
    width = sv.shape[1]
    ev_l = mesh.elem_verts[L]
    nvert = kind.n_vertices
    pos = np.zeros((len(sid), width), dtype=np.int64)
    for m in range(width):
        hit = ev_l[:, :nvert] == sv[:, m:m + 1]
        pos[:, m] = np.argmax(hit, axis=1)
    pts_l = np.take_along_axis(X[L], pos[:, :, None].repeat(dim, axis=2), axis=1)
    normal, meas = _normals(kind, X[L], loc_l, pts_l, cen[L])
    geom = np.zeros((len(sid), dim + 2))
    geom[:, :dim] = normal
    geom[:, dim] = meas / np.abs(detj[L])
    geom[has_r, dim + 1] = meas[has_r] / np.abs(detj[R[has_r]])

    # first / last touch per element over the color sequence (owned only)
    code = (code_l | (code_r << 6)).astype(np.int64)
    big = n_colors + 1
    # first / last color per element from its side list (+ mortar halves)
    pos = np.full(mesh.n_surfaces, -1, dtype=np.int64)
    pos[sid] = np.arange(len(sid))
    es = mesh.elem_surfs
    ent = np.where(es >= 0, pos[np.where(es >= 0, es, 0)], -1)
    ecol = np.where(ent >= 0, col[np.where(ent >= 0, ent, 0)], -1)
    first = np.where(ecol >= 1, ecol, big).min(axis=1)
    last = ecol.max(axis=1).clip(min=0)
    if mortar_r.any():                 # coarse elements also see the mortar halves
        np.minimum.at(first, R[mortar_r], col[mortar_r])
        np.maximum.at(last, R[mortar_r], col[mortar_r])
    if (first[:ne] == big).any():
        raise ValueError("element without surfaces")
    code |= np.where(first[L] == col, FLAG_L_FIRST, 0)
    code |= np.where(last[L] == col, FLAG_L_LAST, 0)
    rr = np.where(has_r, R, 0)
    ghost_r = has_r & (R >= ne)
    own_r = has_r & ~ghost_r          # ghosts are never finalised: no flags
    code |= np.where(own_r & (first[rr] == col), FLAG_R_FIRST, 0)
    code |= np.where(own_r & (last[rr] == col), FLAG_R_LAST, 0)
    code |= np.where(ghost_r, FLAG_R_GHOST, 0)
    if flipped is not None:
        code |= np.where(np.asarray(flipped)[sid], FLAG_FLIPPED, 0)
    if (L >= ne).any():
        raise ValueError("left elements must be owned")

    if code_sort or (owned is not None and ghost_r.any()):
        # partitioned: surfaces touching a ghost go last in their color, so
        # the rest of the first color can run while the ghosts are exchanged
        key2 = (code & 0xFFF) if code_sort else np.zeros(len(sid), dtype=np.int64)
        if code_sort and code_sort_window > 0:
            # windows counted from each color's first surface (col is
            # non-decreasing here), so no color starts with a partial window
            pos = np.arange(len(sid), dtype=np.int64) - np.searchsorted(col, col, side="left")
            key2 = key2 + (pos // code_sort_window) * 4096
        if code_sort and code_sort_skip_first:
            key2 = np.where(col == 1, 0, key2)
        perm = np.lexsort((np.arange(len(sid)), key2, ghost_r.astype(np.int64), col))
        L, R, code, geom, col, sid = L[perm], R[perm], code[perm], geom[perm], col[perm], sid[perm]
        has_r, ghost_r, loc_l, loc_r = has_r[perm], ghost_r[perm], loc_l[perm], loc_r[perm]
        mortar_r = mortar_r[perm]

    bounds = np.zeros(n_colors + 1, dtype=np.int64)
    bounds[1:] = np.cumsum(np.bincount(col, minlength=n_colors + 1)[1:n_colors + 1])
    inner = np.bincount(col[~ghost_r], minlength=n_colors + 1)[1:n_colors + 1].astype(np.int64)

    # CSR of buffer slots per owned element (local side order for conforming
    # sides, mortar halves appended) for the buffer-and-reduce variant
    ent = np.arange(len(sid))
    own_r = has_r & ~ghost_r
    elem = np.concatenate([L, R[own_r]])
    slot = np.concatenate([2 * ent, 2 * ent[own_r] + 1])
    rank = np.concatenate([loc_l, loc_r[own_r] + 4 * mortar_r[own_r]])
    order = np.argsort(elem * 16 + rank, kind="stable")   # slots ascend within ties
    elem, slot = elem[order], slot[order]
    ptr = np.zeros(ne + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(np.bincount(elem, minlength=ne)[:ne])

    return SurfaceList(
        kind=kind, n_elements=ne, n_ghosts=ne_all - ne, bounds=bounds,
        left=L.astype(np.int32), right=np.where(has_r, R, -1).astype(np.int32),
        code=code.astype(np.uint32), geom=np.ascontiguousarray(geom),
        jinv=np.ascontiguousarray(jinv), detj=detj, slot_ptr=ptr,
        slots=slot.astype(np.int32), mesh_surface=sid, inner=inner, ekind=ekind)
