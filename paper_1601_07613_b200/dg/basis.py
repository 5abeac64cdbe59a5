"""Orthonormal modal bases, quadrature and reference-element trace tables.

The paper's DG uses N_p orthonormal modal basis functions
per element.  Definitions used throughout (DESIGN.md §DG discretisation):

* triangle  T = {xi, eta >= 0, xi + eta <= 1}: Dubiner/Koornwinder
  psi_ij = Y^i P_i(X / Y) * P_j^(2i+1,0)(2 eta - 1), X = 2 xi + eta - 1,
  Y = 1 - eta, ordered by total degree n = i + j, then j ascending;
* quadrilateral [0,1]^2: L_i(xi) L_j(eta), L_i = sqrt(2i+1) P_i(2t-1),
  index i * (p+1) + j;
* tetrahedron: psi_ijk = Y^i P_i(X/Y) * Z^j P_j^(2i+1,0)(W/Z)
  * P_k^(2i+2j+2,0)(2 zeta - 1) with X = 2 xi + eta + zeta - 1,
  Y = 1 - eta - zeta, W = 2 eta + zeta - 1, Z = 1 - zeta, ordered by n,
  then i descending, then j descending;
each scaled to unit L2 norm on the reference element, so the mass matrix
of an affine element is |det J| * I.

Modes are evaluated with the homogeneous Jacobi three-term recurrence
(no collapsed-coordinate division, so no singular points) carried in
forward-mode dual numbers for exact gradients; each mode is normalised with
a quadrature rule exact for its square.

Quadrature: Gauss-Legendre on edges (p+1 points, weights summing to 1),
collapsed Gauss-Jacobi on triangles/tetrahedra ((p+1)^d points) and the
tensor Gauss-Legendre rule on quads; for p = 2 the minimal symmetric
degree-5 rules replace the collapsed ones (7 points on triangles and tet
faces, 14 in tetrahedra).  Volume weights sum to the reference
measure (1/2, 1, 1/6); face weights sum to 1.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np
from scipy.special import roots_jacobi

from ..mesh import ElementKind, SIDE_POSITIONS

REF_VERTS = {
    ElementKind.TRIANGLE: np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]),
    ElementKind.QUAD: np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]]),
    ElementKind.TET: np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0],
                               [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]),
}
REF_MEASURE = {ElementKind.TRIANGLE: 0.5, ElementKind.QUAD: 1.0,
               ElementKind.TET: 1.0 / 6.0}
DIM = {ElementKind.TRIANGLE: 2, ElementKind.QUAD: 2, ElementKind.TET: 3}

# 2D side variants: (s0, s1) = local-edge parameter at the surface's first
# and second (sorted) vertex; the last four are mortar halves
EDGE_VARIANTS = ((0.0, 1.0), (1.0, 0.0), (0.0, 0.5), (0.5, 0.0),
                 (0.5, 1.0), (1.0, 0.5))
FACE_PERMS = tuple(itertools.permutations(range(3)))


class _HybridKind:
    """The DG element kind of a conforming triangle + quad mix (the
    reference's hybrid meshes, ``coloring.py:38-42``): quad-sized blocks,
    triangles on their first (p+1)(p+2)/2 modes."""
    value = "hybrid"
    name = "HYBRID"
    n_vertices = 4

    def __repr__(self):
        return "HYBRID"


HYBRID = _HybridKind()
DIM[HYBRID] = 2
# face codes of a hybrid layout: quad sides 0..23, triangle sides from here
HYBRID_TRI_CODE0 = 24


def n_face_codes(kind) -> int:
    if kind is HYBRID:
        return HYBRID_TRI_CODE0 + len(SIDE_POSITIONS[ElementKind.TRIANGLE]) * 6
    return len(SIDE_POSITIONS[kind]) * 6


def basis_size(kind, p: int) -> int:
    if kind is HYBRID:
        kind = ElementKind.QUAD
    if kind is ElementKind.TRIANGLE:
        return (p + 1) * (p + 2) // 2
    if kind is ElementKind.QUAD:
        return (p + 1) ** 2
    return (p + 1) * (p + 2) * (p + 3) // 6


# ------------------------------------------------- basis evaluation
class _Dual:
    """Value and gradient of a polynomial at a set of points (forward-mode
    differentiation of the three-term recurrences: exact and stable)."""

    def __init__(self, val, grad):
        self.v = val
        self.g = grad            # (dim, npts)

    @staticmethod
    def linear(pts, const, grads):
        grads = np.asarray(grads, dtype=np.float64)
        return _Dual(const + pts @ grads,
                     np.repeat(grads[:, None], len(pts), axis=1))

    @staticmethod
    def const(pts, value):
        return _Dual(np.full(len(pts), float(value)),
                     np.zeros((pts.shape[1], len(pts))))

    def __add__(self, o):
        return _Dual(self.v + o.v, self.g + o.g)

    def __sub__(self, o):
        return _Dual(self.v - o.v, self.g - o.g)

    def __mul__(self, o):
        return _Dual(self.v * o.v, self.g * o.v + o.g * self.v)

    def scale(self, s):
        return _Dual(self.v * s, self.g * s)


def _hjacobi(n, alpha, X, Y, pts):
    """Y^n P_n^(alpha,0)(X/Y) via the homogeneous three-term recurrence."""
    beta = 0.0
    k0 = _Dual.const(pts, 1.0)
    if n == 0:
        return k0
    k1 = X.scale((alpha + beta + 2) / 2) + Y.scale((alpha - beta) / 2)
    for m in range(2, n + 1):
        s = 2 * m + alpha + beta
        a1 = 2 * m * (m + alpha + beta) * (s - 2)
        a2 = (s - 1) * (alpha * alpha - beta * beta)
        a3 = (s - 2) * (s - 1) * s
        a4 = 2 * (m + alpha - 1) * (m + beta - 1) * s
        k2 = ((Y.scale(a2) + X.scale(a3)) * k1
              - (Y * Y * k0).scale(a4)).scale(1.0 / a1)
        k0, k1 = k1, k2
    return k1


def basis_index(kind: ElementKind, p: int):
    """Mode tuples in basis order (see module docstring)."""
    if kind is ElementKind.QUAD:
        return [(i, j) for i in range(p + 1) for j in range(p + 1)]
    if kind is ElementKind.TRIANGLE:
        return [(n - j, j) for n in range(p + 1) for j in range(n + 1)]
    return [(i, j, n - i - j) for n in range(p + 1)
            for i in range(n, -1, -1) for j in range(n - i, -1, -1)]


def _raw_modes(kind: ElementKind, p: int, pts):
    """Unnormalised modes as _Dual objects at reference points."""
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    one = _Dual.const(pts, 1.0)
    out = []
    if kind is ElementKind.QUAD:
        X = _Dual.linear(pts, -1.0, [2.0, 0.0])
        Y = _Dual.linear(pts, -1.0, [0.0, 2.0])
        for i, j in basis_index(kind, p):
            out.append(_hjacobi(i, 0.0, X, one, pts) * _hjacobi(j, 0.0, Y, one, pts))
        return out
    if kind is ElementKind.TRIANGLE:
        X = _Dual.linear(pts, -1.0, [2.0, 1.0])
        Y = _Dual.linear(pts, 1.0, [0.0, -1.0])
        B = _Dual.linear(pts, -1.0, [0.0, 2.0])
        for i, j in basis_index(kind, p):
            out.append(_hjacobi(i, 0.0, X, Y, pts) * _hjacobi(j, 2 * i + 1.0, B, one, pts))
        return out
    X = _Dual.linear(pts, -1.0, [2.0, 1.0, 1.0])
    Y = _Dual.linear(pts, 1.0, [0.0, -1.0, -1.0])
    W = _Dual.linear(pts, -1.0, [0.0, 2.0, 1.0])
    Z = _Dual.linear(pts, 1.0, [0.0, 0.0, -1.0])
    C = _Dual.linear(pts, -1.0, [0.0, 0.0, 2.0])
    for i, j, k in basis_index(kind, p):
        out.append(_hjacobi(i, 0.0, X, Y, pts) * _hjacobi(j, 2 * i + 1.0, W, Z, pts)
                   * _hjacobi(k, 2 * i + 2 * j + 2.0, C, one, pts))
    return out


_NORM_CACHE: dict = {}


def _norms(kind, p):
    key = (kind, p)
    if key not in _NORM_CACHE:
        pts, w = volume_rule(kind, p + 1)          # exact for degree 2p+3
        modes = _raw_modes(kind, p, pts)
        _NORM_CACHE[key] = np.array([1.0 / np.sqrt(np.dot(w, m.v * m.v))
                                     for m in modes])
    return _NORM_CACHE[key]


def evaluate_basis(kind: ElementKind, p: int, pts):
    """(values (npts, nb), gradients (dim, npts, nb)) of the orthonormal basis."""
    modes = _raw_modes(kind, p, pts)
    nrm = _norms(kind, p)
    val = np.stack([m.v * c for m, c in zip(modes, nrm)], axis=1)
    grad = np.stack([m.g * c for m, c in zip(modes, nrm)], axis=2)
    return val, grad


# ------------------------------------------------------------ quadrature
def gauss_legendre01(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def _gj(n, alpha):
    x, w = roots_jacobi(n, alpha, 0.0)
    return np.asarray(x, dtype=np.float64), np.asarray(w, dtype=np.float64)


# Minimal symmetric degree-5 rules used for p = 2 (exact to degree 2p+1 like
# the collapsed rules they replace, with fewer points): Radon's 7-point
# triangle rule and the 14-point tetrahedron rule (Walkington).  Their
# exactness is verified in tests/test_dg_oracle.py.
_S15 = np.sqrt(15.0)
_RADON_A, _RADON_B = (6 - _S15) / 21, (9 + 2 * _S15) / 21
_RADON_C, _RADON_D = (6 + _S15) / 21, (9 - 2 * _S15) / 21
TET14 = ((0.0927352503108912, 0.01224884051939366),
         (0.3108859192633006, 0.01878132095300264),
         (0.0455037041256496, 0.007091003462846911))


def _radon7():
    pts = np.array([[1 / 3, 1 / 3], [_RADON_A, _RADON_A], [_RADON_A, _RADON_B],
                    [_RADON_B, _RADON_A], [_RADON_C, _RADON_C], [_RADON_C, _RADON_D],
                    [_RADON_D, _RADON_C]])
    w = np.array([9 / 80] + [(155 - _S15) / 2400] * 3 + [(155 + _S15) / 2400] * 3)
    return pts, w


def _tet14():
    pts, w = [], []
    for v, wv in TET14[:2]:
        for i in range(4):
            bc = [v] * 4
            bc[i] = 1 - 3 * v
            pts.append(bc[1:])
            w.append(wv)
    c, wc = TET14[2]
    for i, j in itertools.combinations(range(4), 2):
        bc = [c] * 4
        bc[i] = bc[j] = 0.5 - c
        pts.append(bc[1:])
        w.append(wc)
    return np.array(pts), np.array(w)


def volume_rule(kind: ElementKind, p: int):
    """(points (nq, dim), weights (nq,)) on the reference element."""
    if p == 2 and kind is ElementKind.TRIANGLE:
        return _radon7()
    if p == 2 and kind is ElementKind.TET:
        return _tet14()
    n = p + 1
    if kind is ElementKind.QUAD:
        t, w = gauss_legendre01(n)
        pts = np.array([(a, b) for a in t for b in t])
        wts = np.array([wa * wb for wa in w for wb in w])
        return pts, wts
    a, wa = np.polynomial.legendre.leggauss(n)
    b, wb = _gj(n, 1.0)
    if kind is ElementKind.TRIANGLE:
        pts, wts = [], []
        for ai, wai in zip(a, wa):
            for bj, wbj in zip(b, wb):
                pts.append(((1 + ai) * (1 - bj) / 4, (1 + bj) / 2))
                wts.append(wai * wbj / 8)
        return np.array(pts), np.array(wts)
    c, wc = _gj(n, 2.0)
    pts, wts = [], []
    for ai, wai in zip(a, wa):
        for bj, wbj in zip(b, wb):
            for ck, wck in zip(c, wc):
                pts.append(((1 + ai) * (1 - bj) * (1 - ck) / 8,
                            (1 + bj) * (1 - ck) / 4, (1 + ck) / 2))
                wts.append(wai * wbj * wck / 64)
    return np.array(pts), np.array(wts)


def face_rule(kind: ElementKind, p: int):
    """Surface rule in the surface's own parameters: (t (nq,1)) on edges,
    barycentric (nq, 3) on tet faces; weights sum to 1."""
    if kind is not ElementKind.TET:
        t, w = gauss_legendre01(p + 1)
        return t[:, None], w
    tri_pts, tri_w = volume_rule(ElementKind.TRIANGLE, p)
    lam = np.stack([1 - tri_pts[:, 0] - tri_pts[:, 1], tri_pts[:, 0],
                    tri_pts[:, 1]], axis=1)
    return lam, tri_w * 2.0


def face_points_ref(kind: ElementKind, code: int, fpts):
    """Reference-element coordinates of the surface quadrature points as
    seen from a side with the given code."""
    f, v = divmod(code, 6)
    side = SIDE_POSITIONS[kind][f]
    rv = REF_VERTS[kind]
    if kind is not ElementKind.TET:
        s0, s1 = EDGE_VARIANTS[v]
        s = s0 + fpts[:, 0] * (s1 - s0)
        return (1 - s)[:, None] * rv[side[0]] + s[:, None] * rv[side[1]]
    perm = FACE_PERMS[v]
    corners = np.stack([rv[side[perm[m]]] for m in range(3)])  # (3, 3)
    return fpts @ corners


@dataclass(frozen=True)
class ReferenceTables:
    kind: ElementKind
    degree: int
    n_basis: int
    n_codes: int
    face_w: np.ndarray      # (nqf,)
    face_phi: np.ndarray    # (codes, nqf, n_basis)
    vol_w: np.ndarray       # (nqv,)
    vol_phi: np.ndarray     # (nqv, n_basis)
    vol_dphi: np.ndarray    # (dim, nqv, n_basis)
    vol_pts: np.ndarray
    face_pts: np.ndarray

    def packed(self) -> np.ndarray:
        """Device table layout: face_phi | face_w | vol_phi | vol_dphi | vol_w."""
        return np.concatenate([self.face_phi.ravel(), self.face_w,
                               self.vol_phi.ravel(), self.vol_dphi.ravel(),
                               self.vol_w]).astype(np.float64)


_TABLE_CACHE: dict = {}


def _hybrid_tables(p: int) -> ReferenceTables:
    """Quad and triangle tables in one layout (``MC_KIND_HYBRID``): face
    codes = the quad's 24 then the triangle's 18, volume rows = the quad
    rule's then the triangle rule's; triangle rows are zero beyond its
    basis size.  Both kinds share the edge rule."""
    q = reference_tables(ElementKind.QUAD, p)
    t = reference_tables(ElementKind.TRIANGLE, p)
    nb = q.n_basis

    def pad(a):
        out = np.zeros(a.shape[:-1] + (nb,))
        out[..., :a.shape[-1]] = a
        return out

    assert np.array_equal(q.face_w, t.face_w)
    face_phi = np.concatenate([q.face_phi, pad(t.face_phi)], axis=0)
    vol_phi = np.concatenate([q.vol_phi, pad(t.vol_phi)], axis=0)
    vol_dphi = np.concatenate([q.vol_dphi, pad(t.vol_dphi)], axis=1)
    vol_w = np.concatenate([q.vol_w, t.vol_w])
    vol_pts = np.concatenate([q.vol_pts, t.vol_pts])
    return ReferenceTables(HYBRID, p, nb, face_phi.shape[0], q.face_w, face_phi, vol_w,
                           vol_phi, vol_dphi, vol_pts, q.face_pts)


def reference_tables(kind, p: int) -> ReferenceTables:
    key = (kind, p)
    if key in _TABLE_CACHE:
        return _TABLE_CACHE[key]
    if kind is HYBRID:
        _TABLE_CACHE[key] = _hybrid_tables(p)
        return _TABLE_CACHE[key]
    nb = basis_size(kind, p)
    vpts, vw = volume_rule(kind, p)
    fpts, fw = face_rule(kind, p)
    vphi, vdphi = evaluate_basis(kind, p, vpts)
    codes = n_face_codes(kind)
    fphi = np.zeros((codes, len(fw), nb))
    for code in range(codes):
        fphi[code] = evaluate_basis(kind, p, face_points_ref(kind, code, fpts))[0]
    t = ReferenceTables(kind, p, nb, codes, fw, fphi, vw, vphi, vdphi,
                        vpts, fpts)
    _TABLE_CACHE[key] = t
    return t
