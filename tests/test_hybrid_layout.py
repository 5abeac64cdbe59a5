"""Host layout of conforming triangle + quad meshes for the DG operator
(no GPU): per-kind side codes (quads 0-23, triangles from 24), per-kind
affine geometry and centroids, race-free color-major list, and the hybrid
reference tables (quad-sized rows, triangles zero-padded)."""

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from conftest import hybrid_patch
from oracle import sweeps_oracle
from paper_1601_07613_b200.dg.basis import (HYBRID, HYBRID_TRI_CODE0, ElementKind,
                                            reference_tables)
from paper_1601_07613_b200.dg.layout import build_surface_list, mesh_kind


def layout(nx=6, ny=5, shuffle=None):
    m = hybrid_patch(nx, ny)
    if shuffle is not None:
        m = P.shuffle_elements(m, shuffle)
    c, _ = P.color(m)
    plan = P.build_plan(m, c)
    return P.apply_plan(m, c, plan)


@pytest.mark.parametrize("shuffle", [None, 3])
def test_hybrid_surface_list(shuffle):
    lm, lc = layout(shuffle=shuffle)
    assert mesh_kind(lm) is HYBRID
    sl = build_surface_list(lm, lc.colors, lc.n_colors)
    ek = sl.ekind
    assert set(np.unique(ek)) == {0, 1}
    side = [(sl.code & 63).astype(np.int64), ((sl.code >> 6) & 63).astype(np.int64)]
    for s, elems in ((0, sl.left), (1, sl.right)):
        has = elems >= 0
        tri = has & (ek[np.where(has, elems, 0)] == 0)
        assert (side[s][tri] >= HYBRID_TRI_CODE0).all()
        assert (side[s][has & ~tri] < HYBRID_TRI_CODE0).all()
    # affine maps: |det J| = 2 x area for triangles, area for unit quads
    assert np.allclose(np.abs(sl.detj[ek == 0]), 1.0) and np.allclose(np.abs(sl.detj[ek == 1]), 1.0)
    se = np.stack([sl.left, sl.right], 1).astype(np.int64)
    col = np.repeat(np.arange(1, lc.n_colors + 1), np.diff(sl.bounds))
    assert sweeps_oracle.first_race(se, col, lc.n_colors) is None
    # every normal points out of its left element (centroid test)
    from paper_1601_07613_b200.dg.layout import element_centroids, unwrapped_element_coords
    cen = element_centroids(lm, unwrapped_element_coords(lm))
    sv = lm.surf_verts[sl.mesh_surface]
    mid = lm.vertices[sv].mean(axis=1)
    assert (((mid - cen[sl.left]) * sl.geom[:, :2]).sum(1) > 0).all()


@pytest.mark.parametrize("p", [1, 2, 3])
def test_hybrid_tables(p):
    t = reference_tables(HYBRID, p)
    q = reference_tables(ElementKind.QUAD, p)
    tr = reference_tables(ElementKind.TRIANGLE, p)
    assert t.n_basis == q.n_basis and t.n_codes == HYBRID_TRI_CODE0 + tr.n_codes
    assert np.array_equal(t.face_phi[:24], q.face_phi)
    assert np.array_equal(t.face_phi[24:, :, :tr.n_basis], tr.face_phi)
    assert np.abs(t.face_phi[24:, :, tr.n_basis:]).max(initial=0.0) == 0.0
    nq = len(q.vol_w)
    assert np.array_equal(t.vol_phi[:nq], q.vol_phi)
    assert np.array_equal(t.vol_dphi[:, nq:, :tr.n_basis], tr.vol_dphi)
    assert np.isclose(t.vol_w[:nq].sum(), 1.0) and np.isclose(t.vol_w[nq:].sum(), 0.5)


@pytest.mark.parametrize("nx,ny", [(4, 4), (7, 5), (6, 9)])
def test_gen_hybrid_rect_is_the_reference_fixture_layout(nx, ny):
    """``gen_hybrid_rect`` builds the reference tests' ``hybrid_patch``
    (pkg/tests/conftest.py) element for element."""
    a, b = P.gen_hybrid_rect(nx, ny), hybrid_patch(nx, ny)
    for f in ("vertices", "elem_kind", "elem_verts", "elem_surfs", "surf_verts", "surf_elems"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    per = P.gen_hybrid_rect(nx, ny, (True, True))
    assert per.n_elements == a.n_elements and (per.surf_elems[:, 1] >= 0).all()
