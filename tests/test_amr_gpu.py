"""GPU AMR color propagation (mc_amr_classify + device assembly; SURVEY
§8(f) rank 3) against the reference's golden refinements — bit-exact."""

import time

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from conftest import AMR_CASES, golden_mesh, load_golden

pytestmark = pytest.mark.gpu

MESH_FIELDS = ("vertices", "elem_kind", "elem_verts", "elem_surfs", "surf_verts", "surf_elems")
REF_FIELDS = ("origin", "child_slot", "surf_origin", "base_surface", "half_index")


@pytest.mark.parametrize("name", AMR_CASES)
def test_device_refine_matches_golden(name, cuda):
    g = load_golden(name)
    base = golden_mesh(g, "base_")
    col = P.SurfaceColoring(g["base_colors"].copy(), 3)
    ref, fine = P.refine(base, col, g["targets"].tolist(), device="cuda")
    for f in MESH_FIELDS:
        assert np.array_equal(getattr(ref.mesh, f), g["fine_" + f]), f
    assert np.array_equal(fine.colors, g["fine_colors"]) and fine.n_colors == 6
    for f in REF_FIELDS:
        assert np.array_equal(getattr(ref, f), g[f]), f
    back, back_col = P.coarsen(ref, fine, g["coarsened_parents"].tolist(), device="cuda")
    assert np.array_equal(back_col.colors, g["coarsened_colors"])


def test_device_refine_twice(cuda):
    """Second refinement request on a refined mesh (amr.py:343-356 path)."""
    m = P.gen_tri_rect(12, 12)
    c, _ = P.color(m)
    r1, f1 = P.refine(m, c, [5, 6, 40])
    coarse = [int(e) for e in np.flatnonzero(r1.child_slot < 0)[:20]]
    h2, hc = P.refine(r1, f1, coarse)
    d2, dc = P.refine(r1, f1, coarse, device="cuda")
    for f in MESH_FIELDS:
        assert np.array_equal(getattr(d2.mesh, f), getattr(h2.mesh, f)), f
    for f in REF_FIELDS:
        assert np.array_equal(getattr(d2, f), getattr(h2, f)), f
    assert np.array_equal(dc.colors, hc.colors)
    assert d2.map == h2.map


def test_device_refine_c5(cuda):
    base = P.gen_tri_rect(708, 708)
    col, _ = P.color(base)
    cen = base.vertices[base.elem_verts[:, :3]].mean(axis=1)
    tg = np.flatnonzero(((cen - 354.0) ** 2).sum(1) <= 177.0 ** 2)
    t0 = time.perf_counter()
    d, dc = P.refine(base, col, tg, device="cuda")
    t1 = time.perf_counter()
    h, hc = P.refine(base, col, tg)
    t2 = time.perf_counter()
    print(f"\nrefine c5: device {t1 - t0:.2f} s, host {t2 - t1:.2f} s")
    assert d.mesh.n_elements == 1_593_024 and d.mesh.n_surfaces == 2_392_776
    for f in MESH_FIELDS:
        assert np.array_equal(getattr(d.mesh, f), getattr(h.mesh, f)), f
    for f in REF_FIELDS:
        assert np.array_equal(getattr(d, f), getattr(h, f)), f
    assert np.array_equal(dc.colors, hc.colors)
    assert np.bincount(dc.colors)[1:].tolist() == [699007, 698929, 698984, 98628, 98610, 98618]
    assert len(d.hanging_interfaces()) == 1216
