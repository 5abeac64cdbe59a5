"""Setup path at BASELINE config scale, pinned to the reference bit for bit.

``tests/golden/config/<cfg>.json`` holds CRC32s the REFERENCE produced
(``tests/golden/make_config_golden.py``, run in the build container) for
c2, c3, c3-shuffled, c4 and c5: mesh incidence (``mesh.py:207-300``,
``generators.py:79-197``), ``color()`` colors and every report counter
(``coloring.py:395-459``), ``build_plan`` permutations, group bounds and
fallback (``reorder.py:64-118``), the reordered mesh (``:121-167``), the
coalescing metric (``:195-221``), ``naive_greedy`` (``coloring.py:462-488``),
the c5 refinement (``amr.py:338-372``) and ``sweep_sequential`` checksums
(``sweeps.py:74-86``).  Here the PRODUCT rebuilds each config — GPU mesh
assembly, native coloring, GPU refinement, GPU Algorithm-1 sweeps — and
must reproduce every fingerprint.
"""

import json
import zlib
from pathlib import Path

import numpy as np
import pytest

import paper_1601_07613_b200 as P

pytestmark = pytest.mark.gpu

CFG_DIR = Path(__file__).resolve().parent / "golden" / "config"
CONFIGS = sorted(p.stem for p in CFG_DIR.glob("*.json"))


def crc(a, dt):
    return zlib.crc32(np.ascontiguousarray(np.asarray(a)).astype(dt).tobytes())


def mesh_crcs(m):
    return {"ne": int(m.n_elements), "ns": int(m.n_surfaces),
            "crc_elem_verts": crc(m.elem_verts, "<i8"),
            "crc_elem_surfs": crc(m.elem_surfs, "<i8"),
            "crc_surf_verts": crc(m.surf_verts, "<i8"),
            "crc_surf_elems": crc(m.surf_elems, "<i8")}


def build(cfg):
    dv = "cuda"
    if cfg == "c2":
        return P.shuffle_elements(P.gen_tri_rect(708, 708, device=dv), 0, device=dv)
    if cfg == "c3":
        return P.gen_quad_rect(2000, 2000, device=dv)
    if cfg == "c3s":
        return P.shuffle_elements(P.gen_quad_rect(2000, 2000, device=dv), 0, device=dv)
    if cfg == "c4":
        return P.gen_tet_prism(110, 110, 110, device=dv)
    if cfg == "c5":
        return P.gen_tri_rect(708, 708, device=dv)
    raise KeyError(cfg)


@pytest.mark.parametrize("cfg", CONFIGS)
def test_setup_path_matches_reference(cuda, cfg):
    want = json.loads((CFG_DIR / f"{cfg}.json").read_text())
    m = build(cfg)
    col, rep = P.color(m)
    got_rep = {k: int(getattr(rep, k)) for k in want["report"]}
    assert got_rep == want["report"]
    if cfg == "c5":
        assert mesh_crcs(m) == want["base"]
        assert crc(col.colors, "<i4") == want["base_crc_colors"]
        cen = m.vertices[m.elem_verts[:, :3]].mean(axis=1)
        tg = np.flatnonzero(((cen - 354.0) ** 2).sum(1) <= 177.0 ** 2)
        assert len(tg) == want["n_targets"] and crc(tg, "<i8") == want["crc_targets"]
        ref, fine = P.refine(m, col, tg, device="cuda")
        hang = np.asarray(ref.hanging_interfaces(), dtype=np.int64).reshape(-1, 3)
        assert len(hang) == want["n_hanging"] and crc(hang, "<i8") == want["crc_hanging"]
        assert crc(ref.origin, "<i8") == want["crc_origin"]
        assert crc(ref.surf_origin, "<i8") == want["crc_surf_origin"]
        assert int(P.max_refined_neighbors(ref)) == want["max_refined_neighbors"]
        m, col = ref.mesh, fine
    assert mesh_crcs(m) == want["mesh"]
    assert int(col.n_colors) == want["n_colors"]
    assert crc(col.colors, "<i4") == want["crc_colors"]
    assert [int(x) for x in np.bincount(col.colors)[1:]] == want["color_counts"]
    pay = P.default_payload(m.n_surfaces, 0)
    assert crc(pay, "<i8") == want["crc_payload_s0"]
    # Algorithm 1 on the GPU (colored and atomic) equals the reference's
    # sequential sweep bit for bit (integer totals)
    assert P.sweep_colored(m, col, pay).checksum() == want["checksum_s0"]
    assert P.sweep_sequential(m, pay).checksum() == want["checksum_s0"]
    plan = P.build_plan(m, col)
    wp = want["plan"]
    assert crc(plan.element_perm, "<i8") == wp["crc_element_perm"]
    assert crc(plan.surface_perm, "<i8") == wp["crc_surface_perm"]
    assert [int(x) for x in plan.group_bounds] == wp["group_bounds"]
    assert int(plan.n_interior_first) == wp["n_interior_first"]
    assert bool(plan.used_fallback) == wp["used_fallback"]
    rm, rc = P.apply_plan(m, col, plan)
    assert crc(rm.surf_elems, "<i8") == wp["reordered_crc_surf_elems"]
    assert crc(rc.colors, "<i4") == wp["reordered_crc_colors"]
    assert P.coalescing_metric(rm, rc).aggregate == pytest.approx(wp["coalescing_aggregate"],
                                                                  abs=0.0)
    assert P.sweep_colored(rm, rc, pay).checksum() == wp["reordered_checksum_s0"]
    nv = P.naive_greedy(m)
    assert int(nv.n_colors) == want["naive"]["n_colors"]
    assert crc(nv.colors, "<i4") == want["naive"]["crc_colors"]
