"""GPU surface extraction (mc_assemble_*) against the
reference's golden meshes and the host assembly — bit-exact ids."""

import time

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from paper_1601_07613_b200.mesh import assemble
from conftest import AMR_CASES, MESH_CASES, load_golden

pytestmark = pytest.mark.gpu

FIELDS = ("elem_surfs", "surf_verts", "surf_elems")


def same(m, ref):
    return all(np.array_equal(getattr(m, f), getattr(ref, f) if not isinstance(ref, dict)
                              else ref[f]) for f in FIELDS)


@pytest.mark.parametrize("name", MESH_CASES)
def test_device_assembly_matches_golden(name, cuda):
    g = load_golden(name)
    m = assemble(g["mesh_vertices"], g["mesh_elem_kind"], g["mesh_elem_verts"], device="cuda")
    assert same(m, {f: g["mesh_" + f] for f in FIELDS})


@pytest.mark.parametrize("name", AMR_CASES)
def test_device_assembly_matches_golden_amr(name, cuda):
    g = load_golden(name)
    m = assemble(g["fine_vertices"], g["fine_elem_kind"], g["fine_elem_verts"], device="cuda")
    assert same(m, {f: g["fine_" + f] for f in FIELDS})


def test_device_assembly_nonmanifold_message(cuda):
    verts = np.array([(0, 0), (1, 0), (0, 1), (1, 1), (2, 2)], dtype=float)
    ev = np.array([(0, 1, 2, -1), (0, 1, 3, -1), (0, 1, 4, -1)], dtype=np.int64)
    kinds = np.zeros(3, dtype=np.int8)
    with pytest.raises(P.NonManifoldError) as host:
        assemble(verts, kinds, ev)
    with pytest.raises(P.NonManifoldError) as dev:
        assemble(verts, kinds, ev, device="cuda")
    assert str(dev.value) == str(host.value)


@pytest.mark.parametrize("build", [
    lambda d: P.shuffle_elements(P.gen_tri_rect(708, 708), 0, device=d),
    lambda d: P.gen_tet_prism(110, 110, 110, device=d),
], ids=["c2", "c4"])
def test_device_assembly_fullsize(build, cuda):
    t0 = time.perf_counter()
    dev = build("cuda")
    t1 = time.perf_counter()
    host = build(None)
    t2 = time.perf_counter()
    print(f"\nassemble device {t1 - t0:.2f} s, host {t2 - t1:.2f} s, "
          f"{dev.n_surfaces} surfaces")
    assert same(dev, host)
