"""Integer Algorithm 1 on the B200: colored / buffered / atomic sweeps and
the race certificate, bit-exact against the reference's sweep_sequential
totals (golden) and the oracle.  Mirrors test_sweeps.py of the reference."""

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from conftest import MESH_CASES, AMR_CASES, golden_mesh, load_golden
from oracle import sweeps_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", MESH_CASES)
def test_three_strategies_bit_exact(cuda, name):
    g = load_golden(name)
    m = golden_mesh(g)
    col = P.SurfaceColoring(g["colors"].copy(), int(g["n_colors"]))
    for seed in (0, 3):
        pay = g[f"payload_s{seed}"]
        want = g[f"totals_s{seed}"]
        assert np.array_equal(P.sweep_colored(m, col, pay).totals, want)
        assert np.array_equal(P.sweep_buffered(m, pay).totals, want)
        assert np.array_equal(P.sweep_atomic(m, pay).totals, want)
        assert np.array_equal(P.sweep_sequential(m, pay).totals, want)
    assert np.array_equal(P.surface_buffer(m, g["payload_s0"]), g["buffer_s0"])
    st = P.sweep_colored(m, col)
    assert st.checksum() == sweeps_oracle.checksum(g["totals_s0"])


@pytest.mark.parametrize("name", MESH_CASES)
def test_reordered_mesh_uses_identity_layout(cuda, name):
    g = load_golden(name)
    m = golden_mesh(g, "reordered_")
    col = P.SurfaceColoring(g["reordered_colors"].copy(), int(g["n_colors"]))
    got = P.sweep_colored(m, col, P.default_payload(m.n_surfaces, 0)).totals
    assert np.array_equal(got, g["reordered_totals_s0"])


@pytest.mark.parametrize("name", AMR_CASES)
def test_amr_fine_mesh_sweeps(cuda, name):
    g = load_golden(name)
    m = golden_mesh(g, "fine_")
    col = P.SurfaceColoring(g["fine_colors"].copy(), 6)
    assert np.array_equal(P.sweep_colored(m, col, g["payload_s0"]).totals, g["totals_s0"])


def test_race_certificate_matches_reference_message(cuda):
    m = P.gen_tri_rect(5, 5)
    c, _ = P.color(m)
    P.assert_race_free(m, c)
    bad = c.copy()
    e = next(i for i in range(m.n_elements) if all(s >= 0 for s in m.element(i).surface_ids[:3]))
    s0, s1 = m.element(e).surface_ids[:2]
    bad.colors[s1] = bad.colors[s0]
    want = sweeps_oracle.first_race(m.surf_elems, bad.colors, bad.n_colors)
    with pytest.raises(P.WriteConflictError) as ei:
        P.assert_race_free(m, bad)
    assert str(ei.value) == f"color {want[0]} writes element {want[1]} {want[2]} times"
    with pytest.raises(P.WriteConflictError):
        P.sweep_colored(m, bad)
    P.sweep_colored(m, bad, check=False)  # no certificate: runs (racy by construction)


def test_incomplete_and_mismatched_inputs(cuda):
    m = P.gen_tri_rect(3, 3)
    c, _ = P.color(m)
    holes = c.copy()
    holes.colors[0] = -1
    with pytest.raises(ValueError):
        P.sweep_colored(m, holes)
    pay = np.arange(m.n_surfaces, dtype=np.int64)
    with pytest.raises(ValueError):
        P.sweep_sequential(m, pay[:-1])
    assert np.array_equal(P.sweep_colored(m, c, pay).totals,
                          sweeps_oracle.sweep_sequential(m.surf_elems, m.n_elements, pay))


def test_closed_and_open_totals(cuda):
    m = P.gen_tri_rect(6, 6, (True, True))
    c, _ = P.color(m)
    assert int(P.sweep_colored(m, c).totals.sum()) == 0
    m = P.gen_tri_rect(5, 4)
    st = P.sweep_colored(m, P.color(m)[0])
    boundary = m.surf_elems[:, 1] < 0
    assert int(st.totals.sum()) == int(st.payload[boundary].sum())


def test_host_entry_points_and_device_payload(cuda):
    import torch
    from paper_1601_07613_b200 import _native
    from paper_1601_07613_b200.sweeps import device_layout
    m = P.shuffle_elements(P.gen_tri_rect(40, 30), 2)
    c, _ = P.color(m)
    pay = P.default_payload(m.n_surfaces, 5)
    want = sweeps_oracle.sweep_sequential(m.surf_elems, m.n_elements, pay)
    lay = device_layout(m, c)
    for strategy in (0, 1, 2):
        lay2 = lay if strategy == 0 else device_layout(m, None)
        assert np.array_equal(lay2.sweep_host(strategy, pay), want)
    d = torch.empty(m.n_surfaces, dtype=torch.int64, device="cuda")
    _native.check(_native.lib().mc_default_payload_dev(m.n_surfaces, 5, d.data_ptr(),
                                                       _native.stream_ptr()))
    assert np.array_equal(d.cpu().numpy(), pay)


def test_larger_mesh_property(cuda):
    """c2-shaped (shuffled tri) at reduced size; exact vs the oracle."""
    m = P.shuffle_elements(P.gen_tri_rect(200, 150), 0)
    c, _ = P.color(m)
    plan = P.build_plan(m, c)
    rm, rc = P.apply_plan(m, c, plan)
    for mesh, col in ((m, c), (rm, rc)):
        pay = P.default_payload(mesh.n_surfaces, 1)
        want = sweeps_oracle.sweep_sequential(mesh.surf_elems, mesh.n_elements, pay)
        assert np.array_equal(P.sweep_colored(mesh, col, pay).totals, want)
        assert np.array_equal(P.sweep_buffered(mesh, pay).totals, want)
