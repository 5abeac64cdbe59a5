"""Pin the oracle to the reference: every restatement in oracle/ must
reproduce the golden outputs the reference produced (tests/golden/)."""

import numpy as np
import pytest

from conftest import AMR_CASES, MESH_CASES, load_golden, manifest
from oracle import amr_oracle, coloring_oracle, mesh_oracle, plan_oracle, sweeps_oracle

MO = mesh_oracle
ORACLE_MESHES = {
    "tri_6x5": lambda: MO.gen_tri_rect(6, 5),
    "tri_8x8": lambda: MO.gen_tri_rect(8, 8),
    "tri_8x8_per": lambda: MO.gen_tri_rect(8, 8, (True, True)),
    "tri_6x6_per": lambda: MO.gen_tri_rect(6, 6, (True, True)),
    "tri_64x64": lambda: MO.gen_tri_rect(64, 64),
    "shuf_tri_64": lambda: MO.shuffle_elements(MO.gen_tri_rect(64, 64), 0),
    "shuf_tri_16": lambda: MO.shuffle_elements(MO.gen_tri_rect(16, 16), 0),
    "quad_5x5": lambda: MO.gen_quad_rect(5, 5),
    "quad_16x16": lambda: MO.gen_quad_rect(16, 16),
    "quad_4x4_per": lambda: MO.gen_quad_rect(4, 4, (True, True)),
    "tet_2x2x2": lambda: MO.gen_tet_prism(2, 2, 2),
    "tet_4x4x4": lambda: MO.gen_tet_prism(4, 4, 4),
    "shuf_tet_3": lambda: MO.shuffle_elements(MO.gen_tet_prism(3, 3, 3), 5),
}


@pytest.mark.parametrize("name", sorted(ORACLE_MESHES))
def test_mesh_oracle_matches_reference(name):
    g = load_golden(name)
    m = ORACLE_MESHES[name]()
    for k in ("vertices", "elem_kind", "elem_verts", "elem_surfs", "surf_verts", "surf_elems"):
        assert np.array_equal(m[k], g["mesh_" + k]), k


def test_mesh_oracle_c2_fingerprint():
    """c2 at full size against the reference's config-scale CRCs."""
    import json
    import zlib
    from conftest import GOLDEN
    want = json.loads((GOLDEN / "config" / "c2.json").read_text())["mesh"]
    m = MO.shuffle_elements(MO.gen_tri_rect(708, 708), 0)
    for k in ("elem_verts", "elem_surfs", "surf_verts", "surf_elems"):
        assert zlib.crc32(np.ascontiguousarray(m[k]).astype("<i8").tobytes()) == want["crc_" + k]


@pytest.mark.parametrize("name", ["tri_64x64", "shuf_tet_3", "quad_16x16"])
def test_threaded_colored_sweep_oracle(name):
    g = load_golden(name)
    ne = len(g["mesh_elem_kind"])
    for workers in (1, 3, 8):
        tot = sweeps_oracle.sweep_colored_threads(g["mesh_surf_elems"], ne, g["payload_s0"],
                                                  g["colors"], int(g["n_colors"]), workers)
        assert np.array_equal(tot, g["totals_s0"])


@pytest.mark.parametrize("name", MESH_CASES)
def test_payload_and_sequential_sweep(name):
    g = load_golden(name)
    ns = len(g["mesh_surf_verts"])
    ne = len(g["mesh_elem_kind"])
    for seed in (0, 3):
        pay = sweeps_oracle.default_payload(ns, seed)
        assert np.array_equal(pay, g[f"payload_s{seed}"])
        assert np.array_equal(sweeps_oracle.default_payload_np(ns, seed), pay)
        tot = sweeps_oracle.sweep_sequential(g["mesh_surf_elems"], ne, pay)
        assert np.array_equal(tot, g[f"totals_s{seed}"])
    assert sweeps_oracle.checksum(g["totals_s0"]) == manifest()["cases"][name]["checksum_s0"]
    loop = sweeps_oracle.sweep_sequential_loop(g["mesh_surf_elems"], ne, g["payload_s0"])
    assert np.array_equal(loop, g["totals_s0"])
    assert np.array_equal(sweeps_oracle.surface_buffer(g["mesh_surf_elems"], g["payload_s0"]),
                          g["buffer_s0"])
    buf = sweeps_oracle.sweep_buffered(g["mesh_surf_elems"], g["mesh_elem_surfs"], g["payload_s0"])
    assert np.array_equal(buf, g["totals_s0"])


@pytest.mark.parametrize("name", MESH_CASES)
def test_coloring_oracle_matches_reference(name):
    g = load_golden(name)
    nc = int(g["n_colors"])
    se, es = g["mesh_surf_elems"], g["mesh_elem_surfs"]
    cols, st = coloring_oracle.color(se, es, nc, seed=0)
    assert np.array_equal(np.asarray(cols, np.int32), g["colors"])
    rep = g["report"]
    assert (st["greedy_conflicts"], st["resolutions"], st["swaps"], st["loop_breaks"],
            st["no_swap_breaks"], st["forced_reswaps"], st["restarts"]) == tuple(rep[:7])
    cols7, _ = coloring_oracle.color(se, es, nc, seed=7)
    assert np.array_equal(np.asarray(cols7, np.int32), g["colors_seed7"])
    greedy = coloring_oracle.greedy_only(se, es, nc, seed=0)
    assert np.array_equal(np.asarray(greedy, np.int32), g["greedy_colors"])
    fixed, stats = coloring_oracle.resolve(se, es, nc, greedy, seed=0)
    assert np.array_equal(np.asarray(fixed, np.int32), g["resolved_colors"])
    assert tuple(stats[k] for k in ("resolutions", "swaps", "loop_breaks", "no_swap_breaks",
                                    "forced_reswaps")) == tuple(g["resolved_stats"])
    naive, top = coloring_oracle.naive_first_fit(se, len(es))
    assert np.array_equal(np.asarray(naive, np.int32), g["naive_colors"])
    assert top == int(g["naive_n_colors"])


@pytest.mark.parametrize("name", MESH_CASES)
def test_plan_oracle_matches_reference(name):
    g = load_golden(name)
    ne = len(g["mesh_elem_kind"])
    for pre, cols, nc in (("plan_", g["colors"], int(g["n_colors"])),
                          ("naive_plan_", g["naive_colors"], int(g["naive_n_colors"]))):
        ep, sp, bounds, n1, fb = plan_oracle.build_plan(g["mesh_surf_elems"], ne, cols, nc)
        assert np.array_equal(ep, g[pre + "element_perm"])
        assert np.array_equal(sp, g[pre + "surface_perm"])
        assert bounds == tuple(g[pre + "group_bounds"])
        assert n1 == int(g[pre + "n_interior_first"])
        assert fb == bool(g[pre + "used_fallback"])


@pytest.mark.parametrize("name", MESH_CASES)
def test_race_oracle(name):
    g = load_golden(name)
    se, cols, nc = g["mesh_surf_elems"], g["colors"], int(g["n_colors"])
    assert sweeps_oracle.first_race(se, cols, nc) is None
    bad = cols.copy()
    es = g["mesh_elem_surfs"][0]
    bad[es[1]] = bad[es[0]]
    assert sweeps_oracle.first_race(se, bad, nc) is not None


@pytest.mark.parametrize("name", AMR_CASES)
def test_amr_oracle_colors(name):
    g = load_golden(name)
    nbv = len(g["base_vertices"])
    fv = g["fine_surf_verts"]
    # recover each midpoint's base edge from coordinates alone
    bverts = g["base_vertices"]
    mids = {}
    for u, w in g["base_surf_verts"].tolist():
        key = tuple(0.5 * (bverts[u] + bverts[w]))
        mids[key] = (u, w)
    fverts = g["fine_vertices"]
    midpoint_of = {m: mids[tuple(fverts[m])] for m in range(nbv, len(fverts))}
    cols = amr_oracle.fine_colors(g["base_surf_verts"], g["base_colors"], nbv, fv, midpoint_of)
    assert np.array_equal(cols, g["fine_colors"])
    for c in (1, 2, 3):
        assert amr_oracle.child_color(c, 1) == c and amr_oracle.child_color(c, 2) == c + 3


def test_memory_table_oracle():
    for p, nbytes, gb in manifest()["memory_table"]:
        b = sweeps_oracle.memory_saved_bytes(p, 4, 3_774_165)
        assert b == nbytes and sweeps_oracle.gb_truncated(b) == gb
