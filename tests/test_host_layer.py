"""Product host layer (mesh assembly, generators, native coloring, plans,
AMR) against the reference's golden outputs — bit-exact."""

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from conftest import AMR_CASES, MESH_CASES, build_case, golden_mesh, load_golden, manifest

MESH_FIELDS = ("vertices", "elem_kind", "elem_verts", "elem_surfs", "surf_verts", "surf_elems")


def same_mesh(m, g, prefix):
    return all(np.array_equal(getattr(m, f), g[prefix + f]) for f in MESH_FIELDS)


@pytest.mark.parametrize("name", MESH_CASES)
def test_generators_and_assembly_match(name):
    g = load_golden(name)
    assert same_mesh(build_case(name), g, "mesh_")


@pytest.mark.parametrize("name", MESH_CASES)
def test_native_coloring_bit_exact(name):
    g = load_golden(name)
    m = golden_mesh(g)
    col, rep = P.color(m)
    assert np.array_equal(col.colors, g["colors"])
    assert col.n_colors == int(g["n_colors"])
    assert (rep.greedy_conflicts, rep.resolutions, rep.swaps, rep.loop_breaks,
            rep.no_swap_breaks, rep.forced_reswaps, rep.restarts,
            rep.vizing_bound) == tuple(int(x) for x in g["report"])
    assert rep.resolutions == rep.greedy_conflicts + rep.loop_breaks + rep.no_swap_breaks
    assert np.array_equal(P.color(m, P.ColoringConfig(rng_seed=7))[0].colors, g["colors_seed7"])
    greedy = P.modified_greedy(m)
    assert np.array_equal(greedy.colors, g["greedy_colors"])
    stats = {}
    fixed = P.resolve_conflicts(m, greedy, stats_out=stats)
    assert np.array_equal(fixed.colors, g["resolved_colors"])
    assert tuple(stats[k] for k in ("resolutions", "swaps", "loop_breaks", "no_swap_breaks",
                                    "forced_reswaps")) == tuple(g["resolved_stats"])
    nv = P.naive_greedy(m)
    assert np.array_equal(nv.colors, g["naive_colors"]) and nv.n_colors == int(g["naive_n_colors"])
    assert P.verify_coloring(m, col) == []


@pytest.mark.parametrize("name", MESH_CASES)
def test_plans_bit_exact(name):
    g = load_golden(name)
    m = golden_mesh(g)
    for pre, cols, nc in (("plan_", g["colors"], int(g["n_colors"])),
                          ("naive_plan_", g["naive_colors"], int(g["naive_n_colors"]))):
        plan = P.build_plan(m, P.SurfaceColoring(cols.copy(), nc))
        assert np.array_equal(plan.element_perm, g[pre + "element_perm"])
        assert np.array_equal(plan.surface_perm, g[pre + "surface_perm"])
        assert plan.group_bounds == tuple(int(x) for x in g[pre + "group_bounds"])
        assert plan.n_interior_first == int(g[pre + "n_interior_first"])
        assert plan.used_fallback == bool(g[pre + "used_fallback"])
    col = P.SurfaceColoring(g["colors"].copy(), int(g["n_colors"]))
    plan = P.build_plan(m, col)
    rm, rc = P.apply_plan(m, col, plan)
    assert same_mesh(rm, g, "reordered_")
    assert np.array_equal(rc.colors, g["reordered_colors"])
    co = P.coalescing_metric(rm, rc)
    assert np.allclose([x for row in co.per_color for x in row[1:]] + [co.aggregate],
                       g["coalescing_after"], rtol=0, atol=0)
    back, back_col = P.apply_plan(rm, rc, P.invert_plan(plan))
    assert np.array_equal(back.elem_verts, m.elem_verts)
    assert np.array_equal(back_col.colors, col.colors)
    assert P.validate(rm) == []


def test_appendix_b_fingerprints():
    import zlib
    for name, rec in manifest()["cases"].items():
        if name.startswith("amr_"):
            continue
        m = build_case(name)
        col, _ = P.color(m)
        plan = P.build_plan(m, col)
        assert zlib.crc32(col.colors.astype("<i4").tobytes()) == rec["crc_colors"]
        assert zlib.crc32(plan.element_perm.astype("<i8").tobytes()) == rec["crc_element_perm"]
        assert zlib.crc32(plan.surface_perm.astype("<i8").tobytes()) == rec["crc_surface_perm"]


@pytest.mark.parametrize("name", AMR_CASES)
def test_amr_bit_exact(name):
    g = load_golden(name)
    base = golden_mesh(g, "base_")
    col = P.SurfaceColoring(g["base_colors"].copy(), 3)
    ref, fine = P.refine(base, col, g["targets"].tolist())
    assert same_mesh(ref.mesh, g, "fine_")
    assert np.array_equal(fine.colors, g["fine_colors"]) and fine.n_colors == 6
    for f in ("origin", "child_slot", "surf_origin", "base_surface", "half_index"):
        assert np.array_equal(getattr(ref, f), g[f]), f
    assert np.array_equal(np.asarray(ref.hanging_interfaces()).reshape(-1, 3), g["hanging"])
    assert P.max_refined_neighbors(ref) == int(g["max_refined_neighbors"])
    plan = P.build_plan(ref.mesh, fine)
    assert np.array_equal(plan.element_perm, g["plan_element_perm"])
    assert np.array_equal(plan.surface_perm, g["plan_surface_perm"])
    assert plan.used_fallback == bool(g["plan_used_fallback"])
    back, back_col = P.coarsen(ref, fine, g["coarsened_parents"].tolist())
    assert np.array_equal(back_col.colors, g["coarsened_colors"])
    assert P.verify_coloring(ref.mesh, fine) == []


def test_memory_table():
    for p, nbytes, gb in manifest()["memory_table"]:
        est = P.memory_saved(p, n_equations=4, n_surfaces=3_774_165)
        assert est.n_bytes == nbytes and est.gb_truncated == gb
        assert est.n_basis == P.basis_count(p, "tri")
    with pytest.raises(ValueError):
        P.basis_count(-1)
    with pytest.raises(ValueError):
        P.basis_count(1, "hex")


# ---- error behaviour mirrors the reference's exception types
def test_coloring_errors():
    m = P.gen_tri_rect(8, 8)
    with pytest.raises(P.SwapBudgetExceededError):
        P.resolve_conflicts(m, P.modified_greedy(m), P.ColoringConfig(max_swaps_per_conflict=1))
    with pytest.raises(P.RestartsExhaustedError):
        P.color(P.gen_quad_rect(5, 5, (True, True)),
                P.ColoringConfig(max_swaps_per_conflict=60, max_restarts=2))
    c, _ = P.color(P.gen_tri_rect(8, 8, (True, True)), P.ColoringConfig(audit=True))
    assert c.is_complete


def test_closed_balance_and_palettes():
    c, _ = P.color(P.gen_tri_rect(6, 6, (True, True)))
    assert c.color_counts() == (36, 36, 36)
    assert P.naive_greedy(P.shuffle_elements(P.gen_tri_rect(16, 16), 0)).n_colors == 5
    for mesh, bound in ((P.gen_tri_rect(10, 10), 5), (P.gen_quad_rect(8, 8), 7),
                        (P.gen_tet_prism(3, 3, 3), 7)):
        assert P.naive_greedy(mesh).n_colors <= bound


def test_mesh_errors():
    with pytest.raises(P.NonManifoldError):
        P.build_surfaces([(0, 0), (1, 0), (0, 1), (1, 1), (2, 2)],
                         [("tri", (0, 1, 2)), ("tri", (0, 1, 3)), ("tri", (0, 1, 4))])
    with pytest.raises(P.DanglingVertexError):
        P.build_surfaces([(0, 0), (1, 0), (0, 1)], [("tri", (0, 1, 7))])
    with pytest.raises(ValueError):
        P.build_surfaces([(0, 0), (1, 0), (0, 1)], [("tri", (0, 1, 1))])


def test_plan_errors():
    m = P.gen_tri_rect(4, 4)
    c, _ = P.color(m)
    holes = c.copy()
    holes.colors[0] = -1
    with pytest.raises(ValueError):
        P.build_plan(m, holes)
    other = P.gen_tri_rect(5, 5)
    oc, _ = P.color(other)
    with pytest.raises(P.PlanMeshMismatchError):
        P.apply_plan(other, oc, P.build_plan(m, c))


def test_amr_errors():
    m = P.gen_tri_rect(3, 3)
    c, _ = P.color(m)
    ref, fine = P.refine(m, c, [4])
    child = int(np.flatnonzero(ref.child_slot >= 0)[0])
    with pytest.raises(P.LevelConstraintError):
        P.refine(ref, fine, [child])
    q = P.gen_quad_rect(2, 2)
    with pytest.raises(P.UnrefinableKindError):
        P.refine(q, P.color(q)[0], [0])
    with pytest.raises(P.PartialFamilyError):
        P.coarsen(ref, fine, [3])
    rec, rec_col = P.reconstruct_refinement(ref.mesh, ref.parents, fine)
    assert rec.map.refined == ref.map.refined
    assert np.array_equal(rec_col.colors, fine.colors)


def test_family_table_worked_example():
    """reference test_amr.py:59-72 (single triangle, colors by edge)."""
    mesh = P.build_surfaces([(0, 0), (1, 0), (0, 1)], [("tri", (0, 1, 2))])
    by_verts = {(0, 1): 2, (1, 2): 1, (0, 2): 3}
    colors = np.array([by_verts[tuple(int(v) for v in mesh.surf_verts[k])]
                       for k in range(mesh.n_surfaces)], dtype=np.int32)
    ref, fine = P.refine(mesh, P.SurfaceColoring(colors, 3), [0])
    assert ref.mesh.n_elements == 4 and ref.mesh.n_surfaces == 9
    fam = ref.map.families[0]
    assert fam == ref.map.family(0) == tuple(ref.map.families)[0]
    assert fam.parent_edge_colors == (2, 1, 3)
    assert fam.child_edge_colors == ((2, 5), (1, 4), (3, 6))
    assert fam.interior_edge_colors == (3, 2, 1)
    assert fam.children == (0, 1, 2, 3)
    assert len(ref.map.families) == 1 and ref.map.families == (fam,)


def test_verify_coloring_diagnostics_match_reference():
    """Defective colorings (repeated colors on an element, uncolored
    surfaces, both) give the reference's exact Diagnostic list
    (tests/golden/verify_cases.json, coloring.py:491-522)."""
    import json
    from conftest import GOLDEN, golden_mesh, load_golden
    cases = json.loads((GOLDEN / "verify_cases.json").read_text())
    assert len(cases) == 15
    for case in cases:
        m = golden_mesh(load_golden(case["mesh"]))
        col = P.SurfaceColoring(np.asarray(case["colors"], dtype=np.int32), case["n_colors"])
        got = [[d.code, d.message, d.element_id, d.surface_id]
               for d in P.verify_coloring(m, col)]
        assert got == case["diagnostics"], (case["mesh"], case["mode"])
        assert got    # every case is defective
