"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container only (needs /root/reference; the GPU box never
reads it):

    python tests/golden/make_golden.py

For every case it imports ``meshchroma`` from /root/reference/pkg/src and
records the reference's own outputs — mesh incidence, seed-0 coloring and
report counters, reordering plan, naive/greedy colorings, splitmix64
payloads, sequential-sweep totals, surface buffers, AMR refinements — into
``<case>.npz``.  Tests compare both the oracle and the product against
these arrays, so parity is pinned to the reference, not to our restatement.
"""

from __future__ import annotations

import json
import sys
import zlib
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _crc(a, dt):
    return zlib.crc32(np.ascontiguousarray(a).astype(dt).tobytes())


def hybrid_patch(R, nx, ny):
    """Same construction as the reference tests' conftest.hybrid_patch."""
    verts = [(i, j) for j in range(ny + 1) for i in range(nx + 1)]
    vid = lambda i, j: j * (nx + 1) + i
    elems = []
    for j in range(ny):
        for i in range(nx):
            a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            if (i + j) % 2 == 0:
                elems += [("tri", (a, b, c)), ("tri", (a, c, d))]
            else:
                elems.append(("quad", (a, b, c, d)))
    return R.build_surfaces(np.asarray(verts, dtype=float), elems)


CASES = {
    # name: (builder, description)
    "tri_6x5": (lambda R: R.gen_tri_rect(6, 5), "gen_tri_rect(6,5)"),
    "tri_8x8": (lambda R: R.gen_tri_rect(8, 8), "gen_tri_rect(8,8)"),
    "tri_8x8_per": (lambda R: R.gen_tri_rect(8, 8, (True, True)),
                    "gen_tri_rect(8,8,periodic)"),
    "tri_6x6_per": (lambda R: R.gen_tri_rect(6, 6, (True, True)),
                    "gen_tri_rect(6,6,periodic)"),
    "tri_64x64": (lambda R: R.gen_tri_rect(64, 64), "c1: gen_tri_rect(64,64)"),
    "shuf_tri_64": (lambda R: R.shuffle_elements(R.gen_tri_rect(64, 64), 0),
                    "shuffle_elements(gen_tri_rect(64,64),0)"),
    "shuf_tri_16": (lambda R: R.shuffle_elements(R.gen_tri_rect(16, 16), 0),
                    "shuffle_elements(gen_tri_rect(16,16),0)"),
    "quad_5x5": (lambda R: R.gen_quad_rect(5, 5), "gen_quad_rect(5,5)"),
    "quad_16x16": (lambda R: R.gen_quad_rect(16, 16), "gen_quad_rect(16,16)"),
    "quad_4x4_per": (lambda R: R.gen_quad_rect(4, 4, (True, True)),
                     "gen_quad_rect(4,4,periodic)"),
    "tet_2x2x2": (lambda R: R.gen_tet_prism(2, 2, 2), "gen_tet_prism(2,2,2)"),
    "tet_4x4x4": (lambda R: R.gen_tet_prism(4, 4, 4), "gen_tet_prism(4,4,4)"),
    "shuf_tet_3": (lambda R: R.shuffle_elements(R.gen_tet_prism(3, 3, 3), 5),
                   "shuffle_elements(gen_tet_prism(3,3,3),5)"),
    "hybrid_4x4": (lambda R: hybrid_patch(R, 4, 4), "conftest.hybrid_patch(4,4)"),
}

# AMR cases: base mesh builder, refinement set
AMR_CASES = {
    "amr_tri_8x8": (lambda R: R.gen_tri_rect(8, 8), [0, 5, 17, 18, 40, 77, 100]),
    "amr_tri_16_disc": (lambda R: R.gen_tri_rect(16, 16), "disc"),
}


def disc_set(mesh, radius_frac=0.25):
    """Elements whose centroid lies inside a centred disc (the c5 recipe)."""
    ev = mesh.elem_verts[:, :3]
    cen = mesh.vertices[ev].mean(axis=1)
    lo, hi = mesh.vertices.min(axis=0), mesh.vertices.max(axis=0)
    c = 0.5 * (lo + hi)
    r = radius_frac * (hi - lo).min()
    return np.flatnonzero(((cen - c) ** 2).sum(axis=1) <= r * r).tolist()


def mesh_arrays(prefix, m):
    return {f"{prefix}{n}": np.asarray(getattr(m, n)) for n in (
        "vertices", "elem_kind", "elem_verts", "elem_surfs", "surf_verts",
        "surf_elems")}


def plan_arrays(prefix, p):
    return {f"{prefix}element_perm": p.element_perm,
            f"{prefix}surface_perm": p.surface_perm,
            f"{prefix}group_bounds": np.asarray(p.group_bounds, dtype=np.int64),
            f"{prefix}n_interior_first": np.int64(p.n_interior_first),
            f"{prefix}used_fallback": np.bool_(p.used_fallback)}


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    import meshchroma as R

    manifest = {"reference": str(REF_SRC), "numpy": np.__version__,
                "cases": {}}
    for name, (build, desc) in CASES.items():
        m = build(R)
        d = mesh_arrays("mesh_", m)
        col, rep = R.color(m)
        d["colors"] = col.colors
        d["n_colors"] = np.int64(col.n_colors)
        d["report"] = np.array([rep.greedy_conflicts, rep.resolutions,
                                rep.swaps, rep.loop_breaks, rep.no_swap_breaks,
                                rep.forced_reswaps, rep.restarts,
                                rep.vizing_bound], dtype=np.int64)
        d["colors_seed7"] = R.color(m, R.ColoringConfig(rng_seed=7))[0].colors
        d["greedy_colors"] = R.modified_greedy(m).colors
        stats = {}
        d["resolved_colors"] = R.resolve_conflicts(
            m, R.modified_greedy(m), stats_out=stats).colors
        d["resolved_stats"] = np.array(
            [stats[k] for k in ("resolutions", "swaps", "loop_breaks",
                                "no_swap_breaks", "forced_reswaps")], np.int64)
        nv = R.naive_greedy(m)
        d["naive_colors"] = nv.colors
        d["naive_n_colors"] = np.int64(nv.n_colors)
        plan = R.build_plan(m, col)
        d.update(plan_arrays("plan_", plan))
        nplan = R.build_plan(m, nv)
        d.update(plan_arrays("naive_plan_", nplan))
        rm, rc = R.apply_plan(m, col, plan)
        d.update(mesh_arrays("reordered_", rm))
        d["reordered_colors"] = rc.colors
        co = R.coalescing_metric(rm, rc)
        d["coalescing_after"] = np.array(
            [x for row in co.per_color for x in row[1:]] + [co.aggregate])
        for seed in (0, 3):
            pay = R.default_payload(m.n_surfaces, seed)
            d[f"payload_s{seed}"] = pay
            d[f"totals_s{seed}"] = R.sweep_sequential(m, pay).totals
        d["buffer_s0"] = R.surface_buffer(m, d["payload_s0"])
        d["reordered_totals_s0"] = R.sweep_sequential(rm, R.default_payload(
            m.n_surfaces, 0)).totals
        np.savez_compressed(OUT / f"{name}.npz", **d)
        manifest["cases"][name] = {
            "desc": desc, "ne": m.n_elements, "ns": m.n_surfaces,
            "crc_colors": _crc(col.colors, "<i4"),
            "crc_element_perm": _crc(plan.element_perm, "<i8"),
            "crc_surface_perm": _crc(plan.surface_perm, "<i8"),
            "checksum_s0": R.AccumulationState(d["totals_s0"], d["payload_s0"]).checksum(),
        }

    for name, (build, targets) in AMR_CASES.items():
        m = build(R)
        col, _ = R.color(m)
        if targets == "disc":
            targets = disc_set(m)
        ref, fine = R.refine(m, col, targets)
        d = mesh_arrays("base_", m)
        d["base_colors"] = col.colors
        d["targets"] = np.asarray(targets, dtype=np.int64)
        d.update(mesh_arrays("fine_", ref.mesh))
        d["fine_colors"] = fine.colors
        d["origin"] = ref.origin
        d["child_slot"] = ref.child_slot
        d["surf_origin"] = ref.surf_origin
        d["base_surface"] = ref.base_surface
        d["half_index"] = ref.half_index
        d["hanging"] = np.asarray(ref.hanging_interfaces(), dtype=np.int64).reshape(-1, 3)
        d["max_refined_neighbors"] = np.int64(R.max_refined_neighbors(ref))
        plan = R.build_plan(ref.mesh, fine)
        d.update(plan_arrays("plan_", plan))
        pay = R.default_payload(ref.mesh.n_surfaces, 0)
        d["payload_s0"] = pay
        d["totals_s0"] = R.sweep_sequential(ref.mesh, pay).totals
        half = sorted(targets)[: len(targets) // 2 + 1]
        back, back_col = R.coarsen(ref, fine, half)
        d["coarsened_parents"] = np.asarray(half, dtype=np.int64)
        d["coarsened_colors"] = back_col.colors
        np.savez_compressed(OUT / f"{name}.npz", **d)
        manifest["cases"][name] = {"ne_fine": ref.mesh.n_elements,
                                   "ns_fine": ref.mesh.n_surfaces,
                                   "n_hanging": len(d["hanging"])}

    # memory table (test_sweeps.py:127-142) and basis counts
    manifest["memory_table"] = [
        [p, R.memory_saved(p, 4, 3_774_165).n_bytes,
         R.memory_saved(p, 4, 3_774_165).gb_truncated] for p in range(1, 6)]
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1))
    print("wrote", len(CASES) + len(AMR_CASES), "fixtures to", OUT)


if __name__ == "__main__":
    main()
