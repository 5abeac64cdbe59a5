"""Config-scale fingerprints of the REFERENCE's setup path (c2..c5).

Run in the build container only (needs /root/reference; the GPU box never
reads it), one config per process so they can run side by side:

    python tests/golden/make_config_golden.py c4      # -> tests/golden/config/c4.json

For each BASELINE config it builds the mesh with the reference's own
generators (``generators.py:79-197``), colors it with ``color()``
(``coloring.py:395-459``, seed 0), plans and applies the color-major layout
(``reorder.py:64-182``), refines for c5 (``amr.py:338-372``) and runs
``sweep_sequential`` (``sweeps.py:74-86``) with ``default_payload(ns, 0)``,
and records CRC32s of every array plus every report counter.  The fixtures
are tiny JSON files; ``tests/test_config_golden_gpu.py`` rebuilds the same
configs with the product (GPU assembly, C++ coloring) and compares.
"""

from __future__ import annotations

import json
import sys
import time
import zlib
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "config"


def crc(a, dt):
    return zlib.crc32(np.ascontiguousarray(np.asarray(a)).astype(dt).tobytes())


def c5_targets(base):
    """The c5 disc (bench.py config c5)."""
    cen = base.vertices[base.elem_verts[:, :3]].mean(axis=1)
    return np.flatnonzero(((cen - 354.0) ** 2).sum(1) <= 177.0 ** 2)


BUILDERS = {
    "c2": lambda R: R.shuffle_elements(R.gen_tri_rect(708, 708), 0),
    "c3": lambda R: R.gen_quad_rect(2000, 2000),
    "c3s": lambda R: R.shuffle_elements(R.gen_quad_rect(2000, 2000), 0),
    "c4": lambda R: R.gen_tet_prism(110, 110, 110),
    "c5": lambda R: R.gen_tri_rect(708, 708),
}

DESC = {
    "c2": "shuffle_elements(gen_tri_rect(708,708),0)",
    "c3": "gen_quad_rect(2000,2000)",
    "c3s": "shuffle_elements(gen_quad_rect(2000,2000),0)",
    "c4": "gen_tet_prism(110,110,110)",
    "c5": "refine(gen_tri_rect(708,708), color(seed 0), centroid disc |c-354|<=177)",
}


def mesh_crcs(m):
    return {"ne": int(m.n_elements), "ns": int(m.n_surfaces),
            "crc_elem_verts": crc(m.elem_verts, "<i8"),
            "crc_elem_surfs": crc(m.elem_surfs, "<i8"),
            "crc_surf_verts": crc(m.surf_verts, "<i8"),
            "crc_surf_elems": crc(m.surf_elems, "<i8")}


def plan_record(R, m, col):
    t = time.perf_counter()
    plan = R.build_plan(m, col)
    rm, rc = R.apply_plan(m, col, plan)
    t = time.perf_counter() - t
    co = R.coalescing_metric(rm, rc)
    pay = R.default_payload(m.n_surfaces, 0)
    return {"crc_element_perm": crc(plan.element_perm, "<i8"),
            "crc_surface_perm": crc(plan.surface_perm, "<i8"),
            "group_bounds": [int(x) for x in plan.group_bounds],
            "n_interior_first": int(plan.n_interior_first),
            "used_fallback": bool(plan.used_fallback),
            "reordered_crc_surf_elems": crc(rm.surf_elems, "<i8"),
            "reordered_crc_colors": crc(rc.colors, "<i4"),
            "coalescing_aggregate": float(co.aggregate),
            "reordered_checksum_s0": R.sweep_sequential(rm, pay).checksum(),
            "plan_seconds": round(t, 2)}


def main(cfg: str) -> None:
    sys.path.insert(0, str(REF_SRC))
    import meshchroma as R

    rec = {"config": cfg, "desc": DESC[cfg], "numpy": np.__version__}
    t = time.perf_counter()
    m = BUILDERS[cfg](R)
    rec["gen_seconds"] = round(time.perf_counter() - t, 2)
    t = time.perf_counter()
    col, rep = R.color(m)
    rec["color_seconds"] = round(time.perf_counter() - t, 2)
    rec["report"] = {k: int(getattr(rep, k)) for k in (
        "greedy_conflicts", "resolutions", "swaps", "loop_breaks", "no_swap_breaks",
        "forced_reswaps", "restarts", "vizing_bound")}
    if cfg == "c5":
        rec["base"] = mesh_crcs(m)
        rec["base_crc_colors"] = crc(col.colors, "<i4")
        tg = c5_targets(m)
        rec["n_targets"] = int(len(tg))
        rec["crc_targets"] = crc(tg, "<i8")
        t = time.perf_counter()
        ref, fine = R.refine(m, col, tg.tolist())
        rec["refine_seconds"] = round(time.perf_counter() - t, 2)
        hang = np.asarray(ref.hanging_interfaces(), dtype=np.int64).reshape(-1, 3)
        rec["n_hanging"] = int(len(hang))
        rec["crc_hanging"] = crc(hang, "<i8")
        rec["crc_origin"] = crc(ref.origin, "<i8")
        rec["crc_surf_origin"] = crc(ref.surf_origin, "<i8")
        rec["max_refined_neighbors"] = int(R.max_refined_neighbors(ref))
        m, col = ref.mesh, fine
    rec["mesh"] = mesh_crcs(m)
    rec["n_colors"] = int(col.n_colors)
    rec["crc_colors"] = crc(col.colors, "<i4")
    rec["color_counts"] = [int(x) for x in np.bincount(col.colors)[1:]]
    pay = R.default_payload(m.n_surfaces, 0)
    t = time.perf_counter()
    st = R.sweep_sequential(m, pay)
    rec["sweep_sequential_seconds"] = round(time.perf_counter() - t, 2)
    rec["checksum_s0"] = st.checksum()
    rec["crc_payload_s0"] = crc(pay, "<i8")
    rec["plan"] = plan_record(R, m, col)
    nv = R.naive_greedy(m)
    rec["naive"] = {"n_colors": int(nv.n_colors), "crc_colors": crc(nv.colors, "<i4")}
    OUT.mkdir(exist_ok=True)
    (OUT / f"{cfg}.json").write_text(json.dumps(rec, indent=1))
    print(cfg, "done", json.dumps(rec))


if __name__ == "__main__":
    for c in sys.argv[1:]:
        main(c)
