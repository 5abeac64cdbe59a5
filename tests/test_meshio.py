"""Native mesh format + MSH 2.2 reader against files
and outcomes produced by the reference's own meshio (tests/golden/io,
made by tests/golden/make_io_golden.py)."""

import json

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from conftest import GOLDEN

IO = GOLDEN / "io"
ERRORS = json.loads((IO / "errors.json").read_text())
MSH = json.loads((IO / "msh_cases.json").read_text())


def _outcome(text, reader, tmp_path):
    p = tmp_path / "in.mesh"
    p.write_bytes(text.encode())
    try:
        got = reader(p)
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__, "message": str(exc).replace(str(p), "<P>")}
    m = got.mesh if hasattr(got, "mesh") else got
    res = {"elem_verts": m.elem_verts.tolist(), "surf_elems": m.surf_elems.tolist(),
           "vertices": m.vertices.tolist()}
    if getattr(got, "coloring", None) is not None:
        res["colors"] = got.coloring.colors.tolist()
        res["n_colors"] = got.coloring.n_colors
    if getattr(got, "parents", None) is not None:
        res["parents"] = got.parents.tolist()
    return res


@pytest.mark.parametrize("name", sorted(ERRORS))
def test_read_native_matches_reference(name, tmp_path):
    want = dict(ERRORS[name])
    text = want.pop("text")
    assert _outcome(text, P.read_native, tmp_path) == want


@pytest.mark.parametrize("name", sorted(MSH))
def test_read_msh_matches_reference(name, tmp_path):
    want = dict(MSH[name])
    text = want.pop("text")
    assert _outcome(text, P.read_msh, tmp_path) == want


def _written(tmp_path, *args, **kw):
    p = tmp_path / "out.mesh"
    P.write_native(p, *args, **kw)
    return p.read_bytes()


def test_writes_byte_identical_to_reference(tmp_path):
    m = P.gen_tri_rect(4, 3)
    assert _written(tmp_path, m, P.color(m)[0]) == (IO / "tri_4x3_colored.mesh").read_bytes()
    t = P.gen_tet_prism(2, 2, 2)
    assert _written(tmp_path, t, P.color(t)[0]) == (IO / "tet_2_colored.mesh").read_bytes()
    q = P.gen_quad_rect(3, 2)
    parents = np.full(q.n_elements, -1, dtype=np.int64)
    parents[[1, 4]] = [0, 2]
    got = _written(tmp_path, q, parents=parents,
                   element_perm=np.arange(q.n_elements)[::-1].copy(),
                   surface_perm=np.roll(np.arange(q.n_surfaces), 5))
    assert got == (IO / "quad_3x2_extras.mesh").read_bytes()
    base = P.gen_tri_rect(4, 4)
    ref, fine = P.refine(base, P.color(base)[0], [5, 6, 17])
    assert _written(tmp_path, ref.mesh, fine, parents=ref.parents) == \
        (IO / "amr_tri_4x4.mesh").read_bytes()
    f = P.build_surfaces([(0.1 + 0.2, 0.0), (1.0 / 3.0, 1e-17), (0.5, np.pi),
                          (1e16, -2.5e-5)], [("tri", (0, 1, 2)), ("tri", (1, 3, 2))])
    assert _written(tmp_path, f) == (IO / "floats.mesh").read_bytes()
    assert not list(tmp_path.glob("*.tmp*"))


@pytest.mark.parametrize("name", ["tri_4x3_colored", "tet_2_colored", "quad_3x2_extras",
                                  "amr_tri_4x4", "floats"])
def test_reference_files_round_trip(name, tmp_path):
    src = IO / f"{name}.mesh"
    nm = P.read_native(src)
    back = _written(tmp_path, nm.mesh, nm.coloring, nm.parents, nm.element_perm,
                    nm.surface_perm)
    assert back == src.read_bytes()
    if nm.coloring is not None:
        assert P.verify_coloring(nm.mesh, nm.coloring) == []


def test_amr_palette_doubles_with_parents():
    nm = P.read_native(IO / "amr_tri_4x4.mesh")
    assert nm.coloring.n_colors == 6 and (nm.parents >= 0).sum() == 12


def test_reordered_mesh_round_trip(tmp_path):
    """colors of a reordered mesh stay aligned."""
    m = P.shuffle_elements(P.gen_tri_rect(12, 9), 3)
    col, _ = P.color(m)
    plan = P.build_plan(m, col)
    rm, rc = P.apply_plan(m, col, plan)
    p = tmp_path / "r.mesh"
    P.write_native(p, rm, rc)
    back = P.read_native(p)
    assert P.verify_coloring(back.mesh, back.coloring) == []
    by_verts = {tuple(v): c for v, c in zip(rm.surf_verts.tolist(), rc.colors.tolist())}
    assert [by_verts[tuple(v)] for v in back.mesh.surf_verts.tolist()] == \
        back.coloring.colors.tolist()


def test_write_errors(tmp_path):
    m = P.gen_tri_rect(2, 2)
    with pytest.raises(ValueError):
        P.write_native(tmp_path / "x.mesh", m, element_perm=np.arange(m.n_elements))
    with pytest.raises(ValueError):
        P.write_native(tmp_path / "x.mesh", m, P.SurfaceColoring(np.ones(3, np.int32), 3))
    with pytest.raises(ValueError):
        P.write_native(tmp_path / "x.mesh", m, parents=np.zeros(3, np.int64))
    assert not list(tmp_path.iterdir())


def test_write_report(tmp_path, capsys):
    m = P.gen_tri_rect(2, 2)
    _, report = P.color(m)
    P.write_report(report)
    assert "n_colors 3" in capsys.readouterr().out
    path = tmp_path / "report.txt"
    P.write_report({"alpha": 1, "beta": "two"}, path)
    assert path.read_text() == "alpha 1\nbeta two\n"


def test_large_round_trip(tmp_path):
    m = P.gen_tet_prism(12, 12, 12)
    col, _ = P.color(m)
    p = tmp_path / "big.mesh"
    P.write_native(p, m, col)
    back = P.read_native(p)
    for f in ("vertices", "elem_kind", "elem_verts", "elem_surfs", "surf_verts", "surf_elems"):
        assert np.array_equal(getattr(back.mesh, f), getattr(m, f)), f
    assert np.array_equal(back.coloring.colors, col.colors)
