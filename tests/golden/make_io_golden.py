"""Golden fixtures for the native mesh format, made by the REFERENCE's own
meshio (/root/reference/pkg/src/meshchroma/meshio.py).  Build container
only:  python tests/golden/make_io_golden.py

* io/<case>.mesh      files written by the reference's write_native
* io/errors.json      malformed inputs with the reference's exception type
                      and message (path placeholder "<P>")
* io/msh_cases.json   MSH 2.2 inputs with the reference's read_msh result
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import meshchroma as R  # noqa: E402

OUT = Path(__file__).resolve().parent / "io"
OUT.mkdir(exist_ok=True)


def files():
    m = R.gen_tri_rect(4, 3)
    c, _ = R.color(m)
    R.write_native(OUT / "tri_4x3_colored.mesh", m, c)
    t = R.gen_tet_prism(2, 2, 2)
    tc, _ = R.color(t)
    R.write_native(OUT / "tet_2_colored.mesh", t, tc)
    q = R.gen_quad_rect(3, 2)
    parents = np.full(q.n_elements, -1, dtype=np.int64)
    parents[[1, 4]] = [0, 2]
    R.write_native(OUT / "quad_3x2_extras.mesh", q, parents=parents,
                   element_perm=np.arange(q.n_elements)[::-1].copy(),
                   surface_perm=np.roll(np.arange(q.n_surfaces), 5))
    base = R.gen_tri_rect(4, 4)
    bc, _ = R.color(base)
    ref, fine = R.refine(base, bc, [5, 6, 17])
    R.write_native(OUT / "amr_tri_4x4.mesh", ref.mesh, fine, parents=ref.parents)
    f = R.build_surfaces([(0.1 + 0.2, 0.0), (1.0 / 3.0, 1e-17), (0.5, np.pi),
                          (1e16, -2.5e-5)], [("tri", (0, 1, 2)), ("tri", (1, 3, 2))])
    R.write_native(OUT / "floats.mesh", f)


ERRORS = {
    "bad_magic": "NOTAMESH 1\n",
    "bad_version": "MESHCHROMA 9\n",
    "empty": "# nothing\n\n",
    "short_vertices": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n",
    "colors_first": "MESHCHROMA 1\nVERTICES 1\n0 0\nCOLORS 0\n",
    "zero_color": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 2\nCOLORS 3\n1\n0\n2\n",
    "not_bijection": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 2\nPERMUTATIONS 1 3\n0\n1\n1\n2\n",
    "width_1": "MESHCHROMA 1\nVERTICES 2\n0\n1\n",
    "width_mixed": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0 0\n0 1\n",
    "bad_float": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 x\n0 1 2\n",
    "empty_vertices": "MESHCHROMA 1\nVERTICES 0\nELEMENTS 0\n",
    "bad_header": "MESHCHROMA 1\nVERTICES three\n",
    "no_elements_header": "MESHCHROMA 1\nVERTICES 1\n0 0\nFACES 2\n",
    "unknown_kind": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\nhex 0 1 2\n",
    "short_element": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 2\ntri 0 1 2\ntri 0 1\n",
    "bad_element_int": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 b\n",
    "elements_eof": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 2\ntri 0 1 2\n",
    "dangling": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 7\n",
    "dup_section": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 2\nPARENTS 1\n-1\nPARENTS 1\n-1\n",
    "parents_count": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 2\nPARENTS 2\n-1\n-1\n",
    "colors_count": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 2\nCOLORS 2\n1\n2\n",
    "colors_bad_int": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 2\nCOLORS 3\n1\n2 3\n3\n",
    "colors_eof": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 2\nCOLORS 3\n1\n2\n",
    "perm_counts": "MESHCHROMA 1\nVERTICES 3\n0 0\n1 0\n0 1\nELEMENTS 1\ntri 0 1 2\nPERMUTATIONS 1\n0\n",
    "mixed_dims": "MESHCHROMA 1\nVERTICES 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nELEMENTS 2\ntri 0 1 2\ntet 0 1 2 3\n",
    "nonmanifold": "MESHCHROMA 1\nVERTICES 5\n0 0\n1 0\n0 1\n1 1\n2 2\nELEMENTS 3\ntri 0 1 2\ntri 0 1 3\ntri 0 1 4\n",
    "ok_comments": "# banner\nMESHCHROMA 1\n\nVERTICES 3  # corners\n0 0\n1 0 # x\n0 1\nELEMENTS 1\ntri 0 1 2\nCOLORS 3\n1\n-1\n3\n",
    "ok_mixed": "MESHCHROMA 1\nVERTICES 5\n0 0\n1 0\n1 1\n0 1\n2 0\nELEMENTS 2\nquad 0 1 2 3\ntri 1 4 2\nPARENTS 2\n-1\n0\nCOLORS 7\n1\n2\n3\n4\n1\n2\n5\n",
    "ok_crlf": "MESHCHROMA 1\r\nVERTICES 3\r\n0 0\r\n1 0\r\n0 1\r\nELEMENTS 1\r\ntri 0 1 2\r\n",
}


def outcome(text, reader):
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "in.mesh"
        p.write_bytes(text.encode())
        try:
            got = reader(p)
        except Exception as exc:  # noqa: BLE001
            return {"error": type(exc).__name__, "message": str(exc).replace(str(p), "<P>")}
    m = got.mesh if hasattr(got, "mesh") else got
    res = {"elem_verts": m.elem_verts.tolist(), "surf_elems": m.surf_elems.tolist(),
           "vertices": m.vertices.tolist()}
    if hasattr(got, "coloring") and got.coloring is not None:
        res["colors"] = got.coloring.colors.tolist()
        res["n_colors"] = got.coloring.n_colors
    if hasattr(got, "parents") and got.parents is not None:
        res["parents"] = got.parents.tolist()
    return res


MSH = {
    "tri": "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Comment\nanything\n$EndComment\n$Nodes\n4\n"
           "1 0 0 0\n2 1 0 0\n3 1 1 0\n4 0 1 0\n$EndNodes\n$Elements\n4\n1 15 2 0 1 1\n"
           "2 1 2 0 1 1 2\n3 2 2 0 1 1 2 3\n4 2 2 0 1 1 3 4\n$EndElements\n",
    "tet": "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n4\n10 0 0 0\n20 1 0 0\n30 0 1 0\n"
           "40 0 0 1\n$EndNodes\n$Elements\n1\n1 4 2 0 1 10 20 30 40\n$EndElements\n",
    "version": "$MeshFormat\n4.1 0 8\n$EndMeshFormat\n",
    "unknown_node": "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n3\n1 0 0 0\n2 1 0 0\n"
                    "3 1 1 0\n$EndNodes\n$Elements\n1\n1 2 2 0 1 1 2 99\n$EndElements\n",
    "bad_type": "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n1\n1 0 0 0\n$EndNodes\n"
                "$Elements\n1\n1 9 2 0 1 1\n$EndElements\n",
    "no_elements": "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n1\n1 0 0 0\n$EndNodes\n",
    "stray": "$MeshFormat\n2.2 0 8\n$EndMeshFormat\nhello\n",
    "node_width": "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n1\n1 0 0\n$EndNodes\n",
}


if __name__ == "__main__":
    files()
    (OUT / "errors.json").write_text(json.dumps(
        {k: outcome(v, R.read_native) | {"text": v} for k, v in ERRORS.items()}, indent=1))
    (OUT / "msh_cases.json").write_text(json.dumps(
        {k: outcome(v, R.read_msh) | {"text": v} for k, v in MSH.items()}, indent=1))
    print("wrote", sorted(p.name for p in OUT.iterdir()))
