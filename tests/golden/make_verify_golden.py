"""Reference diagnostics of DEFECTIVE colorings (verify_coloring,
/root/reference/pkg/src/meshchroma/coloring.py:491-522).

Build container only:  python tests/golden/make_verify_golden.py
For a few golden meshes it damages the reference's own coloring (repeated
colors on an element, uncolored surfaces, both) with a fixed RNG and
records the reference's Diagnostic list -> tests/golden/verify_cases.json.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF_SRC))
    import meshchroma as R
    from meshchroma.mesh import Mesh
    cases = []
    for name in ("tri_8x8", "quad_5x5", "tet_2x2x2", "hybrid_4x4", "shuf_tri_16"):
        with np.load(OUT / f"{name}.npz") as z:
            m = Mesh(*(np.array(z["mesh_" + k]) for k in (
                "vertices", "elem_kind", "elem_verts", "elem_surfs", "surf_verts",
                "surf_elems")))
            base = np.array(z["colors"])
        rng = np.random.default_rng(len(name))
        for mode in ("repeat", "uncolor", "both"):
            cols = base.copy()
            if mode in ("repeat", "both"):
                for e in rng.choice(m.n_elements, size=3, replace=False):
                    s = m.elem_surfs[e][m.elem_surfs[e] >= 0]
                    cols[s[1]] = cols[s[0]]
            if mode in ("uncolor", "both"):
                cols[rng.choice(m.n_surfaces, size=3, replace=False)] = 0
            col = R.SurfaceColoring(cols.astype(np.int32), int(base.max()))
            diags = R.verify_coloring(m, col)
            cases.append({"mesh": name, "mode": mode, "colors": cols.tolist(),
                          "n_colors": int(base.max()),
                          "diagnostics": [[d.code, d.message, d.element_id, d.surface_id]
                                          for d in diags]})
    (OUT / "verify_cases.json").write_text(json.dumps(cases))
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
