"""Surface-list layout on the host: the code-sort modes only permute the
surfaces inside a color (race freedom and per-element accumulation order are
untouched), color 1 keeps its coalesced order when windowed, and inside each
window the side codes ascend."""

import numpy as np

import paper_1601_07613_b200 as P
from paper_1601_07613_b200.dg.layout import build_surface_list


def _layout_mesh():
    mesh = P.shuffle_elements(P.gen_tet_prism(4, 3, 3), 2)
    col, _ = P.color(mesh)
    return P.apply_plan(mesh, col, P.build_plan(mesh, col))


def test_code_sort_windows_permute_within_colors():
    mesh, col = _layout_mesh()
    base = build_surface_list(mesh, col.colors, col.n_colors)
    win = 16
    for kw in (dict(code_sort=True),
               dict(code_sort=True, code_sort_window=win, code_sort_skip_first=True)):
        sl = build_surface_list(mesh, col.colors, col.n_colors, **kw)
        assert np.array_equal(sl.bounds, base.bounds)
        b = base.bounds
        for c in range(col.n_colors):
            a, e = b[c], b[c + 1]
            assert np.array_equal(np.sort(sl.mesh_surface[a:e]), np.sort(base.mesh_surface[a:e]))
        if kw.get("code_sort_skip_first"):
            assert np.array_equal(sl.mesh_surface[b[0]:b[1]], base.mesh_surface[b[0]:b[1]])
            key = sl.code.astype(np.int64) & 0xFFF
            for c in range(1, col.n_colors):          # windows start at each color
                for s0 in range(int(b[c]), int(b[c + 1]), win):
                    m = np.arange(s0, min(s0 + win, int(b[c + 1])))
                    assert (np.diff(key[m]) >= 0).all()
