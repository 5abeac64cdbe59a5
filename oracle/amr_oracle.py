"""AMR split-edge color rule restated (oracle).

/root/reference/pkg/src/meshchroma/amr.py:52-58 and PAPER.md §3.2:
half m (1 = the half holding the lower vertex id) of a parent edge of color
c gets ((c + 3m - 4) mod 6) + 1; interior edges copy the parallel parent
edge.  ``fine_colors`` recomputes every fine color from the fine mesh
geometry alone (midpoints and vertex ids), independent of any bookkeeping.
"""

from __future__ import annotations

import numpy as np


def child_color(c: int, m: int) -> int:
    return (c + 3 * m - 4) % 6 + 1


def fine_colors(base_surf_verts, base_colors, n_base_vertices,
                fine_surf_verts, midpoint_of):
    """midpoint_of: dict fine midpoint vertex id -> (u, w) base edge."""
    key = {(int(u), int(w)): s for s, (u, w) in enumerate(base_surf_verts)}
    out = []
    for a, b in fine_surf_verts.tolist():
        if b < n_base_vertices:                     # whole base edge
            out.append(int(base_colors[key[(a, b)]]))
        elif a < n_base_vertices:                   # half of a split edge
            u, w = midpoint_of[b]
            m = 1 if a == min(u, w) else 2
            out.append(child_color(int(base_colors[key[(min(u, w), max(u, w))]]), m))
        else:                                       # interior edge
            e1, e2 = set(midpoint_of[a]), set(midpoint_of[b])
            common = e1 & e2
            assert len(common) == 1
            x = (e1 - common).pop()
            y = (e2 - common).pop()
            out.append(int(base_colors[key[(min(x, y), max(x, y))]]))
    return np.asarray(out, dtype=np.int32)
