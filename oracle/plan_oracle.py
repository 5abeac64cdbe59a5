"""Color-major renumbering restated with plain loops (oracle).

Follows /root/reference/pkg/src/meshchroma/reorder.py:64-118:
color-1 surfaces (interior first, then boundary) give left -> k and
right -> N1 + k; elements lacking a color-1 surface trigger the
first-occurrence fallback over colors 1..n (left before right); surface
groups >= 2 are stably sorted by new left id.
"""

from __future__ import annotations

import numpy as np


def build_plan(surf_elems, n_elements, colors, n_colors):
    left = [int(x) for x in surf_elems[:, 0]]
    right = [int(x) for x in surf_elems[:, 1]]
    colors = [int(c) for c in colors]
    ns = len(colors)
    ones = [s for s in range(ns) if colors[s] == 1]
    inner = [s for s in ones if right[s] >= 0]
    outer = [s for s in ones if right[s] < 0]
    covered = set(left[s] for s in ones) | set(right[s] for s in inner)
    fallback = len(covered) < n_elements
    ep = [-1] * n_elements
    if fallback:
        nxt = 0
        for c in range(1, n_colors + 1):
            for s in range(ns):
                if colors[s] != c:
                    continue
                for e in (left[s], right[s]):
                    if e >= 0 and ep[e] < 0:
                        ep[e] = nxt
                        nxt += 1
    else:
        order1 = inner + outer
        for k, s in enumerate(order1):
            ep[left[s]] = k
        for k, s in enumerate(inner):
            ep[right[s]] = len(order1) + k
    sp = [-1] * ns
    bounds = [0]
    nxt = 0
    for c in range(1, n_colors + 1):
        group = [s for s in range(ns) if colors[s] == c]
        if c == 1 and not fallback:
            group = inner + outer
        else:
            group = sorted(group, key=lambda s: ep[left[s]])  # stable
        for s in group:
            sp[s] = nxt
            nxt += 1
        bounds.append(nxt)
    return (np.asarray(ep, dtype=np.int64), np.asarray(sp, dtype=np.int64),
            tuple(bounds), len(inner), fallback)
