"""Two-stage fixed-palette coloring restated in plain Python (oracle).

Independent restatement of /root/reference/pkg/src/meshchroma/coloring.py:
  greedy pass          :138-166  random free color, -1 if none
  conflict repair      :207-332  FIFO walk: resolve / swap / loop-break /
                                 forced reswap, chain and total budgets
  color()              :395-459  one stream for both stages, restarts at
                                 seed + attempt
  naive_greedy         :462-488  first fit
The RNG is CPython's ``random.Random`` (the reference's stdlib dependency):
draws only when more than one option exists, options in ascending color
order, carriers searched in local side order.  Small meshes only.
"""

from __future__ import annotations

import random
from collections import deque


class BudgetExceeded(Exception):
    pass


def _colors_in(mask: int) -> list:
    return [c for c in range(1, 8) if mask >> c & 1]


class ColoringState:
    def __init__(self, surf_elems, elem_surfs, n_colors):
        self.L = [int(x) for x in surf_elems[:, 0]]
        self.R = [int(x) for x in surf_elems[:, 1]]
        self.sides = [[int(s) for s in row if s >= 0] for row in elem_surfs]
        self.nc = n_colors
        self.full = ((1 << n_colors) - 1) << 1
        self.stats = dict(resolutions=0, swaps=0, loop_breaks=0,
                          no_swap_breaks=0, forced_reswaps=0)

    # ---- helpers
    def mask(self, e):
        return self.used[e] if e >= 0 else 0

    def paint(self, s, c):
        self.col[s] = c
        for e in (self.L[s], self.R[s]):
            if e >= 0:
                self.used[e] |= 1 << c

    def erase(self, s):
        c = self.col[s]
        self.col[s] = -1
        for e in (self.L[s], self.R[s]):
            if e >= 0:
                self.used[e] &= ~(1 << c)

    def holder(self, e, c):
        for s in self.sides[e]:
            if self.col[s] == c:
                return s
        raise AssertionError("carrier missing")

    @staticmethod
    def choose(rng, options):
        return options[0] if len(options) == 1 else options[int(rng.random() * len(options))]

    # ---- stage 1
    def greedy(self, rng):
        ns = len(self.L)
        self.col = [-1] * ns
        self.used = [0] * len(self.sides)
        conflicts = []
        for s in range(ns):
            free = self.full & ~(self.mask(self.L[s]) | self.mask(self.R[s]))
            if free:
                self.paint(s, self.choose(rng, _colors_in(free)))
            else:
                conflicts.append(s)
        return conflicts

    def load(self, colors):
        self.col = [int(c) for c in colors]
        self.used = [0] * len(self.sides)
        for s, c in enumerate(self.col):
            if c >= 1:
                for e in (self.L[s], self.R[s]):
                    if e >= 0:
                        if self.used[e] >> c & 1:
                            raise ValueError(f"input coloring repeats color {c} on element {e}")
                        self.used[e] |= 1 << c
        return [s for s, c in enumerate(self.col) if c < 1]

    # ---- stage 2
    def repair(self, rng, conflicts, chain_budget, total_budget):
        pending = deque(conflicts)
        total = 0
        while pending:
            e = pending.popleft()
            if self.col[e] != -1:
                continue
            seen = {e}
            chain = 0
            while True:
                l, r = self.L[e], self.R[e]
                ul, ur = self.mask(l), self.mask(r)
                free = self.full & ~(ul | ur)
                if free:
                    self.paint(e, self.choose(rng, _colors_in(free)))
                    self.stats["resolutions"] += 1
                    break
                both = ul & ur
                single = (ul | ur) & ~both
                fresh, old, loops = [], [], []
                for c in _colors_in(single):
                    s = self.holder(l if ul >> c & 1 else r, c)
                    (old if s in seen else fresh).append((c, s))
                for c in _colors_in(both):
                    a, b = self.holder(l, c), self.holder(r, c)
                    if a != b:
                        loops.append((c, a, b))
                    else:
                        (old if a in seen else fresh).append((c, a))
                if not fresh:
                    if loops:
                        c, a, b = self.choose(rng, loops)
                        self.erase(a)
                        self.erase(b)
                        self.paint(e, c)
                        pending.extend((a, b))
                        key = "loop_breaks" if (old or single) else "no_swap_breaks"
                        self.stats[key] += 1
                        break
                    if not old:
                        raise BudgetExceeded(f"conflict on surface {e} has no admissible move")
                    fresh = old
                    self.stats["forced_reswaps"] += 1
                c, s = self.choose(rng, fresh)
                self.erase(s)
                self.paint(e, c)
                self.stats["swaps"] += 1
                chain += 1
                total += 1
                if chain > chain_budget or total > total_budget:
                    raise BudgetExceeded(
                        f"spent {chain} swaps on one conflict chain ({total} in total)")
                seen.add(s)
                e = s


def color(surf_elems, elem_surfs, n_colors, seed=0, budget=None,
          max_restarts=5):
    """Returns (colors list, stats dict incl. greedy_conflicts, restarts)."""
    ns = len(surf_elems)
    budget = 10 * ns if budget is None else budget
    last = None
    for attempt in range(max_restarts + 1):
        st = ColoringState(surf_elems, elem_surfs, n_colors)
        rng = random.Random(seed + attempt)
        conflicts = st.greedy(rng)
        try:
            st.repair(rng, conflicts, budget, 5 * budget)
        except BudgetExceeded as exc:
            last = exc
            continue
        return st.col, dict(st.stats, greedy_conflicts=len(conflicts),
                            restarts=attempt)
    raise RuntimeError(f"no complete coloring after {max_restarts + 1} attempts (last: {last})")


def greedy_only(surf_elems, elem_surfs, n_colors, seed=0):
    st = ColoringState(surf_elems, elem_surfs, n_colors)
    st.greedy(random.Random(seed))
    return st.col


def resolve(surf_elems, elem_surfs, n_colors, colors, seed=0, budget=None):
    st = ColoringState(surf_elems, elem_surfs, n_colors)
    conflicts = st.load(colors)
    budget = 10 * len(surf_elems) if budget is None else budget
    st.repair(random.Random(seed), conflicts, budget, 5 * budget)
    return st.col, st.stats


def naive_first_fit(surf_elems, n_elements):
    used = [0] * n_elements
    out = []
    for l, r in surf_elems.tolist():
        m = used[l] | (used[r] if r >= 0 else 0)
        c = 1
        while m >> c & 1:
            c += 1
        out.append(c)
        used[l] |= 1 << c
        if r >= 0:
            used[r] |= 1 << c
    return out, max(out)
