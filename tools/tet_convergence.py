"""Order-of-accuracy table for tets (GPU): a compact pulse carried by the
free stream (Euler: density pulse; advection: scalar pulse) through a box,
L2 error after a fixed travel, n = 8/16/32 cells per side.
Usage: python tools/tet_convergence.py [cfl] [travel]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07613_b200 as P  # noqa: E402
from paper_1601_07613_b200.dg import DGOperator  # noqa: E402


def err(n, p, physics, cfl, travel, power=6):
    mesh = P.gen_tet_prism(n, n, n)
    op = DGOperator(mesh, P.color(mesh)[0], degree=p, physics=physics)
    if physics == "euler":
        ff = np.asarray(op.farfield)
        rho0, a = ff[0], ff[1:4] / ff[0]
        p0 = (op.gamma - 1) * (ff[-1] - 0.5 * rho0 * (a * a).sum())
    else:
        a = np.asarray(op.velocity[:3])
    c0, R0 = np.full(3, 0.45 * n), 0.4 * n
    T = travel * n / np.linalg.norm(a)

    def exact(t):
        def f(x):
            r = np.linalg.norm(x - c0 - a * t, axis=1) / R0
            bump = np.where(r < 1, np.cos(0.5 * np.pi * np.minimum(r, 1)) ** power, 0.0)
            if physics != "euler":
                return bump[:, None]
            rho = rho0 * (1 + 0.2 * bump)
            out = np.empty((len(x), 5))
            out[:, 0] = rho
            out[:, 1:4] = rho[:, None] * a
            out[:, 4] = p0 / (op.gamma - 1) + 0.5 * rho * (a * a).sum()
            return out
        return op.project(f)
    steps = int(np.ceil(T / op.stable_dt(cfl)))
    U = op.ssprk3(exact(0.0), T / steps, steps)
    e = (U - exact(T)).reshape(op.n_elements, -1)
    detj = np.abs(op.surfaces.detj[op.plan.element_perm])
    return float(np.sqrt((detj[:, None] * e ** 2).sum() / detj.sum())), steps


if __name__ == "__main__":
    cfl = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
    travel = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
    ns = tuple(int(x) for x in sys.argv[3].split(",")) if len(sys.argv) > 3 else (8, 16, 32)
    degrees = tuple(int(x) for x in sys.argv[4].split(",")) if len(sys.argv) > 4 else (1, 2, 3)
    for physics in ("advection", "euler"):
        for p in degrees:
            es = [err(n, p, physics, cfl, travel) for n in ns]
            rates = [np.log2(es[i][0] / es[i + 1][0]) for i in range(len(ns) - 1)]
            print(f"{physics} p={p} cfl={cfl} travel={travel}: errors "
                  f"{[f'{e:.3e}' for e, _ in es]} steps {[s for _, s in es]} rates "
                  f"{[round(r, 2) for r in rates]}", flush=True)
