"""Order of accuracy of the B200 DG path (independent of the oracle): a
smooth wave carried across a periodic box is an exact solution of both
linear advection and the Euler equations (constant velocity and pressure),
so the L2 error after a fixed fraction of a crossing must fall like
h^(p+1) under refinement.  This checks the discretisation itself —
quadrature, basis, flux, lifting, SSP-RK3 — not just agreement with the
numpy restatement."""

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from paper_1601_07613_b200.dg import DGOperator

pytestmark = pytest.mark.gpu


def wave_error(gen, n, p, physics):
    mesh = gen(n)
    op = DGOperator(mesh, P.color(mesh)[0], degree=p, physics=physics, period=(n, n))
    L = float(n)
    if physics == "advection":
        a = np.asarray(op.velocity[:2], dtype=float)

        def exact(t):
            def f(x):
                y = x - a * t
                return (np.sin(2 * np.pi * y[:, 0] / L) * np.cos(2 * np.pi * y[:, 1] / L))[:, None]
            return op.project(f)
    else:
        ff = np.asarray(op.farfield, dtype=float)
        rho0, a = ff[0], ff[1:3] / ff[0]
        p0 = (op.gamma - 1) * (ff[-1] - 0.5 * rho0 * (a * a).sum())

        def exact(t):
            def f(x):
                y = x - a * t
                rho = rho0 * (1 + 0.2 * np.sin(2 * np.pi * y[:, 0] / L)
                              * np.sin(2 * np.pi * y[:, 1] / L))
                return np.stack([rho, rho * a[0], rho * a[1],
                                 p0 / (op.gamma - 1) + 0.5 * rho * (a * a).sum()], axis=1)
            return op.project(f)
    T = 0.25 * L / np.linalg.norm(a)
    dt0 = op.stable_dt(0.3)
    steps = int(np.ceil(T / dt0))
    U = op.ssprk3(exact(0.0), T / steps, steps)
    err = (U - exact(T)).reshape(op.n_elements, -1)
    # orthonormal modal basis: M = |det J| I, so the L2 norm is a weighted sum
    detj = np.abs(op.surfaces.detj[op.plan.element_perm])      # user element order
    return float(np.sqrt((detj[:, None] * err ** 2).sum()))


def gen_hybrid_periodic(n):
    """Periodic conforming triangle + quad mix (``gen_hybrid_rect``)."""
    return P.gen_hybrid_rect(n, n, (True, True))


@pytest.mark.parametrize("gen,physics,p", [
    (gen_hybrid_periodic, "advection", 2),
    (gen_hybrid_periodic, "euler", 2),
    (gen_hybrid_periodic, "euler", 3),
], ids=["hybrid-adv-p2", "hybrid-euler-p2", "hybrid-euler-p3"])
def test_hybrid_convergence_rate(cuda, gen, physics, p):
    """Triangle + quad meshes converge at the design order too."""
    test_convergence_rate(cuda, gen, physics, p)


@pytest.mark.parametrize("gen,physics,p", [
    (lambda n: P.gen_tri_rect(n, n, (True, True)), "advection", 1),
    (lambda n: P.gen_tri_rect(n, n, (True, True)), "advection", 2),
    (lambda n: P.gen_quad_rect(n, n, (True, True)), "advection", 2),
    (lambda n: P.gen_tri_rect(n, n, (True, True)), "euler", 1),
    (lambda n: P.gen_tri_rect(n, n, (True, True)), "euler", 2),
    (lambda n: P.gen_quad_rect(n, n, (True, True)), "euler", 2),
    (lambda n: P.gen_tri_rect(n, n, (True, True)), "euler", 3),
    (lambda n: P.gen_quad_rect(n, n, (True, True)), "advection", 3),
], ids=["tri-adv-p1", "tri-adv-p2", "quad-adv-p2", "tri-euler-p1", "tri-euler-p2",
        "quad-euler-p2", "tri-euler-p3", "quad-adv-p3"])
def test_convergence_rate(cuda, gen, physics, p):
    ns = (16, 32, 64)
    errs = [wave_error(gen, n, p, physics) for n in ns]
    # the domain grows with n (unit cells) while the wave spans it, so the
    # resolution per wavelength doubles; errors are normalised by the domain
    rel = [e / n for e, n in zip(errs, ns)]
    rates = [np.log2(rel[i] / rel[i + 1]) for i in range(len(ns) - 1)]
    print(f"\n{physics} p={p}: rel errors {rel}, rates {rates}")
    assert rates[-1] > p + 1 - 0.35, rates
