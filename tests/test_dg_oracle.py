"""Known-answer anchors for the DG oracle (the reference has no DG, so its
parity is pinned here instead: orthonormality, free-stream preservation,
discrete conservation, p+1 convergence) plus agreement of the product's
reference tables with the oracle's independent basis."""

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from oracle import dg_oracle as D
from paper_1601_07613_b200.dg.basis import evaluate_basis, reference_tables
from paper_1601_07613_b200.mesh import ElementKind as K

KINDS = {"tri": K.TRIANGLE, "quad": K.QUAD, "tet": K.TET}


def problem(mesh, col, kind, p, phys, period=None):
    return D.Problem(kind, p, phys, mesh.vertices, mesh.elem_verts, mesh.surf_verts,
                     mesh.surf_elems, col.colors, col.n_colors, np.ones(mesh.n_surfaces, bool),
                     period)


@pytest.mark.parametrize("kind,p", [("tri", 1), ("tri", 2), ("tri", 3), ("quad", 1),
                                    ("quad", 3), ("tet", 1), ("tet", 2)])
def test_basis_orthonormal_and_matches_product(kind, p):
    B = D.Basis(kind, p)
    X, W = D.vol_rule(kind, p)
    V = B.values(X)
    assert np.abs((V * W[:, None]).T @ V - np.eye(V.shape[1])).max() < 1e-13
    v2, g2 = evaluate_basis(KINDS[kind], p, X)
    assert np.abs(V - v2).max() < 1e-12
    g1 = B.gradients(X)
    assert np.abs(g1 - g2).max() < 1e-11 * max(1.0, np.abs(g1).max())
    t = reference_tables(KINDS[kind], p)
    assert np.isclose(t.vol_w.sum(), W.sum()) and np.isclose(t.face_w.sum(), 1.0)


@pytest.mark.parametrize("kind", ["tri", "quad", "tet"])
def test_free_stream_preservation(kind):
    mesh = {"tri": P.gen_tri_rect(5, 4), "quad": P.gen_quad_rect(4, 3),
            "tet": P.gen_tet_prism(2, 2, 1)}[kind]
    col, _ = P.color(mesh)
    dim = 3 if kind == "tet" else 2
    U0 = np.array([1.0, 0.3, -0.2, 0.1][: dim + 1] + [2.5])
    ph = D.Physics("euler", dim, farfield=tuple(U0))
    pr = problem(mesh, col, kind, 2, ph)
    U = D.project(pr, lambda x: np.tile(U0, (len(x), 1)))
    assert np.abs(D.rhs(pr, U)).max() < 1e-12


def test_conservation_closed_and_open():
    m = P.gen_tri_rect(8, 8, (True, True))
    col, _ = P.color(m)
    U0 = (1.0, 0.3, 0.1, 2.5)
    pr = problem(m, col, "tri", 2, D.Physics("euler", 2, farfield=U0), period=(8, 8))
    f = lambda x: np.stack([1 + 0.2 * np.sin(np.pi * x[:, 0] / 4), 0.3 + 0 * x[:, 0],
                            0.1 * np.cos(np.pi * x[:, 1] / 4), 2.5 + 0 * x[:, 0]], 1)
    R = D.rhs(pr, D.project(pr, f))
    w = D.mass_weights(pr)
    assert np.abs((w[:, None] * R[:, :, 0]).sum(0)).max() < 1e-13
    assert np.abs(R).max() > 1e-3


@pytest.mark.parametrize("kind,p", [("tri", 1), ("tri", 2), ("quad", 1), ("quad", 2)])
def test_advection_converges_at_p_plus_one(kind, p):
    gen = P.gen_tri_rect if kind == "tri" else P.gen_quad_rect
    errs = []
    for n in (6, 12):
        m = gen(n, n, (True, True))
        col, _ = P.color(m)
        pr = problem(m, col, kind, p, D.Physics("advection", 2, velocity=(1.0, 0.5, 0)),
                     period=(n, n))
        f0 = lambda x, t=0.0: (np.sin(2 * np.pi * (x[:, 0] - t) / n)
                               * np.cos(2 * np.pi * (x[:, 1] - 0.5 * t) / n))[:, None]
        U = D.project(pr, f0)
        T = n / 6
        steps = int(np.ceil(T / (0.15 / (2 * p + 1))))
        U = D.ssprk3(pr, U, T / steps, steps)
        c = D.setup(pr)
        e = U - D.project(pr, lambda x: f0(x, T))
        errs.append(np.sqrt(np.sum(np.abs(c["det"])[:, None, None] * e ** 2)) / n)
    rate = np.log2(errs[0] / errs[1])
    assert rate > p + 0.6, (errs, rate)


@pytest.mark.parametrize("kind,p", [("tri", 1), ("tri", 2), ("tri", 3), ("quad", 2), ("tet", 1),
                                    ("tet", 2), ("tet", 3)])
def test_quadrature_exactness(kind, p):
    """Volume rules integrate every monomial up to degree 2p+1 exactly; the
    product and the oracle implement the same rules."""
    from math import factorial
    from paper_1601_07613_b200.dg.basis import volume_rule
    X, W = D.vol_rule(kind, p)
    Xp, Wp = volume_rule(KINDS[kind], p)
    assert np.allclose(X, Xp, atol=1e-15) and np.allclose(W, Wp, atol=1e-15)
    dim = X.shape[1]
    import itertools
    for e in itertools.product(range(2 * p + 2), repeat=dim):
        if sum(e) > 2 * p + 1:
            continue
        num = np.sum(W * np.prod(X ** np.array(e), axis=1))
        if kind == "quad":
            exact = np.prod([1.0 / (k + 1) for k in e])
        else:
            exact = np.prod([factorial(k) for k in e]) / factorial(sum(e) + dim)
        assert abs(num - exact) < 1e-14, (e, num, exact)


# ---------------------------------------------------- hybrid (tri + quad)
def hybrid_problem(mesh, col, p, phys, kinds=None):
    ek = np.asarray(mesh.elem_kind if kinds is None else kinds)
    return D.Problem("hybrid", p, phys, mesh.vertices, mesh.elem_verts, mesh.surf_verts,
                     mesh.surf_elems, col.colors, col.n_colors, np.ones(mesh.n_surfaces, bool),
                     elem_kind=ek)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_hybrid_free_stream_preservation(p):
    from conftest import hybrid_patch
    mesh = hybrid_patch(5, 4)
    col, _ = P.color(mesh)
    U0 = (1.0, 0.3, -0.2, 2.5)
    pr = hybrid_problem(mesh, col, p, D.Physics("euler", 2, farfield=U0))
    U = D.project(pr, lambda x: np.tile(U0, (len(x), 1)))
    tri = np.asarray(mesh.elem_kind) == 0
    assert np.abs(U[tri][:, :, (p + 1) * (p + 2) // 2:]).max() == 0.0
    assert np.abs(D.rhs(pr, U)).max() < 1e-12


@pytest.mark.parametrize("kind,p", [("tri", 2), ("quad", 2), ("tri", 3)])
def test_hybrid_layout_of_a_single_kind_mesh_matches_that_kind(kind, p):
    """A pure mesh described as "hybrid" (every element of one kind, the
    coefficients quad-sized) gives the single-kind operator's residual."""
    mesh = P.gen_tri_rect(5, 4) if kind == "tri" else P.gen_quad_rect(4, 3)
    col, _ = P.color(mesh)
    ph = D.Physics("euler", 2, farfield=(1.0, 0.3, 0.1, 2.5))
    single = problem(mesh, col, kind, p, ph)
    hyb = hybrid_problem(mesh, col, p, ph)
    rng = np.random.default_rng(1)
    nb = D.Basis(kind, p).scale.size
    U = rng.normal(size=(mesh.n_elements, 4, nb)) * 0.05
    U[:, 0, 0] += 1.5
    U[:, 3, 0] += 4.0
    Uh = np.zeros((mesh.n_elements, 4, (p + 1) ** 2))
    Uh[:, :, :nb] = U
    want = D.rhs(single, U)
    got = D.rhs(hyb, Uh)
    assert np.abs(got[:, :, nb:]).max(initial=0.0) == 0.0
    assert np.abs(got[:, :, :nb] - want).max() < 1e-13 * np.abs(want).max()
