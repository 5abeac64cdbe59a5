"""DG on conforming triangle + quad meshes (the reference's hybrid meshes,
``coloring.py:38-42``, ``pkg/tests/conftest.py`` ``hybrid_patch``) on the
B200 against the fp64 oracle: one element layout (quad-sized blocks,
triangles on their first (p+1)(p+2)/2 modes), 24 quad + 18 triangle face
codes, each element's volume integral on its own rule.  Tolerance as
tests/test_dg_gpu.py (1e-12 relative to the largest term of Eq. (2))."""

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from conftest import hybrid_patch
from oracle import dg_oracle as D
from paper_1601_07613_b200.dg import DGOperator
from paper_1601_07613_b200.dg.basis import HYBRID

pytestmark = pytest.mark.gpu
TOL = 1e-12

CASES = [
    ("advection", 1, lambda: hybrid_patch(6, 5)),
    ("advection", 2, lambda: P.shuffle_elements(hybrid_patch(7, 6), 1)),
    ("advection", 3, lambda: hybrid_patch(5, 5)),
    ("euler", 1, lambda: P.shuffle_elements(hybrid_patch(6, 6), 2)),
    ("euler", 2, lambda: hybrid_patch(8, 7)),
    ("euler", 2, lambda: P.shuffle_elements(hybrid_patch(9, 8), 3)),
    ("euler", 3, lambda: hybrid_patch(6, 5)),
]


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def make(physics, p, build, **kw):
    mesh = build()
    op = DGOperator(mesh, P.color(mesh)[0], degree=p, physics=physics, **kw)
    return mesh, op, D.problem_from(op.oracle_problem())


@pytest.mark.parametrize("physics,p,build", CASES)
def test_hybrid_rhs_all_strategies_match_oracle(cuda, physics, p, build):
    mesh, op, prob = make(physics, p, build)
    assert op.kind is HYBRID and op.n_basis == (p + 1) ** 2
    U = op.initial_state("wave")
    want = D.rhs(prob, U)
    tri = np.asarray(mesh.elem_kind) == 0
    for strategy in ("colored", "buffered", "atomic"):
        got = op.rhs(U, strategy)
        assert D.rel_error(got, want, prob, U) < TOL, (strategy, rel(got, want))
        # triangle modes beyond their N_p stay exactly zero
        assert np.abs(got[tri][:, :, (p + 1) * (p + 2) // 2:]).max() == 0.0


@pytest.mark.parametrize("physics,p,build", CASES[1::2])
def test_hybrid_fused_ssprk3_matches_oracle(cuda, physics, p, build):
    mesh, op, prob = make(physics, p, build)
    U = op.initial_state("wave")
    dt = op.stable_dt(0.2)
    got = op.ssprk3(U, dt, 3)
    assert rel(got, D.ssprk3(prob, U, dt, 3)) < TOL
    tri = np.asarray(mesh.elem_kind) == 0
    assert np.abs(got[tri][:, :, (p + 1) * (p + 2) // 2:]).max() == 0.0


def test_hybrid_free_stream_and_multi_tile_grid(cuda):
    """Free stream is preserved; a capped grid (every warp loops over many
    tiles, the production loop) gives bit-identical steps."""
    mesh, op, prob = make("euler", 2, lambda: P.shuffle_elements(hybrid_patch(16, 12), 5))
    Uf = op.initial_state("freestream")
    assert np.abs(op.rhs(Uf)).max() < 1e-12
    U = op.initial_state("wave")
    dt = op.stable_dt(0.2)
    want = op.ssprk3(U, dt, 2)
    assert rel(want, D.ssprk3(prob, U, dt, 2)) < TOL
    op.set_grid_cap(1)
    assert np.array_equal(op.ssprk3(U, dt, 2), want)


@pytest.mark.parametrize("world", [2, 3])
def test_hybrid_partitioned_matches_single_domain(cuda, world):
    import torch
    from test_partition_gpu import emulated_exchange
    mesh = P.shuffle_elements(hybrid_patch(10, 8), 4)
    col, _ = P.color(mesh)
    single = DGOperator(mesh, col, degree=2, physics="euler")
    U = single.initial_state("wave")
    dt = single.stable_dt(0.2)
    want = single.ssprk3(U, dt, 2)
    ops = [DGOperator(mesh, col, degree=2, physics="euler", world=world, rank=r)
           for r in range(world)]
    Us = [torch.from_numpy(op.to_internal(U)).cuda() for op in ops]
    works = [op.work_device() for op in ops]
    for _ in range(2):
        for mode, a, b in DGOperator.STAGES:
            emulated_exchange(ops, Us)
            for op, Ud, w in zip(ops, Us, works):
                for c in range(1, op.n_colors + 1):
                    op.color_pass_device(c, Ud, w[0], w[1], mode, a, b, dt)
    torch.cuda.synchronize()
    got = np.empty_like(want)
    for op, Ud in zip(ops, Us):
        rows = Ud[: op.n_elements, : op.block_width()].cpu().numpy()
        got[op.owned_user_ids()] = rows.reshape(op.n_elements, op.n_equations, op.n_basis)
    assert np.array_equal(got, want), np.abs(got - want).max()


def test_hybrid_fp32_state_within_1e5(cuda):
    mesh, op, prob = make("euler", 2, lambda: hybrid_patch(8, 8), state="f32")
    U = op.initial_state("wave")
    dt = op.stable_dt(0.2)
    assert rel(op.ssprk3(U, dt, 2), D.ssprk3(prob, U, dt, 2)) < 1e-5


@pytest.mark.parametrize("ordering", ["sfc", "reorder", "renumber", "none"])
def test_hybrid_layouts(cuda, ordering):
    """Every element / surface layout of the operator on a hybrid mesh."""
    mesh = P.shuffle_elements(P.gen_hybrid_rect(9, 7), 2)
    op = DGOperator(mesh, P.color(mesh)[0], degree=2, physics="euler", ordering=ordering)
    prob = D.problem_from(op.oracle_problem())
    U = op.initial_state("wave")
    assert D.rel_error(op.rhs(U), D.rhs(prob, U), prob, U) < TOL
    dt = op.stable_dt(0.2)
    assert rel(op.ssprk3(U, dt, 2), D.ssprk3(prob, U, dt, 2)) < TOL
