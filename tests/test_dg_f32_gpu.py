"""fp32 state storage (the north star's "within 1e-5 (fp32)"): element
blocks of U, U0, R stored as floats, arithmetic in fp64.  Residuals and
SSP-RK3 solutions stay within 1e-5 of the fp64 oracle on every register
kernel family; the fp32 partitioned step is bit-identical to the fp32
single domain; unsupported combinations fail loudly."""

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from oracle import dg_oracle as D
from paper_1601_07613_b200.dg import DGOperator

pytestmark = pytest.mark.gpu
TOL32 = 1e-5

CASES = [
    ("tri-p2", lambda: P.shuffle_elements(P.gen_tri_rect(16, 13), 0), 2, 0),
    ("quad-p3", lambda: P.gen_quad_rect(12, 10), 3, 1),
    # two lanes per side with an odd basis size: lane runs only 8-byte aligned
    ("quad-p2", lambda: P.shuffle_elements(P.gen_quad_rect(11, 9), 1), 2, 1),
    ("tet-p2", lambda: P.gen_tet_prism(5, 4, 4), 2, 1),
    ("tet-p1", lambda: P.shuffle_elements(P.gen_tet_prism(4, 4, 3), 2), 1, 0),
]


@pytest.mark.parametrize("name,build,p,cap", CASES, ids=[c[0] for c in CASES])
def test_f32_state_within_1e5_of_oracle(cuda, name, build, p, cap):
    mesh = build()
    op = DGOperator(mesh, P.color(mesh)[0], degree=p, physics="euler", state="f32",
                    grid_cap=cap)
    prob = D.problem_from(op.oracle_problem())
    U = op.initial_state("wave")
    got = op.rhs(U)
    want = D.rhs(prob, U)
    err = D.rel_error(got, want, prob, U)
    assert 1e-12 < err < TOL32, err              # really fp32 storage, within 1e-5
    dt = op.stable_dt(0.2)
    s = op.ssprk3(U, dt, 3)
    w = D.ssprk3(prob, U, dt, 3)
    assert np.abs(s - w).max() / np.abs(w).max() < TOL32


def test_f32_partitioned_bit_identical(cuda):
    import torch
    mesh = P.gen_tet_prism(6, 3, 3)
    col, _ = P.color(mesh)
    single = DGOperator(mesh, col, degree=2, physics="euler", state="f32")
    U = single.initial_state("wave")
    dt = single.stable_dt(0.2)
    want = single.ssprk3(U, dt, 2)
    ops = [DGOperator(mesh, col, degree=2, physics="euler", world=2, rank=r, state="f32")
           for r in (0, 1)]
    Us = [op.to_device(U) for op in ops]
    assert Us[0].dtype == torch.float32
    works = [op.work_device() for op in ops]
    for _ in range(2):
        for mode, a, b in DGOperator.STAGES:
            for r, op in enumerate(ops):
                for q, (a0, b0) in op.part.recv.items():
                    Us[r][a0:b0] = Us[q][ops[q].part.send[r]]
            for op, Ud, w in zip(ops, Us, works):
                for c in range(1, op.n_colors + 1):
                    op.color_pass_device(c, Ud, w[0], w[1], mode, a, b, dt)
    torch.cuda.synchronize()
    got = np.empty_like(want)
    for op, Ud in zip(ops, Us):
        rows = Ud[: op.n_elements, : op.block_width()].double().cpu().numpy()
        got[op.owned_user_ids()] = rows.reshape(op.n_elements, op.n_equations, op.n_basis)
    # the single-domain path rounds U to float on the way in; so do the ranks
    assert np.array_equal(got, want)


def test_f32_unsupported_combinations_fail_loudly(cuda):
    mesh = P.gen_tet_prism(2, 2, 2)
    col, _ = P.color(mesh)
    with pytest.raises(NotImplementedError):        # tet p=3: group kernel, fp64 only
        DGOperator(mesh, col, degree=3, physics="euler", state="f32")
    op = DGOperator(mesh, col, degree=2, physics="euler", state="f32")
    with pytest.raises(NotImplementedError):
        op.rhs(op.initial_state("wave"), "buffered")
