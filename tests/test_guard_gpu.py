"""Out-of-bounds writes, checked with guard zones (compute-sanitizer is
closed on this GPU pool).  Every device array the colored kernels touch —
the state U, the RK base U0, the residual R, the partitioned send buffer —
is a view into a larger allocation whose leading and trailing guard rows
hold a NaN-payload sentinel; after residuals, fused SSP-RK3 steps, the
buffered / atomic strategies and the device permutations on every kernel
family (capped grids included) the guards must be bit-for-bit intact and
the padding columns of every element block must still be zero."""

import numpy as np
import pytest

import paper_1601_07613_b200 as P
from paper_1601_07613_b200.dg import DGOperator

pytestmark = pytest.mark.gpu
G = 64                                    # guard rows on each side
SENTINEL = np.frombuffer(np.uint64(0x7FF4DEADBEEF0001).tobytes(), dtype=np.float64)[0]

CASES = [
    ("tri-p2", lambda: P.shuffle_elements(P.gen_tri_rect(14, 11), 1), 2, 0),
    ("quad-p3", lambda: P.gen_quad_rect(9, 8), 3, 1),
    ("tet-p2", lambda: P.gen_tet_prism(4, 3, 3), 2, 1),
    ("tet-p3", lambda: P.gen_tet_prism(2, 2, 2), 3, 0),
]


def guarded(rows, cols):
    import torch
    big = torch.full((rows + 2 * G, cols), float(SENTINEL), dtype=torch.float64, device="cuda")
    return big, big[G:G + rows]


def guards_intact(big, rows):
    import torch
    torch.cuda.synchronize()
    g = torch.cat([big[:G], big[G + rows:]]).cpu().numpy()
    return np.array_equal(g.view(np.uint64), np.full(g.shape, 0x7FF4DEADBEEF0001, np.uint64))


@pytest.mark.parametrize("name,build,p,cap", CASES, ids=[c[0] for c in CASES])
def test_kernels_stay_inside_their_arrays(cuda, name, build, p, cap):
    import torch
    mesh = build()
    op = DGOperator(mesh, P.color(mesh)[0], degree=p, physics="euler", grid_cap=cap)
    n, st, W = op.n_local, op.stride, op.block_width()
    bigU, U = guarded(n, st)
    bigW, work = guarded(2 * n, st)
    work = work.view(2, n, st)
    bigR, R = guarded(n, st)
    U.copy_(torch.from_numpy(op.to_internal(op.initial_state("wave"))))
    work.zero_()
    R.zero_()
    for strat in ("colored", "buffered", "atomic"):
        op.rhs_device(U, R, strat)
    dt = op.stable_dt(0.2)
    op.ssprk3_device(U, work.reshape(2 * n, st), dt, 2)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        op.ssprk3_device(U, work.reshape(2 * n, st), dt, 1, stream=s)   # graph replay path
    s.synchronize()
    bigUs, Us = guarded(mesh.n_elements, W)
    op.device_to_user(U, Us)
    op.user_to_device(Us, U)
    assert guards_intact(bigU, n) and guards_intact(bigW, 2 * n) and guards_intact(bigR, n)
    assert guards_intact(bigUs, mesh.n_elements)
    assert torch.isfinite(U).all()
    if st > W:                                      # block padding stays zero
        assert (U[:, W:] == 0).all()


def test_send_buffer_packing_stays_inside(cuda):
    """Partitioned operator: the last-touch kernels write the interface
    rows into the send buffer and nowhere else."""
    import torch
    from paper_1601_07613_b200 import _native
    mesh = P.gen_tet_prism(6, 3, 2)
    col = P.color(mesh)[0]
    op = DGOperator(mesh, col, degree=2, physics="euler", world=2, rank=0)
    h = op.halo
    slot = h.send_slots()
    big, buf = guarded(h.n_send, op.stride)
    _native.check(op._lib.mc_dg_set_send_rows(op._h, _native.ptr(slot), _native.ptr(buf),
                                              int(h.n_send)))
    Uu = op.initial_state("wave")
    Ui = op.to_internal(Uu)
    inv = np.argsort(op.plan.element_perm)              # layout id -> user id
    Ui[op.n_elements:, : op.block_width()] = Uu[inv[op.part.ghosts]].reshape(len(op.part.ghosts), -1)
    U = torch.from_numpy(Ui).cuda()
    w = op.work_device()
    for c in range(1, op.n_colors + 1):
        op.color_pass_device(c, U, w[0], w[1], 2, 0.0, 1.0, 1e-3)
    torch.cuda.synchronize()
    assert guards_intact(big, h.n_send)
    rows = torch.as_tensor(h.rows, device="cuda")
    assert torch.isfinite(U).all()
    W = op.block_width()                     # the padding of send rows is never written
    assert torch.equal(buf[: h.n_send, :W], U.index_select(0, rows)[:, :W])
