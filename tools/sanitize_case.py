"""Small invocations of every kernel family, for compute-sanitizer
(tests/test_sanitizer_gpu.py): integer sweeps (colored, buffered, atomic,
race certificate), DG colored / buffered / atomic RHS and fused SSP-RK3
steps for one-lane triangles, two-lane quads and tets (per-warp flux
scratch), the tet group kernel, an AMR mesh with mortars, and a
partitioned operator with the in-kernel send-row packing.  Grids are
capped so warps loop over several tiles."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07613_b200 as P  # noqa: E402
from paper_1601_07613_b200.dg import DGOperator  # noqa: E402


def main():
    import torch
    m = P.shuffle_elements(P.gen_tri_rect(12, 10), 0)
    c, _ = P.color(m)
    pay = P.default_payload(m.n_surfaces, 0)
    a = P.sweep_colored(m, c, pay).totals
    assert np.array_equal(a, P.sweep_buffered(m, pay).totals)
    assert np.array_equal(a, P.sweep_atomic(m, pay).totals)
    cases = [(P.shuffle_elements(P.gen_tri_rect(10, 9), 1), 2),
             (P.gen_quad_rect(8, 7), 3),
             (P.gen_tet_prism(3, 3, 2), 2),
             (P.gen_tet_prism(2, 2, 1), 3)]
    for mesh, p in cases:
        for cap in (0, 1):
            op = DGOperator(mesh, P.color(mesh)[0], degree=p, physics="euler", grid_cap=cap)
            U = op.initial_state("wave")
            for s in ("colored", "buffered", "atomic"):
                assert np.isfinite(op.rhs(U, s)).all()
            assert np.isfinite(op.ssprk3(U, op.stable_dt(0.2), 2)).all()
    base = P.gen_tri_rect(8, 8)
    col, _ = P.color(base)
    ref, fine = P.refine(base, col, [0, 5, 17, 18, 40])
    op = DGOperator(ref, fine, degree=2, physics="euler")
    assert np.isfinite(op.ssprk3(op.initial_state("wave"), op.stable_dt(0.2), 1)).all()
    mesh = P.gen_tet_prism(6, 2, 2)
    colm = P.color(mesh)[0]
    ops = [DGOperator(mesh, colm, degree=2, physics="euler", world=2, rank=r) for r in (0, 1)]
    U0 = ops[0].initial_state("wave")
    for op in ops:
        Ud = torch.from_numpy(op.to_internal(U0)).cuda()
        w = op.work_device()
        for c in range(1, op.n_colors + 1):
            op.color_pass_device(c, Ud, w[0], w[1], 2, 0.0, 1.0, 1e-3)
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
