import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1601_07613_b200 as P
from paper_1601_07613_b200.dg import DGOperator
mesh = P.shuffle_elements(P.gen_tri_rect(14, 11), 3)
col, _ = P.color(mesh)
single = DGOperator(mesh, col, degree=2, physics="euler")
U = single.initial_state("wave"); dt = single.stable_dt(0.2)
a = single.ssprk3(U, dt, 1)
Ud = single.to_device(U); w = single.work_device()
for mode, aa, b in DGOperator.STAGES:
    for c in range(1, single.n_colors + 1):
        single.color_pass_device(c, Ud, w[0], w[1], mode, aa, b, dt)
bb = single.from_device(Ud)
print("host vs color_pass:", np.abs(a - bb).max())
Ud = single.to_device(U); w = single.work_device()
single.ssprk3_device(Ud, w, dt, 1)
print("host vs device ssprk3:", np.abs(a - single.from_device(Ud)).max())
# one stage only, RHS compare
R1 = single.rhs(U)
ops = [DGOperator(mesh, col, degree=2, physics="euler", world=2, rank=r) for r in range(2)]
Us = [torch.from_numpy(op.to_internal(U)).cuda() for op in ops]
for r, op in enumerate(ops):
    for q, (lo, hi) in op.part.recv.items():
        Us[r][lo:hi] = Us[q][ops[q].part.send[r]]
for r, op in enumerate(ops):
    R = torch.zeros_like(Us[r])
    op.rhs_device(Us[r], R)
    rows = R[:op.n_elements, :op.block_width()].cpu().numpy().reshape(op.n_elements, 4, 6)
    d = np.abs(rows - R1[op.owned_user_ids()])
    bad = np.flatnonzero(d.reshape(len(d), -1).max(1) > 0)
    inter = set(np.flatnonzero(op.surfaces.code & (1 << 16)).tolist())
    print("rank", r, "rhs diff", d.max(), "n bad", len(bad), "of", op.n_elements)
