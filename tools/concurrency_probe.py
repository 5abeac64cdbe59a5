"""Feasibility probe: do two half-mesh subdomains of c4 stepped on two
streams (phase-shifted, grids capped so their blocks co-reside) beat the
same launches issued back to back?  Timing only (ghost rows are filled once
and left stale).  python tools/concurrency_probe.py [config]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1601_07613_b200 as P  # noqa: E402
from paper_1601_07613_b200.dg import DGOperator  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
spec = bench.config_spec(cfg)
mesh = spec["build"]()
col, _ = P.color(mesh)
ops = [DGOperator(mesh, col, degree=spec["p"], physics=spec["physics"], world=2, rank=r)
       for r in (0, 1)]
U = ops[0].initial_state("wave")
Us, works = [], []
for op in ops:
    Ui = op.to_internal(U)
    import numpy as np
    inv = np.argsort(op.plan.element_perm)
    Ui[op.n_elements:, : op.block_width()] = U[inv[op.part.ghosts]].reshape(len(op.part.ghosts), -1)
    Us.append(torch.from_numpy(Ui).cuda())
    works.append(op.work_device())
dt = ops[0].stable_dt(0.2)
STAGES = DGOperator.STAGES


def stage_launches(r, mode, a, b, s):
    op = ops[r]
    for c in range(1, op.n_colors + 1):
        op.color_pass_device(c, Us[r], works[r][0], works[r][1], mode, a, b, dt, s)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()


def seq():
    st = torch.cuda.current_stream()
    for mode, a, b in STAGES:
        for r in (0, 1):
            stage_launches(r, mode, a, b, st)


def conc(shift):
    cur = torch.cuda.current_stream()
    s0.wait_stream(cur)
    s1.wait_stream(cur)
    # rank 1 starts `shift` colors late, then both stream their stages
    ev = []
    for k, (mode, a, b) in enumerate(STAGES):
        op = ops[0]
        for c in range(1, op.n_colors + 1):
            op.color_pass_device(c, Us[0], works[0][0], works[0][1], mode, a, b, dt, s0)
            e = torch.cuda.Event()
            e.record(s0)
            ev.append(e)
    for k, (mode, a, b) in enumerate(STAGES):
        for c in range(1, ops[1].n_colors + 1):
            if k == 0 and c == 1 and shift:
                s1.wait_event(ev[shift - 1])
            ops[1].color_pass_device(c, Us[1], works[1][0], works[1][1], mode, a, b, dt, s1)
    cur.wait_stream(s0)
    cur.wait_stream(s1)


for cap in (0, 148, 296):
    for op in ops:
        op.set_grid_cap(cap)
    t_seq = timed(seq)
    res = {sh: timed(lambda: conc(sh)) for sh in (0, 1, 2)}
    print(f"{cfg} cap {cap}: sequential {t_seq:.3f} ms/step; concurrent (shift 0/1/2 colors) "
          + " / ".join(f"{v:.3f}" for v in res.values()), flush=True)
