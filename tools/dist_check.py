"""Run under torchrun: the distributed SSP-RK3 stepper
(``DGOperator.ssprk3_distributed``: ``stage_distributed`` + ``HaloExchange``
with kernel-packed send rows) through a real process group must reproduce
the single-domain ``ssprk3`` bit for bit.  With MC_DIST_BACKEND=gloo the
ranks may share one GPU (host-staged exchange): a functional check of the
code path the N>1 bench runs, not a measurement.
Writes ok / mismatch to $DIST_CHECK_OUT."""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1601_07613_b200 as P  # noqa: E402
from paper_1601_07613_b200.dg import DGOperator  # noqa: E402


def main():
    backend = os.environ.get("MC_DIST_BACKEND", "nccl")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    dist.init_process_group(backend)
    kind = os.environ.get("DIST_CHECK_KIND", "tet")
    mesh = (P.gen_tet_prism(8, 3, 3) if kind == "tet"
            else P.shuffle_elements(P.gen_tri_rect(16, 12), 1))
    col, _ = P.color(mesh)
    op = DGOperator(mesh, col, degree=2, physics="euler", world=world, rank=rank)
    U = op.initial_state("wave")
    dt = op.stable_dt(0.2)
    t = torch.tensor([dt])
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    dt = float(t.item())
    Ud = op.to_device(U)
    work = op.work_device()
    op.ssprk3_distributed(Ud, work, dt, 3)
    torch.cuda.synchronize()
    mine = Ud[: op.n_elements, : op.block_width()].cpu().numpy()
    ids = op.owned_user_ids()
    out = [None] * world
    dist.all_gather_object(out, (ids, mine))
    if rank == 0:
        single = DGOperator(mesh, col, degree=2, physics="euler")
        want = single.ssprk3(U, dt, 3).reshape(mesh.n_elements, -1)
        got = np.empty_like(want)
        for i, rows in out:
            got[i] = rows
        ok = np.array_equal(got, want) and bool(op.halo.packed_by_kernel)
        Path(os.environ.get("DIST_CHECK_OUT", "dist_check.txt")).write_text(
            "ok" if ok else f"mismatch {np.abs(got - want).max()}")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
