"""Domain decomposition of the colored surface layout.

The path shards naturally: one ghost exchange per RK stage, no reduction.
The reference has no partitioning; this module is new.

* ``slab_owner`` — contiguous slabs of element centroids along one axis
  (x for tets, y for 2D generator meshes); balanced counts.
* ``build_partition`` — for one rank: owned elements first (ascending
  global ids of the renumbered mesh, so color-1 coalescing survives), ghost
  elements after them; local surfaces = global surfaces with an owned
  element, kept in global color-major order (the restricted coloring stays
  valid); interface surfaces whose left element is remote are flipped so
  the owned element is left and marked; the kernels evaluate every side's
  flux from its own element's view (register kernels) or in the original
  orientation (group kernel), so owned residuals are bit-identical to the
  single domain.
* ``HaloExchange`` — ghost blocks in, owned interface blocks out, with
  ``torch.distributed`` point-to-point ops (NCCL on B200s, gloo in tests),
  grouped in one ``batch_isend_irecv`` per stage; ``start``/``finish`` let
  the ghost-free part of the first color run while it is in flight.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import Mesh


def slab_owner(mesh: Mesh, world: int, axis: int | None = None, period=None) -> np.ndarray:
    """Rank of every element: equal-count slabs of centroid coordinate."""
    from .dg.layout import unwrapped_element_coords
    cen = unwrapped_element_coords(mesh, period).mean(axis=1)
    if axis is None:
        axis = 0 if mesh.dim == 3 else 1
    order = np.argsort(cen[:, axis], kind="stable")
    owner = np.empty(mesh.n_elements, dtype=np.int64)
    bounds = np.linspace(0, mesh.n_elements, world + 1).round().astype(np.int64)
    for r in range(world):
        owner[order[bounds[r]:bounds[r + 1]]] = r
    return owner


@dataclass
class Partition:
    rank: int
    world: int
    owned: np.ndarray          # global ids, ascending
    ghosts: np.ndarray         # global ids, grouped by owning rank, ascending within
    mesh: Mesh                 # local mesh: owned then ghost elements
    colors: np.ndarray         # local surface colors (non-decreasing)
    n_colors: int
    global_surface: np.ndarray  # global surface id of every local surface
    flipped: np.ndarray        # local surface had its sides swapped
    send: dict                 # peer -> local owned indices (peer's ghost order)
    recv: dict                 # peer -> (start, stop) local ghost rows

    @property
    def n_owned(self) -> int:
        return len(self.owned)

    @property
    def n_local(self) -> int:
        return len(self.owned) + len(self.ghosts)


def build_partition(mesh: Mesh, colors, n_colors: int, owner: np.ndarray,
                    rank: int) -> Partition:
    """Local view of ``rank``.  ``mesh`` must be grouped by color (a mesh
    produced by ``reorder.apply_plan``)."""
    colors = np.asarray(colors)
    world = int(owner.max()) + 1
    L = mesh.surf_elems[:, 0]
    R = mesh.surf_elems[:, 1]
    own_l = owner[L] == rank
    own_r = (R >= 0) & (owner[np.where(R >= 0, R, 0)] == rank)
    local_s = np.flatnonzero(own_l | own_r)
    owned = np.flatnonzero(owner == rank)
    touch = np.concatenate([L[local_s], R[local_s][R[local_s] >= 0]])
    ghosts = np.unique(touch[owner[touch] != rank])
    ghosts = ghosts[np.lexsort((ghosts, owner[ghosts]))]   # grouped by owner, then id
    gids = np.concatenate([owned, ghosts])
    loc = np.full(mesh.n_elements, -1, dtype=np.int64)
    loc[gids] = np.arange(len(gids))

    sl = L[local_s].copy()
    sr = R[local_s].copy()
    flip = ~own_l[local_s]                     # left is remote: owned element goes left
    sl[flip], sr[flip] = sr[flip], sl[flip]
    surf_elems = np.stack([loc[sl], np.where(sr >= 0, loc[np.where(sr >= 0, sr, 0)], -1)], 1)
    sloc = np.full(mesh.n_surfaces, -1, dtype=np.int64)
    sloc[local_s] = np.arange(len(local_s))
    es = mesh.elem_surfs[gids]
    elem_surfs = np.where(es >= 0, sloc[np.where(es >= 0, es, 0)], -1)
    local = Mesh(mesh.vertices, mesh.elem_kind[gids], mesh.elem_verts[gids], elem_surfs,
                 mesh.surf_verts[local_s], surf_elems)

    send, recv = {}, {}
    gowner = owner[ghosts]
    for q in range(world):
        if q == rank:
            continue
        sel = np.flatnonzero(gowner == q)
        if len(sel):
            recv[q] = (len(owned) + int(sel[0]), len(owned) + int(sel[-1]) + 1)
        # my owned elements that are ghosts of q: elements on surfaces shared with q
        shared = (own_l & (R >= 0) & (owner[np.where(R >= 0, R, 0)] == q)) | \
                 (own_r & (owner[L] == q))
        mine = np.unique(np.concatenate([L[shared & own_l], R[shared & own_r]]))
        if len(mine):
            send[q] = loc[mine]                 # ascending global id = q's ghost order
    return Partition(rank, world, owned, ghosts, local, colors[local_s], n_colors, local_s,
                     flip, send, recv)


class HaloExchange:
    """Grouped point-to-point ghost exchange of element blocks (rows of a
    (n_local, stride) tensor) with ``torch.distributed``."""

    def __init__(self, part: Partition, device):
        import torch
        self.part = part
        self.device = device
        self.send_idx = {q: torch.as_tensor(ix, dtype=torch.int64, device=device)
                         for q, ix in part.send.items()}

    def start(self, U):
        """Gather the owned interface rows and post all sends / receives;
        returns a handle for ``finish``.  With NCCL nothing blocks the host:
        the transfers run on NCCL's stream, ordered after the gather."""
        import torch
        import torch.distributed as dist
        ops, bufs = [], []
        for q, ix in self.send_idx.items():
            buf = U.index_select(0, ix).contiguous()
            bufs.append(buf)
            ops.append(dist.P2POp(dist.isend, buf, q))
        recv = []
        for q, (a, b) in self.part.recv.items():
            buf = torch.empty((b - a,) + tuple(U.shape[1:]), dtype=U.dtype, device=U.device)
            recv.append((a, b, buf))
            ops.append(dist.P2POp(dist.irecv, buf, q))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, recv, bufs

    def finish(self, U, handle) -> None:
        """Wait for the transfers (the current stream waits, not the host,
        with NCCL) and write the ghost rows."""
        reqs, recv, _bufs = handle
        for req in reqs:
            req.wait()
        for a, b, buf in recv:
            U[a:b] = buf

    def exchange(self, U) -> None:
        self.finish(U, self.start(U))
