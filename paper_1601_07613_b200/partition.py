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
    from .dg.layout import element_centroids, unwrapped_element_coords
    cen = element_centroids(mesh, unwrapped_element_coords(mesh, period))
    if axis is None:
        axis = 0 if mesh.dim == 3 else 1
    order = np.argsort(cen[:, axis], kind="stable")
    owner = np.empty(mesh.n_elements, dtype=np.int64)
    bounds = np.linspace(0, mesh.n_elements, world + 1).round().astype(np.int64)
    for r in range(world):
        owner[order[bounds[r]:bounds[r + 1]]] = r
    return owner


def mortar_aligned_owner(mesh: Mesh, mortars, owner: np.ndarray) -> np.ndarray:
    """``owner`` with every hanging interface made rank-local.  The coarse
    element of each (full, half_lo, half_hi) triple (left of ``full``) and
    the fine elements of its halves (``layout.py`` mortar surfaces: fine
    child left, coarse element right) are linked; each connected group
    (a corner child can hang on two coarse neighbours, a level-2 child on a
    level-1 one) moves to the rank that owns most of its elements (ties:
    the lowest rank).  Mortar surfaces then never cross a cut; only
    conforming surfaces carry ghosts."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    mortars = np.asarray(mortars, dtype=np.int64).reshape(-1, 3)
    owner = np.asarray(owner, dtype=np.int64).copy()
    if not len(mortars):
        return owner
    L = mesh.surf_elems[:, 0]
    coarse = L[mortars[:, 0]]
    a = np.concatenate([coarse, coarse])
    b = np.concatenate([L[mortars[:, 1]], L[mortars[:, 2]]])
    ne = mesh.n_elements
    g = coo_matrix((np.ones(len(a)), (a, b)), shape=(ne, ne))
    _, comp = connected_components(g, directed=False)
    linked = np.zeros(ne, dtype=bool)
    linked[a] = linked[b] = True
    ids = np.flatnonzero(linked)
    world = int(owner.max()) + 1
    votes = np.zeros((comp.max() + 1, world), dtype=np.int64)
    np.add.at(votes, (comp[ids], owner[ids]), 1)
    owner[ids] = votes.argmax(axis=1)[comp[ids]]
    return owner


def local_mortars(part: "Partition", mortars) -> np.ndarray:
    """The hanging triples of ``part``'s owned coarse elements in its local
    surface ids (all three surfaces are local after
    ``mortar_aligned_owner``)."""
    mortars = np.asarray(mortars, dtype=np.int64).reshape(-1, 3)
    loc = np.full(int(max(part.global_surface.max(initial=-1), mortars.max(initial=-1))) + 1, -1,
                  dtype=np.int64)
    loc[part.global_surface] = np.arange(len(part.global_surface))
    m = loc[mortars]
    keep = (m >= 0).any(axis=1)
    if not (m[keep] >= 0).all():
        raise AssertionError("hanging interface split across ranks")
    m = m[keep]
    if (part.mesh.surf_elems[m[:, 0], 0] >= part.n_owned).any():
        raise AssertionError("coarse element of a local hanging interface is a ghost")
    return m


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
    (n_local, stride) tensor) with ``torch.distributed``.

    Sends go out of one persistent buffer, the owned interface rows grouped
    by peer (each peer's rows in its ghost order); receives land directly in
    the ghost rows of U (contiguous per peer), so nothing is copied after
    the transfer.  With ``attach(op)`` the operator's last-touch passes
    write every interface element's updated block into its send-buffer row
    (``mc_dg_set_send_rows``), so a stage that follows an RK stage posts the
    buffer as is; otherwise ``start`` gathers it first."""

    def __init__(self, part: Partition, device):
        import torch
        self.part = part
        self.device = device
        self.peers = sorted(part.send)
        self.offs, n = {}, 0
        for q in self.peers:
            self.offs[q] = (n, n + len(part.send[q]))
            n += len(part.send[q])
        rows = (np.concatenate([part.send[q] for q in self.peers]) if self.peers
                else np.zeros(0, dtype=np.int64))
        self.rows = rows
        self.n_send = n
        self.send_idx = torch.as_tensor(rows, dtype=torch.int64, device=device)
        self.send_buf = None
        self.packed_by_kernel = False
        self.fresh = False

    def _buffer(self, U):
        import torch
        if self.send_buf is None or self.send_buf.shape[1:] != U.shape[1:]:
            self.send_buf = torch.empty((max(self.n_send, 1),) + tuple(U.shape[1:]),
                                        dtype=U.dtype, device=U.device)
        return self.send_buf

    def send_slots(self) -> np.ndarray | None:
        """Send-buffer row of every owned element (-1: not sent), or None
        when some element goes to several peers (a slab one layer thick)."""
        if self.n_send == 0 or len(np.unique(self.rows)) != len(self.rows):
            return None
        slot = np.full(self.part.n_owned, -1, dtype=np.int32)
        slot[self.rows] = np.arange(self.n_send, dtype=np.int32)
        return slot

    def attach(self, op, stride: int) -> bool:
        """Let ``op``'s last-touch passes fill the send buffer."""
        import torch
        from . import _native
        slot = self.send_slots()
        if slot is None:
            return False
        buf = self._buffer(torch.empty((0, stride), dtype=getattr(op, "torch_dtype", torch.float64),
                                       device=self.device))
        _native.check(op._lib.mc_dg_set_send_rows(op._h, _native.ptr(slot), _native.ptr(buf),
                                                  int(self.n_send)))
        self.packed_by_kernel = True
        return True

    def stage_done(self, rk: bool) -> None:
        """Called after a stage's color passes: with ``rk`` (an RK stage,
        last touches updated U) the kernel-packed buffer is current."""
        self.fresh = self.packed_by_kernel and rk

    def start(self, U):
        """Post all sends / receives; returns a handle for ``finish``.  With
        NCCL nothing blocks the host: the transfers run on NCCL's stream,
        ordered after the work already on the current stream."""
        import torch
        import torch.distributed as dist
        buf = self._buffer(U)
        if not self.fresh and self.n_send:
            torch.index_select(U, 0, self.send_idx, out=buf[: self.n_send])
        self.fresh = False
        # a CPU backend (gloo) with device tensors: stage through host memory
        staged = U.is_cuda and dist.get_backend() != "nccl"
        if staged:
            buf = buf.cpu()
        ops, landing = [], []
        for q in self.peers:
            a, b = self.offs[q]
            ops.append(dist.P2POp(dist.isend, buf[a:b], q))
        for q, (a, b) in self.part.recv.items():
            dst = torch.empty((b - a,) + tuple(U.shape[1:]), dtype=U.dtype) if staged else U[a:b]
            landing.append((a, b, dst))
            ops.append(dist.P2POp(dist.irecv, dst, q))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, (landing if staged else None), buf

    def finish(self, U, handle) -> None:
        """Wait for the transfers (with NCCL the current stream waits, not
        the host); the ghost rows are already in place (host-staged
        backends: copied in here)."""
        reqs, landing, _buf = handle
        for req in reqs:
            req.wait()
        for a, b, dst in landing or ():
            U[a:b].copy_(dst)

    def exchange(self, U) -> None:
        self.finish(U, self.start(U))


class HaloPush:
    """Peer-push ghost exchange fused into the last-touch kernel (one node,
    NVLink / NVSwitch peer memory): instead of packing a send buffer and
    posting NCCL transfers, every rank's last-touch pass of an RK stage
    stores each interface element's updated block straight into the peers'
    ghost rows (``mc_dg_set_push_rows``).  Ghost rows are double-buffered
    (ghost g at rows n_owned + 2g + parity, ``mc_dg_set_ghost_parity``):
    stage s reads parity s % 2 and pushes parity (s + 1) % 2, so with one
    barrier per stage (all ranks finished stage s - 1) no rank can
    overwrite ghosts a peer is still reading.  The state array therefore
    has ``n_owned + 2 * n_ghosts`` rows.

    ``layout[q] = (n_owned_q, recv_q)`` describes every peer q (its owned
    count and its ``Partition.recv``), which each rank learns with one
    ``all_gather_object`` (or, emulated, from the other ranks' partitions)."""

    def __init__(self, part: Partition, layout: dict):
        self.part = part
        self.layout = layout
        self.peers = sorted(part.send)
        for q in self.peers:
            if part.rank not in layout[q][1]:
                raise ValueError(f"peer {q} receives nothing from rank {part.rank}")

    @staticmethod
    def state_rows(part: Partition) -> int:
        return part.n_owned + 2 * len(part.ghosts)

    def ghost_row(self, q: int, k: int, parity: int = 0) -> int:
        """Row of peer q's state array holding the k-th block this rank
        sends q (q's ghost order), in the given parity copy."""
        ne_q, recv_q = self.layout[q]
        a_q, _ = recv_q[self.part.rank]
        return ne_q + 2 * (a_q - ne_q + k) + parity

    def destinations(self, bases: dict, stride: int, esize: int):
        """CSR (ptr (n_owned+1,), dst (nnz,) uint64 byte addresses of the
        parity-0 rows) for ``mc_dg_set_push_rows``; ``bases[q]`` = the
        address of peer q's state array as mapped in this process."""
        per = [[] for _ in range(self.part.n_owned)]
        for q in self.peers:
            for k, e in enumerate(self.part.send[q]):
                per[int(e)].append(int(bases[q]) + self.ghost_row(q, k) * stride * esize)
        ptr = np.zeros(self.part.n_owned + 1, dtype=np.int64)
        ptr[1:] = np.cumsum([len(x) for x in per])
        dst = np.asarray([a for x in per for a in x], dtype=np.uint64)
        return ptr, dst

    def fill(self, U, peers: dict, parity: int = 0) -> None:
        """Write this rank's current interface blocks into the peers' ghost
        rows of the given parity (``peers[q]``: a tensor view of peer q's
        state array, mapped peer memory); the run's first stage needs it."""
        import torch
        for q in self.peers:
            rows = torch.as_tensor([self.ghost_row(q, k, parity)
                                    for k in range(len(self.part.send[q]))],
                                   dtype=torch.int64, device=U.device)
            src = torch.as_tensor(self.part.send[q], dtype=torch.int64, device=U.device)
            peers[q].index_copy_(0, rows, U.index_select(0, src))


def setup_symmetric_push(op, group=None):
    """Multi-GPU wiring of ``HaloPush`` on one node: the state array is
    allocated in torch symmetric memory (every rank maps every peer's copy
    over NVLink / NVSwitch), peer layouts are exchanged once, the
    operator's last-touch kernel gets the peers' ghost-row addresses, and
    the stage barrier is symmetric memory's device-side barrier (signal
    pads, no host round trip).  Returns ``(U, fill, barrier)``:
    ``fill(parity)`` writes this rank's current interface blocks into the
    peers' ghost rows of that parity and waits for every rank (call it
    after loading a state, with the parity ``stage % 2`` of the next
    ``stage_push``); ``barrier()`` is the
    per-stage barrier for ``stage_push``.  Single node only; written for an
    8-GPU NVSwitch box, exercised here only through the single-process
    emulation (tests/test_partition_gpu.py)."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    group = group or dist.group.WORLD
    rows = torch.tensor([HaloPush.state_rows(op.part)], device="cuda")
    dist.all_reduce(rows, op=dist.ReduceOp.MAX, group=group)
    if hasattr(symm_mem, "enable_symm_mem_for_group"):
        try:
            symm_mem.enable_symm_mem_for_group(group.group_name)
        except Exception:
            pass
    U = symm_mem.empty(int(rows.item()), op.stride, dtype=op.torch_dtype, device="cuda")
    U.zero_()
    hdl = symm_mem.rendezvous(U, group)
    infos = [None] * dist.get_world_size(group)
    dist.all_gather_object(infos, (op.part.n_owned, op.part.recv), group=group)
    peers = sorted(op.part.send)
    op.enable_push({q: infos[q] for q in peers}, {q: int(hdl.buffer_ptrs[q]) for q in peers})
    views = {q: hdl.get_buffer(q, tuple(U.shape), U.dtype) for q in peers}

    def barrier():
        hdl.barrier(channel=0)

    def fill(parity: int = 0):
        op.push.fill(U, views, parity)
        barrier()

    return U, fill, barrier
