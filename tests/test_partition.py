"""Domain decomposition: partition invariants, and a
world-size-2 gloo run in which every rank evaluates Eq. (2) on its local
layout after a real halo exchange; owned residuals must equal the
single-domain residuals bit for bit (the oracle is the arithmetic here,
so this tests the partition / flip / exchange logic, on CPU)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1601_07613_b200 as P
from oracle import dg_oracle as D
from oracle import sweeps_oracle
from paper_1601_07613_b200.partition import build_partition, slab_owner


def layout_case(n=(10, 8), shuffle=1, kind="tri"):
    if kind == "tri":
        m = P.shuffle_elements(P.gen_tri_rect(*n), shuffle)
    else:
        m = P.gen_tet_prism(3, 2, 2)
    c, _ = P.color(m)
    plan = P.build_plan(m, c)
    return P.apply_plan(m, c, plan)


def problem(mesh, colors, n_colors, kind, p=2):
    dim = mesh.dim
    ff = (1.0, 0.3, 0.2, 2.6) if dim == 2 else (1.0, 0.3, 0.2, 0.1, 2.6)
    ph = D.Physics("euler", dim, farfield=ff)
    return D.Problem(kind, p, ph, mesh.vertices, mesh.elem_verts, mesh.surf_verts,
                     mesh.surf_elems, np.asarray(colors), n_colors,
                     np.ones(mesh.n_surfaces, bool))


def state(mesh, kind, p=2, seed=0):
    nb = D.Basis(kind, p).scale.size
    neq = mesh.dim + 2
    rng = np.random.default_rng(seed)
    U = rng.normal(size=(mesh.n_elements, neq, nb)) * 0.01
    U[:, 0, 0] += 1.5
    U[:, -1, 0] += 4.0
    return U


@pytest.mark.parametrize("world", [2, 3, 4])
def test_partition_invariants(world):
    lm, lc = layout_case()
    owner = slab_owner(lm, world)
    assert np.bincount(owner).min() >= lm.n_elements // world - 1
    seen = np.zeros(lm.n_surfaces, int)
    owned_all = []
    for r in range(world):
        part = build_partition(lm, lc.colors, lc.n_colors, owner, r)
        owned_all.append(part.owned)
        seen[part.global_surface] += 1
        loc = part.mesh
        # owned element is always on the left of a local surface
        assert (loc.surf_elems[:, 0] < part.n_owned).all()
        # restricted coloring stays race free and grouped
        assert (np.diff(part.colors) >= 0).all()
        assert sweeps_oracle.first_race(loc.surf_elems, part.colors, lc.n_colors) is None
        for q, ix in part.send.items():
            other = build_partition(lm, lc.colors, lc.n_colors, owner, q)
            a, b = other.recv[r]
            assert np.array_equal(part.owned[ix], other.ghosts[a - other.n_owned:b - other.n_owned])
    assert np.array_equal(np.sort(np.concatenate(owned_all)), np.arange(lm.n_elements))
    interior = lm.surf_elems[:, 1] >= 0
    cut = owner[lm.surf_elems[:, 0]] != owner[np.where(interior, lm.surf_elems[:, 1], 0)]
    assert ((seen == 2) == (interior & cut)).all() and (seen >= 1).all()


@pytest.mark.parametrize("world", [2, 3])
def test_local_layout_orders_ghost_surfaces_last(world):
    """Every color of a rank's device layout lists the surfaces that touch
    no ghost first (``inner``), so that part of color 1 can run while the
    ghost exchange is in flight; flags and CSR stay consistent."""
    from paper_1601_07613_b200.dg.layout import FLAG_R_GHOST, build_surface_list
    lm, lc = layout_case()
    owner = slab_owner(lm, world)
    for r in range(world):
        part = build_partition(lm, lc.colors, lc.n_colors, owner, r)
        sl = build_surface_list(part.mesh, part.colors, lc.n_colors, owned=part.n_owned,
                                flipped=part.flipped)
        assert sl.inner.sum() + (sl.code & FLAG_R_GHOST > 0).sum() == sl.n_surfaces
        for c in range(lc.n_colors):
            seg = (sl.code[sl.bounds[c]:sl.bounds[c + 1]] & FLAG_R_GHOST) > 0
            k = int(sl.inner[c])
            assert not seg[:k].any() and seg[k:].all()
            assert (sl.right[sl.bounds[c]:sl.bounds[c] + k] < part.n_owned).all()
        # the reordered list is still a race-free coloring of the local mesh
        se = np.stack([sl.left, sl.right], 1).astype(np.int64)
        col = np.repeat(np.arange(1, lc.n_colors + 1), np.diff(sl.bounds))
        assert sweeps_oracle.first_race(se, col, lc.n_colors) is None


def amr_layout_case(targets=(0, 5, 17, 18, 40, 77, 100), levels=1):
    base = P.gen_tri_rect(10, 8)
    col, _ = P.color(base)
    ref, fine = P.refine(base, col, list(targets))
    if levels == 2:
        kids = np.flatnonzero(ref.child_slot < 0)[::9]
        ref, fine = P.refine(ref, fine, kids.tolist())
    mortars = ref.hanging_array()
    plan = P.build_plan(ref.mesh, fine)
    lm, lc = P.apply_plan(ref.mesh, fine, plan)
    return lm, lc, plan.surface_perm[mortars]


@pytest.mark.parametrize("world,levels", [(2, 1), (3, 1), (4, 2)])
def test_partitioned_amr_keeps_hanging_interfaces_rank_local(world, levels):
    """Partitioned AMR: the fine halves of every hanging edge follow the
    coarse element's rank, so each rank's local layout carries whole mortar
    triples; every local surface that touches no ghost has the same sides
    and flags as in the single-domain layout."""
    from paper_1601_07613_b200.dg.layout import FLAG_R_GHOST, build_surface_list
    from paper_1601_07613_b200.partition import local_mortars, mortar_aligned_owner
    lm, lc, mortars = amr_layout_case(levels=levels)
    assert len(mortars)
    owner = mortar_aligned_owner(lm, mortars, slab_owner(lm, world))
    L = lm.surf_elems[:, 0]
    for k in (1, 2):
        assert np.array_equal(owner[L[mortars[:, k]]], owner[L[mortars[:, 0]]])
    assert len(np.unique(owner)) == world
    single = build_surface_list(lm, lc.colors, lc.n_colors, mortars=mortars)
    ref = {int(ms): (int(a), int(b), int(c)) for ms, a, b, c in
           zip(single.mesh_surface, single.left, single.right, single.code)}
    n_triples = 0
    for r in range(world):
        part = build_partition(lm, lc.colors, lc.n_colors, owner, r)
        lmort = local_mortars(part, mortars)
        n_triples += len(lmort)
        sl = build_surface_list(part.mesh, part.colors, lc.n_colors, owned=part.n_owned,
                                flipped=part.flipped, mortars=lmort)
        gids = np.concatenate([part.owned, part.ghosts])
        for ms, a, b, c in zip(sl.mesh_surface, sl.left, sl.right, sl.code):
            if c & FLAG_R_GHOST or part.flipped[ms]:
                continue
            g = int(part.global_surface[ms])
            assert ref[g] == (int(gids[a]), int(gids[b]) if b >= 0 else -1, int(c))
        se = np.stack([sl.left, sl.right], 1).astype(np.int64)
        col = np.repeat(np.arange(1, lc.n_colors + 1), np.diff(sl.bounds))
        assert sweeps_oracle.first_race(se, col, lc.n_colors) is None
    assert n_triples == len(mortars)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, out):
    import torch
    import torch.distributed as dist
    from paper_1601_07613_b200.partition import HaloExchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lm, lc = layout_case(kind=kind)
    owner = slab_owner(lm, world)
    part = build_partition(lm, lc.colors, lc.n_colors, owner, rank)
    Ug = state(lm, kind)
    Ul = np.full((part.n_local,) + Ug.shape[1:], np.nan)
    Ul[: part.n_owned] = Ug[part.owned]
    t = torch.from_numpy(Ul.reshape(part.n_local, -1).copy())
    HaloExchange(part, "cpu").exchange(t)
    Ul = t.numpy().reshape(Ul.shape)
    assert np.isfinite(Ul).all()
    Rl = D.rhs(problem(part.mesh, part.colors, lc.n_colors, kind), Ul)
    np.save(out + f"/r{rank}.npy", Rl[: part.n_owned])
    np.save(out + f"/o{rank}.npy", part.owned)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["tri", "tet"])
def test_two_rank_halo_exchange_reproduces_single_domain(tmp_path, kind):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), kind, str(tmp_path)), nprocs=world, join=True)
    lm, lc = layout_case(kind=kind)
    Ug = state(lm, kind)
    Rg = D.rhs(problem(lm, lc.colors, lc.n_colors, kind), Ug)
    for r in range(world):
        owned = np.load(tmp_path / f"o{r}.npy")
        Rl = np.load(tmp_path / f"r{r}.npy")
        assert np.array_equal(Rl, Rg[owned]), np.abs(Rl - Rg[owned]).max()


def _worker_packed(rank, world, port, out):
    """Three tet slabs: a gathered exchange, then an 'RK update' whose new
    interface blocks are written into the send buffer through the send
    slots (what the last-touch kernel does on the GPU), then an exchange
    that posts the buffer as is."""
    import torch
    import torch.distributed as dist
    from paper_1601_07613_b200.partition import HaloExchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = P.gen_tet_prism(9, 2, 2)
    c, _ = P.color(m)
    lm, lc = P.apply_plan(m, c, P.build_plan(m, c))
    owner = slab_owner(lm, world)
    part = build_partition(lm, lc.colors, lc.n_colors, owner, rank)
    Ug = np.arange(lm.n_elements * 4, dtype=np.float64).reshape(-1, 4)
    U = torch.full((part.n_local, 4), np.nan, dtype=torch.float64)
    U[: part.n_owned] = torch.from_numpy(Ug[part.owned])
    halo = HaloExchange(part, "cpu")
    halo.exchange(U)
    ok1 = np.array_equal(U.numpy(), Ug[np.concatenate([part.owned, part.ghosts])])
    slot = halo.send_slots()
    assert slot is not None
    U[: part.n_owned] += 1000.0                     # the stage's update of owned rows
    buf = halo._buffer(U)
    sel = slot >= 0
    buf[torch.from_numpy(slot[sel]).long()] = U[: part.n_owned][torch.from_numpy(sel)]
    halo.packed_by_kernel = True
    halo.stage_done(rk=True)
    assert halo.fresh
    U[: part.n_owned] = torch.from_numpy(Ug[part.owned] + 1000.0)
    halo.exchange(U)
    ok2 = np.array_equal(U.numpy(), Ug[np.concatenate([part.owned, part.ghosts])] + 1000.0)
    np.save(out + f"/ok{rank}.npy", np.array([ok1, ok2, not halo.fresh]))
    dist.barrier()
    dist.destroy_process_group()


def test_three_rank_exchange_with_kernel_packed_send_rows(tmp_path):
    world = 3
    mp.spawn(_worker_packed, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.load(tmp_path / f"ok{r}.npy").all()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_peer_push_destinations(world):
    """HaloPush (exchange fused into the last-touch kernel): every pushed
    block lands in the peer's ghost row of the same global element, in the
    double-buffered layout (ghost g at n_owned + 2g + parity)."""
    from paper_1601_07613_b200.partition import HaloPush
    lm, lc = layout_case()
    owner = slab_owner(lm, world)
    parts = [build_partition(lm, lc.colors, lc.n_colors, owner, r) for r in range(world)]
    layout = {r: (p.n_owned, p.recv) for r, p in enumerate(parts)}
    stride, esize = 24, 8
    bases = {q: (q + 1) << 32 for q in range(world)}
    for p in parts:
        hp = HaloPush(p, {q: layout[q] for q in p.send})
        ptr, dst = hp.destinations({q: bases[q] for q in p.send}, stride, esize)
        assert ptr[-1] == len(dst) == sum(len(v) for v in p.send.values())
        for e in range(p.n_owned):
            for addr in dst[ptr[e]:ptr[e + 1]]:
                q = (int(addr) >> 32) - 1
                row = (int(addr) - bases[q]) // (stride * esize)
                ne_q = parts[q].n_owned
                assert row >= ne_q and (row - ne_q) % 2 == 0
                g = (row - ne_q) // 2
                assert parts[q].ghosts[g] == p.owned[e]
        assert HaloPush.state_rows(p) == p.n_owned + 2 * len(p.ghosts)
