"""DG operator: the RHS / SSP-RK API the north star asks for.

``DGOperator(mesh, coloring, degree, physics)`` builds, once on the host:
the color-major renumbering (``reorder.build_plan`` + ``apply_plan``,
reference reorder.py:64-167), the DG surface list and element geometry
(``dg.layout``), the reference-element tables (``dg.basis``) — and uploads
them through ``mc_dg_create``.  Every evaluation then runs on the B200:

* ``rhs(U, strategy)`` — Eq. (2) by Algorithm 1
  (PAPER.md:64-82): one launch per color, no atomics, no buffer
  (``strategy="colored"``), or the paper's comparison variants
  ``"buffered"`` (2*ns slot buffer + gather) and ``"atomic"``;
* ``ssprk3(U, dt, steps)`` — SSP-RK3 with the volume integral fused into
  each element's first color pass and the stage update into its last.

Host arrays are in the caller's (original) element order, shape
(ne, n_equations, n_basis); device tensors (``*_device``) use the internal
layout: renumbered elements, blocks of ``stride`` doubles (32-byte padded).
There is no CPU fallback.
"""

from __future__ import annotations

import os

import numpy as np

from .. import _native
from ..amr import RefinedMesh
from ..coloring import SurfaceColoring, color
from ..mesh import ElementKind, Mesh
from ..reorder import ReorderingPlan, apply_plan, build_plan
from .basis import DIM, HYBRID, REF_MEASURE, evaluate_basis, reference_tables, volume_rule
from .layout import (build_surface_list, element_centroids, element_kinds, mesh_kind,
                     unwrapped_element_coords)

_KIND_CODE = {ElementKind.TRIANGLE: 0, ElementKind.QUAD: 1, ElementKind.TET: 2, HYBRID: 3}
_STRATEGY = {"colored": 0, "buffered": 1, "atomic": 2}
# tets: unsorted.  The windowed side-code sort (colors >= 2 sorted inside
# windows of 4096 surfaces so warps read the same face-table rows) paid in
# round 1 (c4 1.223 -> 1.239 G edges/s); since the face-table row is read
# once per point it costs more coalescing than it saves (c4 1.454 -> 1.487
# unsorted).  MC_CODE_SORT=4096 restores it.
_TET_CODE_SORT = False


def _sort_options(code_sort, kind) -> dict:
    """Surface order inside each color (any order is race free and keeps
    every element's accumulation order).  ``code_sort``: False / 0 = keep
    the layout order; True / 1 = sort every color by side codes (warps read
    the same face-table rows); an int n >= 2 = sort colors >= 2 inside
    windows of n surfaces counted from the color's first surface (color 1
    stays coalesced).  None = the measured default per element kind
    (whole-color sort +2 % on quads, unsorted on tets and
    triangles), overridable with MC_CODE_SORT."""
    if code_sort is None:
        env = os.environ.get("MC_CODE_SORT")
        if env is not None:
            try:
                code_sort = int(env)
            except ValueError:
                raise ValueError(f"MC_CODE_SORT must be an integer (0, 1 or a window >= 2), "
                                 f"got {env!r}") from None
        else:
            code_sort = {ElementKind.QUAD: True,
                         ElementKind.TET: _TET_CODE_SORT}.get(kind, False)
    if isinstance(code_sort, (bool, np.bool_)) or code_sort in (0, 1):
        return dict(code_sort=bool(code_sort))
    n = int(code_sort)
    if n < 0:
        raise ValueError(f"code_sort window must be >= 2, got {n}")
    return dict(code_sort=True, code_sort_window=n, code_sort_skip_first=True)


def default_freestream(dim: int, gamma: float = 1.4):
    rho, p = 1.0, 1.0
    vel = (0.3, 0.2, 0.1)[:dim]
    E = p / (gamma - 1.0) + 0.5 * rho * sum(v * v for v in vel)
    return (rho, *[rho * v for v in vel], E)


def _morton_key(x: np.ndarray) -> np.ndarray:
    """Z-order key of points (n, dim), 21 bits per axis."""
    lo, hi = x.min(axis=0), x.max(axis=0)
    q = ((x - lo) / np.maximum(hi - lo, 1e-300) * ((1 << 21) - 1)).astype(np.uint64)
    key = np.zeros(len(x), dtype=np.uint64)
    dim = x.shape[1]
    for b in range(21):
        for d in range(dim):
            key |= ((q[:, d] >> np.uint64(b)) & np.uint64(1)) << np.uint64(b * dim + d)
    return key


def sfc_plan(mesh: Mesh, coloring: SurfaceColoring, period=None) -> ReorderingPlan:
    """build_plan's color-major layout (color-1 pairs at k and N1 + k, the
    other colors sorted by new left id) with the color-1 pairs taken in
    Z-order of their midpoints instead of surface-id order, so that spatial
    neighbours get nearby block addresses and the random-access colors read
    fewer, denser DRAM pages (a shuffled input mesh gets its locality back).
    Falls back to build_plan when an element lacks a color-1 surface (AMR)."""
    full = build_plan(mesh, coloring)
    if full.used_fallback:
        return full
    colors = np.asarray(coloring.colors)
    left, right = mesh.surf_elems[:, 0], mesh.surf_elems[:, 1]
    cen = element_centroids(mesh, unwrapped_element_coords(mesh, period))
    ones = np.flatnonzero(colors == 1)
    mid = cen[left[ones]].copy()
    inner = right[ones] >= 0
    mid[inner] = 0.5 * (mid[inner] + cen[right[ones[inner]]])
    key = _morton_key(mid)
    interior = ones[inner][np.argsort(key[inner], kind="stable")]
    boundary = ones[~inner][np.argsort(key[~inner], kind="stable")]
    order1 = np.concatenate([interior, boundary])
    ep = np.empty(mesh.n_elements, dtype=np.int64)
    ep[left[order1]] = np.arange(len(order1))
    ep[right[interior]] = len(order1) + np.arange(len(interior))
    sp = np.empty(mesh.n_surfaces, dtype=np.int64)
    sp[order1] = np.arange(len(order1))
    nxt = len(order1)
    for c in range(2, int(coloring.n_colors) + 1):
        sids = np.flatnonzero(colors == c)
        sids = sids[np.argsort(ep[left[sids]], kind="stable")]
        sp[sids] = nxt + np.arange(len(sids))
        nxt += len(sids)
    rest = np.flatnonzero(colors > coloring.n_colors)
    sp[rest] = nxt + np.arange(len(rest))
    return ReorderingPlan(ep, sp, full.group_bounds, full.n_interior_first, False)


def ordering_plan(mesh: Mesh, coloring: SurfaceColoring, ordering: str,
                  period=None) -> ReorderingPlan:
    """The three layouts of the paper's Table 7:
    "reorder" = element renumbering + edge reordering (build_plan),
    "renumber" = element renumbering only, surfaces grouped by color in
    original id order, "none" = original numbering, surfaces grouped by
    color; plus "sfc" = "reorder" with the color-1 pairs in
    Z-order (``sfc_plan``)."""
    colors = np.asarray(coloring.colors)
    if ordering == "sfc":
        return sfc_plan(mesh, coloring, period)
    full = build_plan(mesh, coloring)
    if ordering == "reorder":
        return full
    order = np.argsort(colors, kind="stable")
    sp = np.empty(mesh.n_surfaces, dtype=np.int64)
    sp[order] = np.arange(mesh.n_surfaces)
    ep = full.element_perm if ordering == "renumber" else np.arange(mesh.n_elements)
    if ordering not in ("renumber", "none"):
        raise ValueError(f"unknown ordering {ordering!r}")
    return ReorderingPlan(np.asarray(ep, dtype=np.int64).copy(), sp, full.group_bounds,
                          full.n_interior_first, full.used_fallback)


class DGOperator:
    def __init__(self, mesh, coloring: SurfaceColoring | None = None, degree: int = 1,
                 physics: str = "euler", *, period=None, gamma: float = 1.4,
                 velocity=(1.0, 0.5, 0.25), farfield=None, ordering: str | None = None,
                 world: int = 1, rank: int = 0, code_sort: bool | int | None = None,
                 grid_cap: int | None = None, state: str = "f64"):
        mortars = None
        if isinstance(mesh, RefinedMesh):
            mortars = mesh.hanging_array()
            mesh = mesh.mesh
        self.mesh = mesh
        self._sort = _sort_options(code_sort, mesh_kind(mesh))
        if coloring is None:
            coloring, _ = color(mesh)
        self.coloring = coloring
        self.kind = mesh_kind(mesh)
        self.dim = DIM[self.kind]
        self.degree = int(degree)
        self.physics = physics
        if physics not in ("advection", "euler"):
            raise ValueError(f"unknown physics {physics!r}")
        if state not in ("f64", "f32"):
            raise ValueError(f"state must be 'f64' or 'f32', got {state!r}")
        # "f32": element blocks stored as floats (half the bytes), arithmetic
        # in fp64; colored strategy only; the north star's 1e-5 tolerance
        self.state = state
        self.n_equations = 1 if physics == "advection" else self.dim + 2
        self.gamma = float(gamma)
        self.velocity = tuple(float(v) for v in velocity) + (0.0,) * (3 - len(velocity))
        if farfield is None:
            farfield = (0.0,) if physics == "advection" else default_freestream(self.dim, gamma)
        self.farfield = tuple(float(x) for x in farfield)
        if len(self.farfield) != self.n_equations:
            raise ValueError("far-field state needs one value per equation")
        self.period = period
        if ordering is None:        # Z-ordered pairs, c2 3.49 -> 3.64 G edges/s
            ordering = os.environ.get("MC_ORDERING", "sfc")
        self.ordering = ordering

        self.plan = ordering_plan(mesh, coloring, ordering, period)
        self.layout_mesh, lcol = apply_plan(mesh, coloring, self.plan)
        self.layout_coloring = lcol
        if mortars is not None and len(mortars):
            mortars = self.plan.surface_perm[mortars]
        self.mortars = mortars
        self.world, self.rank, self.part = int(world), int(rank), None
        if self.world > 1:
            # domain decomposition of the renumbered mesh (partition.py)
            from ..partition import (build_partition, local_mortars, mortar_aligned_owner,
                                     slab_owner)
            owner = slab_owner(self.layout_mesh, self.world, period=period)
            part_mortars = None
            if mortars is not None and len(mortars):
                # nonconforming interfaces stay rank-local: the fine halves
                # of every hanging edge go to the coarse element's rank
                owner = mortar_aligned_owner(self.layout_mesh, mortars, owner)
            self.part = build_partition(self.layout_mesh, lcol.colors, lcol.n_colors, owner,
                                        self.rank)
            if mortars is not None and len(mortars):
                part_mortars = local_mortars(self.part, mortars)
            self.surfaces = build_surface_list(self.part.mesh, self.part.colors, lcol.n_colors,
                                               period=period, owned=self.part.n_owned,
                                               flipped=self.part.flipped, mortars=part_mortars,
                                               **self._sort)
            self.n_elements = self.part.n_owned
            self.n_local = self.part.n_local
        else:
            self.surfaces = build_surface_list(self.layout_mesh, lcol.colors, lcol.n_colors,
                                               period=period, mortars=mortars, **self._sort)
            self.n_elements = mesh.n_elements
            self.n_local = mesh.n_elements
        self.tables = reference_tables(self.kind, self.degree)
        self.n_basis = self.tables.n_basis
        self._create()
        self._set_user_rows()
        if grid_cap is not None:
            self.set_grid_cap(grid_cap)
        self.halo = None
        if self.part is not None:
            from ..partition import HaloExchange
            self.halo = HaloExchange(self.part, "cuda")
            if os.environ.get("MC_KERNEL_PACK", "1") != "0":
                self.halo.attach(self, self.stride)

    # ---------------------------------------------------------- native
    def _create(self):
        lib = _native.lib()
        _native.require_device()
        sl, t = self.surfaces, self.tables
        keep = dict(
            bounds=np.ascontiguousarray(sl.bounds, dtype=np.int64),
            left=np.ascontiguousarray(sl.left), right=np.ascontiguousarray(sl.right),
            code=np.ascontiguousarray(sl.code), geom=np.ascontiguousarray(sl.geom),
            jinv=np.ascontiguousarray(sl.jinv.reshape(-1)),
            ptr=np.ascontiguousarray(sl.slot_ptr, dtype=np.int64),
            slots=np.ascontiguousarray(sl.slots, dtype=np.int32),
            fphi=np.ascontiguousarray(t.face_phi), fw=np.ascontiguousarray(t.face_w),
            vphi=np.ascontiguousarray(t.vol_phi), vdphi=np.ascontiguousarray(t.vol_dphi),
            vw=np.ascontiguousarray(t.vol_w),
            ekind=np.ascontiguousarray(sl.ekind, dtype=np.uint8))
        d = _native.DGDesc()
        d.kind = _KIND_CODE[self.kind]
        d.physics = 0 if self.physics == "advection" else 1
        d.degree = self.degree
        d.n_colors = sl.n_colors
        d.n_elements = sl.n_elements
        d.n_ghosts = sl.n_ghosts
        d.n_surfaces = sl.n_surfaces
        P = _native.ptr
        d.group_bounds, d.surf_left, d.surf_right = P(keep["bounds"]), P(keep["left"]), P(keep["right"])
        d.surf_code, d.surf_geom, d.elem_jinv = P(keep["code"]), P(keep["geom"]), P(keep["jinv"])
        d.elem_slot_ptr, d.elem_slots = P(keep["ptr"]), P(keep["slots"])
        d.n_face_codes, d.n_face_q = t.n_codes, len(t.face_w)
        d.n_vol_q, d.n_basis = len(t.vol_w), t.n_basis
        d.face_phi, d.face_w = P(keep["fphi"]), P(keep["fw"])
        d.vol_phi, d.vol_dphi, d.vol_w = P(keep["vphi"]), P(keep["vdphi"]), P(keep["vw"])
        d.gamma = self.gamma
        d.state_f32 = 1 if self.state == "f32" else 0
        d.elem_kind = P(keep["ekind"]) if self.kind is HYBRID else None
        for k in range(3):
            d.velocity[k] = self.velocity[k]
        ff = list(self.farfield) + [0.0] * (5 - len(self.farfield))
        for k in range(5):
            d.farfield[k] = ff[k]
        h = _native.C.c_void_p()
        _native.check(lib.mc_dg_create(_native.C.byref(d), _native.C.byref(h)))
        self._lib = lib
        self._h = h
        self.stride = int(lib.mc_dg_block_stride(h))

    def _set_user_rows(self):
        """Tell the library where each internal owned row lives in the
        caller's (user) element order, for the user-layout entry points.
        Single domain: the whole state in user order.  Partitioned: this
        rank's owned elements in ascending user id (``user_rows``)."""
        ids = self.owned_user_ids()
        if self.part is None:
            src, n = ids, self.mesh.n_elements
        else:
            src, n = np.searchsorted(np.sort(ids), ids), len(ids)
        src = np.ascontiguousarray(src, dtype=np.int64)
        _native.check(self._lib.mc_dg_set_user_rows(self._h, _native.ptr(src), int(n)))

    def user_rows(self, U: np.ndarray) -> np.ndarray:
        """The caller-order rows this operator's user-layout entry points
        take: the whole state, or (partitioned) this rank's owned elements
        in ascending user id, as (rows, N_eq * N_p)."""
        U = np.asarray(U, dtype=np.float64).reshape(self.mesh.n_elements, -1)
        if self.part is None:
            return np.ascontiguousarray(U)
        return np.ascontiguousarray(U[np.sort(self.owned_user_ids())])

    def user_to_device(self, user_dev, U_dev, stream=None) -> None:
        """Device permutation: caller-order rows -> internal blocks."""
        _native.check(self._lib.mc_dg_user_to_internal(self._h, _native.ptr(user_dev),
                                                        _native.ptr(U_dev),
                                                        _native.stream_ptr(stream)))

    def device_to_user(self, U_dev, user_dev, stream=None) -> None:
        """Device permutation: internal blocks -> caller-order rows."""
        _native.check(self._lib.mc_dg_internal_to_user(self._h, _native.ptr(U_dev),
                                                        _native.ptr(user_dev),
                                                        _native.stream_ptr(stream)))

    def set_grid_cap(self, max_blocks: int) -> None:
        """Cap every persistent-grid launch at ``max_blocks`` blocks (0 =
        the occupancy-sized default), so each warp loops over many tiles."""
        _native.check(self._lib.mc_dg_set_grid_cap(self._h, int(max_blocks)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.mc_dg_destroy(h)
            self._h = None

    # ----------------------------------------------------- layout maps
    @property
    def n_colors(self) -> int:
        return self.surfaces.n_colors

    @property
    def n_surfaces(self) -> int:
        return self.surfaces.n_surfaces

    def block_width(self) -> int:
        return self.n_equations * self.n_basis

    def to_internal(self, U: np.ndarray) -> np.ndarray:
        """(ne, neq, nb) user order -> (n_local, stride) renumbered, padded.
        On a partitioned operator: this rank's owned rows (ghost rows zero
        until the first halo exchange)."""
        U = np.asarray(U, dtype=np.float64).reshape(self.mesh.n_elements, -1)
        if self.part is not None:
            inv = np.empty_like(self.plan.element_perm)
            inv[self.plan.element_perm] = np.arange(len(inv))
            out = np.zeros((self.n_local, self.stride))
            out[: self.n_elements, : self.block_width()] = U[inv[self.part.owned]]
            return out
        out = np.zeros((self.n_elements, self.stride))
        out[self.plan.element_perm, : self.block_width()] = U
        return out

    def owned_user_ids(self) -> np.ndarray:
        """Original (user) element ids of this rank's internal rows."""
        inv = np.empty_like(self.plan.element_perm)
        inv[self.plan.element_perm] = np.arange(len(inv))
        if self.part is None:
            return inv
        return inv[self.part.owned]

    def from_internal(self, B: np.ndarray) -> np.ndarray:
        B = np.asarray(B).reshape(self.n_elements, self.stride)
        return B[self.plan.element_perm, : self.block_width()].reshape(
            self.n_elements, self.n_equations, self.n_basis).copy()

    @property
    def torch_dtype(self):
        import torch
        return torch.float32 if self.state == "f32" else torch.float64

    def empty_device(self):
        import torch
        return torch.zeros((self.n_local, self.stride), dtype=self.torch_dtype, device="cuda")

    def to_device(self, U: np.ndarray):
        import torch
        return torch.from_numpy(self.to_internal(U)).to("cuda", dtype=self.torch_dtype)

    def from_device(self, t) -> np.ndarray:
        import torch
        torch.cuda.current_stream().synchronize()
        return self.from_internal(t.double().cpu().numpy())

    # ------------------------------------------------------- evaluation
    def rhs_device(self, U_dev, R_dev, strategy: str = "colored", stream=None) -> None:
        _native.check(self._lib.mc_dg_rhs(self._h, _native.ptr(U_dev), _native.ptr(R_dev),
                                          _STRATEGY[strategy], _native.stream_ptr(stream)))

    def rk_stage_device(self, U_dev, U0_dev, R_dev, a, b, dt, stream=None) -> None:
        _native.check(self._lib.mc_dg_rk_stage(
            self._h, _native.ptr(U_dev), _native.ptr(U0_dev), _native.ptr(R_dev),
            float(a), float(b), float(dt), _native.stream_ptr(stream)))

    def color_pass_device(self, color: int, U_dev, U0_dev, R_dev, rk_mode: int = 0,
                          a: float = 0.0, b: float = 1.0, dt: float = 0.0, stream=None,
                          part: str | None = None) -> None:
        """One color launch.  ``part``: None = the whole color, "inner" =
        the surfaces that touch no ghost element, "interface" = the rest
        (a partitioned layout orders each color inner-first)."""
        if part is None:
            _native.check(self._lib.mc_dg_color_pass(
                self._h, int(color), _native.ptr(U_dev), _native.ptr(U0_dev), _native.ptr(R_dev),
                int(rk_mode), float(a), float(b), float(dt), _native.stream_ptr(stream)))
            return
        sl = self.surfaces
        n = int(sl.bounds[color] - sl.bounds[color - 1])
        k = int(sl.inner[color - 1])
        lo, hi = (0, k) if part == "inner" else (k, n)
        if part not in ("inner", "interface"):
            raise ValueError(f"unknown part {part!r}")
        _native.check(self._lib.mc_dg_color_range_pass(
            self._h, int(color), lo, hi, _native.ptr(U_dev), _native.ptr(U0_dev),
            _native.ptr(R_dev), int(rk_mode), float(a), float(b), float(dt),
            _native.stream_ptr(stream)))

    def stage_distributed(self, U_dev, U0_dev, R_dev, mode: int, a: float, b: float, dt: float,
                          stream=None, marker=None) -> None:
        """One SSP-RK stage on a partitioned operator with the ghost exchange
        overlapped: post the exchange, run the part of color 1 that touches
        no ghost, complete the exchange, then the rest of color 1 and the
        other colors.  ``marker(color)`` (optional) is called before each
        color's first launch (the bench records CUDA events there)."""
        import torch
        cs = stream if stream is not None else torch.cuda.current_stream()
        # halo work on the compute stream: the send gather (when needed) is
        # ordered after the previous stage's last-touch updates, the ghost
        # rows are read only after the transfers complete
        with torch.cuda.stream(cs):
            h = self.halo.start(U_dev) if self.halo is not None else None
        if marker:
            marker(1)
        self.color_pass_device(1, U_dev, U0_dev, R_dev, mode, a, b, dt, cs, part="inner")
        if h is not None:
            with torch.cuda.stream(cs):
                self.halo.finish(U_dev, h)
        self.color_pass_device(1, U_dev, U0_dev, R_dev, mode, a, b, dt, cs, part="interface")
        for c in range(2, self.n_colors + 1):
            if marker:
                marker(c)
            self.color_pass_device(c, U_dev, U0_dev, R_dev, mode, a, b, dt, cs)
        if self.halo is not None:
            self.halo.stage_done(rk=mode != 0)

    # ------------------------------------------------ peer-push exchange
    def enable_push(self, layout: dict, bases: dict) -> None:
        """Fuse the ghost exchange into the last-touch kernel
        (``partition.HaloPush``): ``layout[q] = (n_owned_q, recv_q)`` for the
        peers, ``bases[q]`` the mapped address of peer q's state array
        (``HaloPush.state_rows`` rows)."""
        from ..partition import HaloPush
        if self.part is None:
            raise ValueError("peer push needs a partitioned operator")
        sl = self.surfaces
        last1 = sl.code[sl.bounds[0]:sl.bounds[1]] & ((1 << 13) | (1 << 15))
        if last1.any():
            raise NotImplementedError("an element's last touch in color 1 (its inner part "
                                      "runs before the stage barrier)")
        self.push = HaloPush(self.part, layout)
        esize = 4 if self.state == "f32" else 8
        ptr, dst = self.push.destinations(bases, self.stride, esize)
        _native.check(self._lib.mc_dg_set_push_rows(self._h, _native.ptr(ptr), _native.ptr(dst),
                                                    int(len(dst))))

    def push_state_device(self):
        """A zeroed state array with double-buffered ghost rows."""
        import torch
        from ..partition import HaloPush
        return torch.zeros((HaloPush.state_rows(self.part), self.stride), dtype=self.torch_dtype,
                           device="cuda")

    def stage_push(self, U_dev, U0_dev, R_dev, mode: int, a: float, b: float, dt: float,
                   stage: int, barrier=None, stream=None, marker=None) -> None:
        """One SSP-RK stage with the peer-push exchange: the part of color 1
        that touches no ghost, the stage barrier (every rank finished stage
        ``stage - 1``, so the ghost copy of parity ``stage % 2`` is complete
        and no peer still reads the other copy), then the rest; last-touch
        passes push parity ``(stage + 1) % 2``."""
        import torch
        cs = stream if stream is not None else torch.cuda.current_stream()
        _native.check(self._lib.mc_dg_set_ghost_parity(self._h, stage % 2, (stage + 1) % 2))
        if marker:
            marker(1)
        self.color_pass_device(1, U_dev, U0_dev, R_dev, mode, a, b, dt, cs, part="inner")
        if barrier is not None:
            with torch.cuda.stream(cs):
                barrier()
        self.color_pass_device(1, U_dev, U0_dev, R_dev, mode, a, b, dt, cs, part="interface")
        for c in range(2, self.n_colors + 1):
            if marker:
                marker(c)
            self.color_pass_device(c, U_dev, U0_dev, R_dev, mode, a, b, dt, cs)

    def ssprk3_push(self, U_dev, work_dev, dt: float, steps: int = 1, barrier=None,
                    stream=None, stage0: int = 0) -> int:
        """SSP-RK3 with the peer push; returns the next stage index."""
        U0, R = work_dev[0], work_dev[1]
        s = stage0
        for _ in range(steps):
            for mode, a, b in self.STAGES:
                self.stage_push(U_dev, U0, R, mode, a, b, dt, s, barrier, stream)
                s += 1
        return s

    def work_device(self):
        import torch
        return torch.zeros((2, self.n_local, self.stride), dtype=self.torch_dtype, device="cuda")

    STAGES = ((2, 0.0, 1.0), (1, 0.75, 0.25), (1, 1.0 / 3.0, 2.0 / 3.0))

    def ssprk3_distributed(self, U_dev, work_dev, dt: float, steps: int = 1, stream=None) -> None:
        """SSP-RK3 on a partitioned operator: every stage exchanges the ghost
        rows, overlapped with the ghost-free part of color 1
        (``stage_distributed``); volume fused into first touch, update into
        last touch, U0 saved in stage 1."""
        U0, R = work_dev[0], work_dev[1]
        for _ in range(steps):
            for mode, a, b in self.STAGES:
                self.stage_distributed(U_dev, U0, R, mode, a, b, dt, stream)

    def ssprk3_device(self, U_dev, work_dev, dt: float, steps: int = 1, stream=None) -> None:
        _native.check(self._lib.mc_dg_ssprk3(self._h, _native.ptr(U_dev), _native.ptr(work_dev),
                                             float(dt), int(steps), _native.stream_ptr(stream)))

    def _user_array(self, U) -> np.ndarray:
        U = np.asarray(U, dtype=np.float64)
        if U.size != self.mesh.n_elements * self.block_width():
            raise ValueError(f"state must have shape ({self.mesh.n_elements}, "
                             f"{self.n_equations}, {self.n_basis})")
        return np.ascontiguousarray(U).reshape(self.mesh.n_elements, self.n_equations,
                                               self.n_basis)

    def rhs(self, U: np.ndarray, strategy: str = "colored", out: np.ndarray | None = None
            ) -> np.ndarray:
        """Eq. (2) residual of a host state in the caller's element order,
        end to end (``mc_dg_rhs_user_host``: H2D, device permutation into
        the color-major layout, the strategy's launches, permutation back,
        D2H)."""
        if self.part is not None:
            raise ValueError("partitioned operator: use rhs_device / stage_distributed")
        U = self._user_array(U)
        R = np.empty_like(U) if out is None else out
        if R.shape != U.shape or R.dtype != np.float64 or not R.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float64 array shaped like U")
        _native.check(self._lib.mc_dg_rhs_user_host(self._h, _native.ptr(U), _native.ptr(R),
                                                    _STRATEGY[strategy]))
        return R

    def ssprk3(self, U: np.ndarray, dt: float, steps: int = 1, inplace: bool = False
               ) -> np.ndarray:
        """``steps`` SSP-RK3 steps of a host state in the caller's element
        order, end to end (``mc_dg_ssprk3_user_host``: H2D, device
        permutation, the fused colored launches replayed as one CUDA graph
        per step, permutation back, D2H).  ``inplace=True`` updates a
        C-contiguous float64 ``U`` (e.g. in pinned memory) and returns it."""
        if self.part is not None:
            raise ValueError("partitioned operator: use ssprk3_distributed")
        if inplace:
            if not (isinstance(U, np.ndarray) and U.dtype == np.float64 and U.flags.c_contiguous
                    and U.size == self.mesh.n_elements * self.block_width()):
                raise ValueError("inplace needs a C-contiguous float64 array of the state size")
            B = U
        else:
            B = self._user_array(U).copy()
        _native.check(self._lib.mc_dg_ssprk3_user_host(self._h, _native.ptr(B), float(dt),
                                                       int(steps)))
        return B

    def ssprk3_host_internal(self, B: np.ndarray, dt: float, steps: int = 1) -> None:
        """In-place SSP-RK3 on a host array already in the internal layout
        (pinned or pageable); the bench's end-to-end leg."""
        _native.check(self._lib.mc_dg_ssprk3_host(self._h, _native.ptr(B), float(dt), int(steps)))

    # ------------------------------------------------------------ setup
    def element_coords(self) -> np.ndarray:
        return unwrapped_element_coords(self.mesh, self.period)

    def project(self, fn) -> np.ndarray:
        """L2 projection of fn(x (n, dim)) -> (n, neq) (user order).  Hybrid
        meshes: each element on its own basis (triangles zero beyond their
        N_p)."""
        X = self.element_coords()
        out = np.zeros((self.mesh.n_elements, self.n_equations, self.n_basis))
        if self.kind is HYBRID:
            ek = element_kinds(self.mesh)
            parts = [(ek == 0, ElementKind.TRIANGLE), (ek == 1, ElementKind.QUAD)]
        else:
            parts = [(np.ones(self.mesh.n_elements, bool), self.kind)]
        for sel, kind in parts:
            idx = np.flatnonzero(sel)
            if not len(idx):
                continue
            pts, w = volume_rule(kind, self.degree + 1)
            phi, _ = evaluate_basis(kind, self.degree, pts)
            Xk = X[idx]
            if kind is ElementKind.QUAD:
                J = np.stack([Xk[:, 1] - Xk[:, 0], Xk[:, 3] - Xk[:, 0]], axis=2)
            else:
                J = np.stack([Xk[:, r + 1] - Xk[:, 0] for r in range(self.dim)], axis=2)
            chunk = 1 << 16
            for a in range(0, len(idx), chunk):
                b = min(a + chunk, len(idx))
                x = Xk[a:b, 0][:, None, :] + np.einsum("erk,qk->eqr", J[a:b], pts)
                vals = fn(x.reshape(-1, self.dim)).reshape(b - a, len(w), self.n_equations)
                out[idx[a:b], :, :phi.shape[1]] = np.einsum("q,qj,eqk->ekj", w, phi, vals)
        return out

    def domain(self):
        X = self.element_coords().reshape(-1, self.dim)
        lo, hi = X.min(axis=0), X.max(axis=0)
        if self.period is not None:
            for d, L in enumerate(self.period):
                if L:
                    lo[d], hi[d] = 0.0, float(L)
        return lo, hi

    def initial_state(self, name: str = "wave") -> np.ndarray:
        lo, hi = self.domain()
        ext = np.maximum(hi - lo, 1e-12)
        if self.physics == "advection":
            def f(x):
                s = np.sin(2 * np.pi * (x[:, 0] - lo[0]) / ext[0])
                for d in range(1, self.dim):
                    s = s * np.cos(2 * np.pi * (x[:, d] - lo[d]) / ext[d])
                return s[:, None]
            return self.project(f)
        ff = np.asarray(self.farfield)
        rho0 = ff[0]
        vel = ff[1:1 + self.dim] / rho0
        p0 = (self.gamma - 1) * (ff[-1] - 0.5 * rho0 * (vel * vel).sum())

        def g(x):
            if name == "freestream":
                rho = np.full(len(x), rho0)
            else:  # smooth density wave carried by the free stream
                rho = rho0 * (1.0 + 0.2 * np.prod(
                    [np.sin(2 * np.pi * (x[:, d] - lo[d]) / ext[d]) for d in range(self.dim)],
                    axis=0))
            out = np.empty((len(x), self.n_equations))
            out[:, 0] = rho
            for d in range(self.dim):
                out[:, 1 + d] = rho * vel[d]
            out[:, -1] = p0 / (self.gamma - 1) + 0.5 * rho * (vel * vel).sum()
            return out
        return self.project(g)

    def stable_dt(self, cfl: float = 0.1) -> float:
        """CFL-type step h / (max wave speed * (2p+1))."""
        detj = np.abs(self.surfaces.detj[: self.n_elements])
        if self.kind is HYBRID:
            ref = np.where(self.surfaces.ekind[: self.n_elements] == 0,
                           REF_MEASURE[ElementKind.TRIANGLE], REF_MEASURE[ElementKind.QUAD])
        else:
            ref = REF_MEASURE[self.kind]
        h = (detj / ref) ** (1.0 / self.dim)
        ff = np.asarray(self.farfield)
        if self.physics == "advection":
            speed = np.linalg.norm(self.velocity[: self.dim]) + 1e-30
        else:
            rho = ff[0]
            vel = ff[1:1 + self.dim] / rho
            p = (self.gamma - 1) * (ff[-1] - 0.5 * rho * (vel * vel).sum())
            speed = np.linalg.norm(vel) + np.sqrt(self.gamma * p / rho * 1.3)
        return float(cfl * h.min() / (speed * (2 * self.degree + 1)))

    # ------------------------------------------------------------ oracle
    def oracle_problem(self) -> dict:
        """Plain description (user order) a checker can rebuild the same
        discretisation from; mortar halves carry their coarse neighbour as
        right element and full coarse edges are inactive."""
        m = self.mesh
        surf_elems = m.surf_elems.copy()
        active = np.ones(m.n_surfaces, dtype=bool)
        if self.mortars is not None and len(self.mortars):
            inv = np.empty_like(self.plan.surface_perm)
            inv[self.plan.surface_perm] = np.arange(len(inv))
            mt = inv[self.mortars]
            for k in (1, 2):
                surf_elems[mt[:, k], 1] = surf_elems[mt[:, 0], 0]
            active[mt[:, 0]] = False
        return dict(kind=self.kind.value, p=self.degree, physics=self.physics, dim=self.dim,
                    gamma=self.gamma, velocity=self.velocity, farfield=self.farfield,
                    vertices=m.vertices, elem_verts=m.elem_verts, surf_verts=m.surf_verts,
                    surf_elems=surf_elems, colors=np.asarray(self.coloring.colors),
                    n_colors=int(self.coloring.n_colors), active=active, period=self.period,
                    elem_kind=np.asarray(m.elem_kind) if self.kind is HYBRID else None)
