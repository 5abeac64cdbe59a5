"""Algorithm 1 on every host core: the oracle's fp64 DG SSP-RK3 step run
by a pool of forked worker processes (oracle; TEST/BENCH INFRASTRUCTURE).

bench.py's reference arm and CPU baseline time this — the reference has no
DG, so its CPU path for the north star's workload is the
oracle restatement (``dg_oracle``), parallelised the way the paper's
Algorithm 1 allows: within one color no two surfaces
write the same element, so a color's surfaces split into independent
chunks; colors are separated by a barrier (one ``Pool.map`` per color, the
reference's per-color future join, sweeps.py:143-151).  The volume term
and the RK update split by element.  State arrays live in anonymous shared
memory, so workers update them in place.  Arithmetic per element is the
oracle's (volume, then colors in order), so results equal
``dg_oracle.ssprk3`` to rounding of the summation order (identical order:
bit-identical).
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os

import numpy as np

from . import dg_oracle as D

_W: dict = {}          # state inherited by the forked workers


def _shared(shape) -> np.ndarray:
    n = int(np.prod(shape))
    buf = mmap.mmap(-1, max(8 * n, 8))
    return np.frombuffer(buf, dtype=np.float64, count=n).reshape(shape)


def _init_worker():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # noqa: BLE001
        pass


def _volume(task):
    lo, hi = task
    _W["R"][lo:hi] = D.volume_term(_W["prob"], _W["U"], lo, hi)
    return 0


def _surfaces(task):
    color, lo, hi = task
    sel = _W["sel"][color][lo:hi]
    L, R, cl, cr = D.surface_contributions(_W["prob"], _W["U"], sel)
    Rr = _W["R"]
    Rr[L] += cl                              # race free inside one color
    inner = R >= 0
    Rr[R[inner]] += cr[inner]
    return 0


def _update(task):
    lo, hi, a, b, dt, save = task
    U, U0, R = _W["U"], _W["U0"], _W["R"]
    if save:
        U0[lo:hi] = U[lo:hi]
    if a == 0.0:
        U[lo:hi] = U[lo:hi] + dt * R[lo:hi]
    else:
        U[lo:hi] = a * U0[lo:hi] + b * (U[lo:hi] + dt * R[lo:hi])
    return 0


def _chunks(n, parts):
    edges = np.linspace(0, n, parts + 1).astype(np.int64)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]


class ParallelStepper:
    """SSP-RK3 of ``prob`` with ``workers`` processes.  ``U`` is the shared
    state (ne, neq, nb); ``step(dt)`` advances it in place."""

    def __init__(self, prob: D.Problem, U0: np.ndarray, workers: int | None = None):
        c = D.setup(prob)
        self.workers = int(workers or len(os.sched_getaffinity(0)))
        shape = U0.shape
        self.U, self.U0, self.R = _shared(shape), _shared(shape), _shared(shape)
        self.U[:] = U0
        sel = {col: np.flatnonzero(c["col"] == col) for col in range(1, prob.n_colors + 1)}
        _W.update(prob=prob, U=self.U, U0=self.U0, R=self.R, sel=sel)
        self.ne = shape[0]
        self.parts = max(1, self.workers)
        self.vol_tasks = _chunks(self.ne, self.parts)
        self.surf_tasks = [[(col, a, b) for a, b in _chunks(len(s), self.parts)]
                           for col, s in sel.items()]
        self.pool = mp.get_context("fork").Pool(self.workers, initializer=_init_worker)

    def close(self):
        self.pool.close()
        self.pool.join()

    def rhs(self) -> None:
        """R := Eq. (2) of the current U (volume, then colors in order)."""
        self.pool.map(_volume, self.vol_tasks, chunksize=1)
        for tasks in self.surf_tasks:
            if tasks:
                self.pool.map(_surfaces, tasks, chunksize=1)

    def step(self, dt: float) -> None:
        for a, b, save in ((0.0, 1.0, True), (0.75, 0.25, False), (1.0 / 3.0, 2.0 / 3.0, False)):
            self.rhs()
            self.pool.map(_update, [(lo, hi, a, b, dt, save) for lo, hi in self.vol_tasks],
                          chunksize=1)
