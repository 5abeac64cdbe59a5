#!/usr/bin/env python
"""Benchmark of the colored DG surface-integral hot path (driver contract).

One "step" = one SSP-RK3 time step of the colored DG operator on a
BASELINE config, i.e. three fused colored RHS evaluations (volume integral
fused into each element's first color pass, the RK update into its last).
Default config c4 (BASELINE.json configs[3], the largest single-GPU mesh):
``gen_tet_prism(110,110,110)`` = 7,986,000 tetrahedra, 16,044,600 faces,
4 colors, 3D Euler p=2, Lax-Friedrichs, fp64.  Inputs are synthetic (a
smooth density wave on the far-field stream) and device resident (3.3 GB
per state array, far larger than the 126 MB L2).

value     = surface-integral edge evaluations per second = 3 * n_surfaces / t_step
            (dof_updates_per_s = n_elements * N_p * N_eq * 3 / t_step)
e2e       = the same through the public API a user calls,
            ``DGOperator.ssprk3(U, dt, 1)`` on a pinned host array in the
            caller's element order: H2D, device permutation into the
            color-major layout, the step, permutation back, D2H
roofline  = the colored kernel (``k_tpe_colored``): algorithmic bytes per
            launch / its CUDA-event duration, against the
            measured HBM copy peak in MEASURED_PEAKS.json
comparisons = the paper's: colored vs buffer-and-reduce vs atomics RHS, the
            buffer memory the coloring avoids, the integer Algorithm 1
            sweeps on the GPU, and the reference's integer CPU path
            (``sweep_sequential`` and ``sweep_colored(workers=cpu_count)``
            restated in oracle/sweeps_oracle.py) on the same mesh
cpu_baseline / --impl reference = the numpy fp64 DG oracle (a port: the
            reference has no DG) stepping a bounded sample of the same mesh
            family on every host core (oracle/dg_parallel.py); the
            reference arm builds its mesh, coloring and problem with
            oracle/ only and never loads the product library.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                       [--config c1|c2|c3|c4|c5|h1] [--no-variants] [--no-cpu]
                       [--exchange nccl|push] [--state f64|f32]
       python bench.py --layouts     # the paper's Table 7 layouts on c2
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "surface-integral edges/sec & DOF-updates/sec; % of HBM roofline; 1/2/4/8 GPU"
UNIT = "edges/s"
STAGES = ((2, 0.0, 1.0), (1, 0.75, 0.25), (1, 1.0 / 3.0, 2.0 / 3.0))
PRODUCT_SO = "libmeshchroma_b200"

# name: (description, physics, degree, oracle sample recipe)
CONFIGS = {
    "c1": ("2D scalar advection DG p=1, gen_tri_rect(64,64), 3 colors", "advection", 1,
           ("tri", (64, 64), None)),
    "c2": ("2D Euler DG p=2, shuffle_elements(gen_tri_rect(708,708),0), LF, 3 colors",
           "euler", 2, ("tri", (177, 177), 0)),
    "c3": ("2D Euler DG p=3, gen_quad_rect(2000,2000), LF, 4 colors", "euler", 3,
           ("quad", (250, 250), None)),
    "c4": ("3D Euler DG p=2, gen_tet_prism(110,110,110), LF, 4 colors", "euler", 2,
           ("tet", (28, 28, 28), None)),
    "c5": ("2D Euler DG p=2, 1:4 refined disc r=177 in gen_tri_rect(708,708), 6 colors, "
           "mortars", "euler", 2, ("tri", (177, 177), None)),
    # not a BASELINE config: the hybrid (triangle + quad) layout at c2's scale
    "h1": ("2D Euler DG p=2, gen_hybrid_rect(708,708) (triangles + quads, conftest."
           "hybrid_patch layout), LF, 4 colors", "euler", 2, ("hybrid", (177, 177), None)),
}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def product_library_loaded() -> bool:
    try:
        return PRODUCT_SO in Path("/proc/self/maps").read_text()
    except OSError:
        return False


# ------------------------------------------------------------- workloads
def config_spec(name: str, device: str | None = "cuda"):
    """The product's build of a BASELINE config (GPU mesh assembly, native
    coloring, GPU AMR: bit-identical to the reference, see
    tests/test_config_golden_gpu.py)."""
    import paper_1601_07613_b200 as P
    if name not in CONFIGS:
        raise SystemExit(f"unknown config {name}")
    desc, physics, p, _ = CONFIGS[name]
    dv = device
    builds = {
        "c1": lambda: P.gen_tri_rect(64, 64),
        "c2": lambda: P.shuffle_elements(P.gen_tri_rect(708, 708, device=dv), 0, device=dv),
        "c3": lambda: P.gen_quad_rect(2000, 2000, device=dv),
        "c4": lambda: P.gen_tet_prism(110, 110, 110, device=dv),
        "h1": lambda: P.gen_hybrid_rect(708, 708, device=dv),
    }

    def c5():
        base = P.gen_tri_rect(708, 708, device=dv)
        col, _ = P.color(base)
        cen = base.vertices[base.elem_verts[:, :3]].mean(axis=1)
        tg = np.flatnonzero(((cen - 354.0) ** 2).sum(1) <= 177.0 ** 2)
        return P.refine(base, col, tg, device=dv)
    return dict(name=name, desc=desc, physics=physics, p=p, build=builds.get(name, c5))


def build_operator(spec, world=1, rank=0, **kw):
    from paper_1601_07613_b200.dg import DGOperator
    import paper_1601_07613_b200 as P
    obj = spec["build"]()
    if isinstance(obj, tuple):          # (RefinedMesh, 6-coloring)
        return DGOperator(obj[0], obj[1], degree=spec["p"], physics=spec["physics"], **kw)
    col, _ = P.color(obj)
    return DGOperator(obj, col, degree=spec["p"], physics=spec["physics"], world=world,
                      rank=rank, **kw)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """NVML clock / throttle-reason sampling during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int = 0, period_s: float = 0.005):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
            self.max_mhz = None

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nvml:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nvml:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# -------------------------------------------------------------- roofline
def launch_bytes(op, color: int, rk_mode: int, a: float) -> int:
    """Algorithmic bytes of one colored launch: per surface
    the metadata (ids, code word, geometry), per present side its U block,
    the inverse Jacobian at first touch, the residual block read unless
    first touch, and either the residual write or, at the last touch of an
    RK stage, the U0 read (a != 0) / U0 save / U write."""
    sl = op.surfaces
    b0, b1 = sl.bounds[color - 1], sl.bounds[color]
    code = sl.code[b0:b1].astype(np.int64)
    right = sl.right[b0:b1]
    D = op.n_equations * op.n_basis * (4 if getattr(op, "state", "f64") == "f32" else 8)
    dim = op.dim
    meta = 4 + 4 + 4 + 8 * (dim + 2)
    total = meta * (b1 - b0)
    for side, fbit, lbit in ((0, 1 << 12, 1 << 13), (1, 1 << 14, 1 << 15)):
        present = np.ones(b1 - b0, bool) if side == 0 else right >= 0
        ghost = np.zeros(b1 - b0, bool) if side == 0 else (code & (1 << 16)) != 0
        first = present & ~ghost & ((code & fbit) != 0)
        last = present & ~ghost & ((code & lbit) != 0)
        owner = present & ~ghost
        total += D * int(present.sum())                       # U read
        total += 8 * dim * dim * int(first.sum())             # Jinv at first touch
        total += D * int((owner & ~first).sum())              # R read
        if rk_mode == 0:
            total += D * int(owner.sum())                     # R write
        else:
            total += D * int((owner & ~last).sum())           # R write
            total += D * int(last.sum())                      # U write
            if a != 0.0:
                total += D * int(last.sum())                  # U0 read
            if rk_mode == 2:
                total += D * int(last.sum())                  # U0 save
    return int(total)


def kernel_name(op) -> str:
    """Which colored kernel the library dispatches (csrc/dg_tpe.cuh Tpe::OK)."""
    w = op.n_equations * op.n_basis
    if w <= 24:
        return "k_tpe_colored (1 lane per element side)"
    neqh = (op.n_equations + 1) // 2
    pairs = op.n_basis % 2 == 0 or (neqh % 2 == 0 and (op.n_equations - neqh) % 2 == 0)
    if w <= 64 and op.n_equations >= 2 and pairs:
        return "k_tpe_colored (2 lanes per element side)"
    return "k_surface_colored (2*N_eq lanes per surface, warp flux tasks)"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------- CPU (oracle) workloads
def oracle_sample(config: str):
    """The config's bounded sample built with oracle/ only (mesh, coloring,
    DG problem, initial density wave): what the reference arm and the
    cpu_baseline leg step on the host cores.  Never imports the product."""
    from oracle import coloring_oracle as CO
    from oracle import dg_oracle as D
    from oracle import mesh_oracle as MO
    desc, physics, p, (kind, dims, shuffle) = CONFIGS[config]
    gen = {"tri": MO.gen_tri_rect, "quad": MO.gen_quad_rect, "tet": MO.gen_tet_prism,
           "hybrid": MO.gen_hybrid_rect}[kind]
    m = gen(*dims)
    if shuffle is not None:
        m = MO.shuffle_elements(m, shuffle)
    nc = 4 if kind in ("quad", "tet", "hybrid") else 3
    cols, _ = CO.color(m["surf_elems"], m["elem_surfs"], nc, seed=0)
    dim = 3 if kind == "tet" else 2
    gamma = 1.4
    vel = np.array((0.3, 0.2, 0.1)[:dim])
    if physics == "euler":
        E = 1.0 / (gamma - 1) + 0.5 * float((vel * vel).sum())
        ff = (1.0, *vel.tolist(), E)
    else:
        ff = (0.0,)
    phys = D.Physics(physics, dim, gamma=gamma, farfield=ff)
    ns = len(cols)
    prob = D.Problem(kind, p, phys, m["vertices"], m["elem_verts"], m["surf_verts"],
                     m["surf_elems"], np.asarray(cols, dtype=np.int32), nc, np.ones(ns, bool),
                     elem_kind=np.asarray(m["elem_kind"]) if kind == "hybrid" else None)
    D.setup(prob)
    lo, hi = m["vertices"].min(axis=0), m["vertices"].max(axis=0)

    def wave(x):
        rho = 1.0 + 0.2 * np.prod([np.sin(2 * np.pi * (x[:, d] - lo[d]) / (hi[d] - lo[d]))
                                   for d in range(dim)], axis=0)
        if physics == "advection":
            return rho[:, None]
        out = np.empty((len(x), dim + 2))
        out[:, 0] = rho
        out[:, 1:1 + dim] = rho[:, None] * vel
        out[:, -1] = 1.0 / (gamma - 1) + 0.5 * rho * (vel * vel).sum()
        return out
    U = D.project(prob, wave)
    ne = len(m["elem_kind"])
    sample = (f"{gen.__name__}{dims}" + (f" shuffled (seed {shuffle})" if shuffle is not None
                                          else "") + f": {ne} elements / {ns} surfaces")
    return prob, U, ne, ns, sample


def cpu_dg_rate(config: str, steps: int, warmup: int, min_seconds: float = 0.0):
    """Oracle SSP-RK3 on the sample with every host core (per-color process
    chunks, oracle/dg_parallel.py).  Returns edges/s, DOF-updates/s and a
    description."""
    from oracle import dg_parallel as DP
    prob, U, ne, ns, sample = oracle_sample(config)
    cores = host_cores()
    st = DP.ParallelStepper(prob, U, workers=cores)
    dt = 1e-3
    try:
        for _ in range(max(warmup, 0)):
            st.step(dt)
        done, t_all, times = 0, 0.0, []
        while True:
            t0 = time.perf_counter()
            st.step(dt)
            times.append(time.perf_counter() - t0)
            t_all += times[-1]
            done += 1
            if done >= steps and t_all >= min_seconds:
                break
        finite = bool(np.isfinite(st.U).all())
    finally:
        st.close()
    nb, neq = U.shape[2], U.shape[1]
    return dict(edges_per_s=3 * ns * done / t_all, dofs_per_s=ne * nb * neq * 3 * done / t_all,
                seconds=t_all, steps=done, ms_per_step=1e3 * t_all / done, cores=cores,
                ne=ne, ns=ns, finite=finite,
                sample=f"oracle/dg_oracle.py numpy fp64 SSP-RK3 on {sample} (same family as "
                       f"the config; oracle mesh, coloring and problem), {cores} worker "
                       f"processes (Algorithm 1 per-color chunks), {done} steps in "
                       f"{t_all:.1f} s; CPU {cpu_model()}")


def run_reference(args):
    """--impl reference: the reference's CPU path for this workload on the
    box's host cores — the oracle port (the reference has no DG), built
    from oracle/ only; rank 0 alone runs, other ranks exit 0."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = args.config
    r = cpu_dg_rate(cfg, args.steps, args.warmup)
    loaded = product_library_loaded()
    if loaded:
        raise SystemExit("reference arm loaded the product library")
    value = r["edges_per_s"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": r["steps"], "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if cfg == "c4" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (density wave on far-field stream)",
        "config": {"workload": CONFIGS[cfg][0], "sample": r["sample"],
                   "sample_elements": r["ne"], "sample_surfaces": r["ns"],
                   "host_cores": host_cores(), "os_cpu_count": os.cpu_count(),
                   "cpu_model": cpu_model()},
        "dof_updates_per_s": r["dofs_per_s"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": "port",
                         "sample": r["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_library_loaded": loaded,
        "finite": r["finite"],
    }
    print(json.dumps(line))


# ------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the paper's comparisons (buffered/atomic, integer sweeps)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--layouts", action="store_true",
                    help="time the paper's Table 7 layouts on c2 instead")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "push"],
                    help="N>1 ghost exchange: NCCL send/recv of kernel-packed rows (default) "
                         "or the peer push fused into the last-touch kernel (symmetric memory)")
    ap.add_argument("--state", default="f64", choices=["f64", "f32"],
                    help="element-block storage (f32: half the bytes, fp64 arithmetic, the north "
                         "star's 1e-5 tolerance; not the headline)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.layouts:
        return run_layouts(args)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # MC_DIST_BACKEND=gloo: functional run of the N>1 path with host-staged
    # exchanges (e.g. several ranks on one GPU to exercise the code); never a
    # measurement — the scaling numbers are NCCL over NVLink, one rank per GPU
    backend = os.environ.get("MC_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local % torch.cuda.device_count())
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def reduce_scalar(x, op):
        t = torch.tensor([x], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=op)
        return float(t.item())
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")

    spec = config_spec(args.config)
    t_setup = time.perf_counter()
    op = build_operator(spec, world=world, rank=rank, state=args.state)
    t_setup = time.perf_counter() - t_setup
    U_host = op.initial_state("wave")
    dt = op.stable_dt(0.2)
    if world > 1:                      # one global time step; also initialises NCCL P2P
        dt = reduce_scalar(dt, dist.ReduceOp.MIN)
        dist.barrier()
    push = world > 1 and args.exchange == "push"
    if push:   # exchange fused into the last-touch kernel over NVLink peer memory
        from paper_1601_07613_b200.partition import setup_symmetric_push
        U, push_fill, push_barrier = setup_symmetric_push(op)
        U[: op.n_elements] = op.to_device(U_host)[: op.n_elements]
        push_fill()
    else:
        U = op.to_device(U_host)
    work = op.work_device()
    U0, R = work[0], work[1]
    stream = torch.cuda.current_stream()
    nc = op.n_colors
    stage_no = [0]

    def mark(events, mode, a, c):
        if events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            events.append((mode, a, c, ev))

    def step(events=None):
        for mode, a, b in STAGES:
            if op.halo is None:
                for c in range(1, nc + 1):
                    mark(events, mode, a, c)
                    op.color_pass_device(c, U, U0, R, mode, a, b, dt, stream)
                continue
            if push:   # ghosts pushed by the peers' last touches; one barrier per stage
                op.stage_push(U, U0, R, mode, a, b, dt, stage_no[0], push_barrier, stream,
                              marker=lambda c, m=mode, aa=a: mark(events, m, aa, c))
                stage_no[0] += 1
                continue
            # ghost exchange overlapped with the ghost-free part of color 1;
            # the send rows were packed by the previous stage's last touches
            op.stage_distributed(U, U0, R, mode, a, b, dt, stream,
                                 marker=lambda c, m=mode, aa=a: mark(events, m, aa, c))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    events = []
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record(stream)
        for _ in range(args.steps):
            step(events)
        end.record(stream)
        end.synchronize()
    barrier()
    total_ms = start.elapsed_time(end)
    if world > 1:
        total_ms = reduce_scalar(total_ms, dist.ReduceOp.MAX)
    ms_per_step = total_ms / max(args.steps, 1)
    ns_global = op.n_surfaces if world == 1 else op.mesh.n_surfaces
    ne_global = op.mesh.n_elements
    value = 3 * ns_global / (ms_per_step * 1e-3)
    dof_rate = ne_global * op.n_basis * op.n_equations * 3 / (ms_per_step * 1e-3)

    # per-launch durations of the colored kernel from the timed region
    per = {}
    marks = events + [(None, None, None, end)]
    for (mode, a, c, ev), (_, _, _, nxt) in zip(events, marks[1:]):
        per.setdefault((mode, a, c), []).append(ev.elapsed_time(nxt))
    bytes_step, ms_step = 0, 0.0
    by_color = {}
    for (mode, a, c), ts in per.items():
        avg = float(np.mean(ts))
        by = launch_bytes(op, c, mode, a)
        bytes_step += by
        ms_step += avg
        by_color.setdefault(c, [0, 0.0])
        by_color[c][0] += by
        by_color[c][1] += avg
    peak, peak_src = peaks()
    achieved = bytes_step / (ms_step * 1e-3) / 1e9
    traffic, traffic_src = None, None
    tf = ROOT / "profiles" / f"traffic_{args.config}.json"
    if tf.exists():
        try:
            d = json.loads(tf.read_text())
            traffic = d.get("bytes_per_launch_avg")
            traffic_src = f"profiles/{tf.name} (ncu --set full capture {d.get('tag')})"
        except Exception:
            traffic = None
    finite = bool(torch.isfinite(U).all().item())

    # end to end through the public API (DGOperator.ssprk3, caller's order)
    W = op.block_width()
    if world == 1:
        pinned = torch.empty((ne_global, W), dtype=torch.float64, pin_memory=True)
        host = pinned.numpy()
        host[:] = U_host.reshape(ne_global, W)
        op.ssprk3(host, dt, 1, inplace=True)                    # warm (staging, graph)
        host[:] = U_host.reshape(ne_global, W)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            op.ssprk3(host, dt, 1, inplace=True)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        io_bytes = ne_global * W * 8
    else:
        own = op.n_elements
        pinned = torch.empty((own, W), dtype=torch.float64, pin_memory=True)
        pinned.copy_(torch.from_numpy(op.user_rows(U_host)))
        dev_user = torch.empty_like(pinned, device="cuda")
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            dev_user.copy_(pinned, non_blocking=True)
            op.user_to_device(dev_user, U)
            if push:
                push_fill(stage_no[0] % 2)
                stage_no[0] = op.ssprk3_push(U, work, dt, 1, push_barrier, stage0=stage_no[0])
            else:
                op.ssprk3_distributed(U, work, dt, 1)
            op.device_to_user(U, dev_user)
            pinned.copy_(dev_user, non_blocking=True)
            torch.cuda.synchronize()
        barrier()
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        e2e_s = reduce_scalar(e2e_s, dist.ReduceOp.MAX)
        io_bytes = own * W * 8 * world
    e2e_value = 3 * ns_global / e2e_s

    comparisons = None
    if not args.no_variants and world == 1 and args.state == "f64":
        comparisons = variants(op, U_host, stream)

    cpu = None
    if rank == 0 and not args.no_cpu:
        r = cpu_dg_rate(args.config, 1, 1, min_seconds=10.0)
        cpu = {"value": r["edges_per_s"], "unit": UNIT, "cores": r["cores"], "kind": "port",
               "sample": r["sample"], "dof_updates_per_s": r["dofs_per_s"]}

    strong = world > 1 or args.config == "c4"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": "f64" if args.state == "f64" else "f32 storage, f64 arithmetic",
        "data": "synthetic (density wave on far-field stream)",
        "config": {"workload": spec["desc"] + ("" if world == 1 else
                                               f", split over {world} GPUs"),
                   "elements": ne_global, "surfaces": ns_global, "colors": nc,
                   "degree": op.degree, "n_basis": op.n_basis, "n_equations": op.n_equations,
                   "step": "1 SSP-RK3 step = 3 fused colored RHS (volume fused into first "
                           "color pass, RK update into last)",
                   "layout": f"{op.ordering} (color-major: reorder.build_plan structure, "
                             "color-1 pairs in Z-order)" if op.ordering == "sfc"
                             else op.ordering,
                   "kernel": kernel_name(op),
                   "l2": f"inputs larger than L2 (state "
                         f"{op.n_local * op.stride * (4 if args.state == 'f32' else 8) / 1e9:.2f}"
                         " GB x 3 arrays, no flush needed)",
                   "parallelism": "single-GPU" if world == 1 else
                   (f"domain decomposition x{world} (slabs, ghost blocks pushed into the peers' "
                    "double-buffered ghost rows by the last-touch kernel over NVLink symmetric "
                    "memory, one device barrier per stage)" if push else
                    f"domain decomposition x{world} (slabs, {backend.upper()} ghost exchange per "
                    f"stage{'' if backend == 'nccl' else ', host-staged: functional run only'})"),
                   "setup_s": round(t_setup, 2)},
        "dof_updates_per_s": dof_rate,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src, "frac_of_8tbs_nominal": achieved / 8000.0,
                     "kernel": kernel_name(op),
                     "algorithmic_bytes_per_step": bytes_step,
                     "kernel_ms_per_step": ms_step,
                     "per_color_gbs": {str(c): v[0] / (v[1] * 1e-3) / 1e9
                                       for c, v in sorted(by_color.items())},
                     "per_color_ms": {str(c): v[1] for c, v in sorted(by_color.items())}},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": io_bytes,
                "d2h_bytes_per_step": io_bytes,
                "api": "DGOperator.ssprk3(U_pinned, dt, 1, inplace=True) (caller's element "
                       "order; device permutation)" if world == 1 else
                       "per rank: owned rows H2D, device permutation, ssprk3_distributed, "
                       "permutation back, D2H"},
        # our kernel launches in the timed region: one per color per stage
        # (partitioned: color 1 in two parts around the ghost exchange)
        "gpu_launches": args.steps * 3 * (nc + (1 if op.halo is not None else 0)),
        "clocks": clk.summary(),
        "finite": finite,
    }
    if comparisons is not None:
        line["comparisons"] = comparisons
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def variants(op, U_host, stream, reps=5):
    """The paper's comparisons on the same mesh: colored vs buffered vs
    atomic RHS, buffer memory avoided, the integer Algorithm 1 sweeps on
    the GPU, and the reference's integer CPU path beside them."""
    import torch
    import paper_1601_07613_b200 as P
    from oracle import sweeps_oracle as SO
    from paper_1601_07613_b200.sweeps import DeviceLayout
    out = {}
    U = torch.from_numpy(op.to_internal(U_host)).cuda()
    R = torch.zeros_like(U)

    def timeit(fn):
        fn()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b) / reps

    for strat in ("colored", "buffered", "atomic"):
        ms = timeit(lambda: op.rhs_device(U, R, strat, stream))
        out[f"rhs_{strat}_ms"] = ms
        out[f"rhs_{strat}_edges_per_s"] = op.n_surfaces / (ms * 1e-3)
    out["colored_vs_buffered"] = out["rhs_buffered_ms"] / out["rhs_colored_ms"]
    out["colored_vs_atomic"] = out["rhs_atomic_ms"] / out["rhs_colored_ms"]
    mem = P.memory_saved(op.degree, op.n_equations, op.n_surfaces,
                         {"tri": "tri", "quad": "quad", "tet": "tet",
                          "hybrid": "quad"}[op.kind.value])   # hybrid slots are quad-sized
    out["buffer_bytes_avoided"] = mem.n_bytes
    out["buffer_gb_truncated"] = mem.gb_truncated
    del R
    torch.cuda.empty_cache()
    # integer Algorithm 1 on the reordered mesh
    lay = DeviceLayout(op.layout_mesh, op.layout_coloring)
    m = op.layout_mesh
    nsm = m.n_surfaces                 # mesh surfaces (AMR: incl. coarse full edges)
    pay_h = P.default_payload(nsm)
    pay = torch.from_numpy(pay_h).cuda()
    tot = torch.zeros(m.n_elements, dtype=torch.int64, device="cuda")
    buf = torch.zeros(2 * nsm, dtype=torch.int64, device="cuda")
    for name, fn in (("int_colored", lambda: lay.sweep_colored(pay, tot, stream)),
                     ("int_buffered", lambda: lay.sweep_buffered(pay, buf, tot, stream)),
                     ("int_atomic", lambda: lay.sweep_atomic(pay, tot, stream))):
        ms = timeit(fn)
        out[f"{name}_ms"] = ms
        out[f"{name}_edges_per_s"] = nsm / (ms * 1e-3)
    lay.sweep_colored(pay, tot, stream)
    torch.cuda.synchronize()
    gpu_tot = tot.cpu().numpy()
    # the reference's integer CPU path (sweeps.py:74-86 and :114-152,
    # restated in oracle/sweeps_oracle.py) on the same mesh, beside it
    se = np.ascontiguousarray(m.surf_elems)
    cores = host_cores()
    t0 = time.perf_counter()
    seq = SO.sweep_sequential_loop(se, m.n_elements, pay_h)
    t_seq = time.perf_counter() - t0
    t0 = time.perf_counter()
    thr = SO.sweep_colored_threads(se, m.n_elements, pay_h, op.layout_coloring.colors,
                                   int(op.layout_coloring.n_colors), cores)
    t_thr = time.perf_counter() - t0
    out["cpu_int_sequential"] = {
        "kind": "port", "cores": 1, "seconds": t_seq, "edges_per_s": nsm / t_seq,
        "sample": "oracle/sweeps_oracle.sweep_sequential_loop (the reference's "
                  "sweep_sequential: interpreted per-surface loop), full mesh"}
    out["cpu_int_colored_threads"] = {
        "kind": "port", "cores": cores, "seconds": t_thr, "edges_per_s": nsm / t_thr,
        "sample": f"oracle/sweeps_oracle.sweep_colored_threads (the reference's "
                  f"sweep_colored(workers=os.cpu_count()={cores})), full mesh"}
    out["cpu_model"] = cpu_model()
    out["int_colored_equals_cpu"] = bool(np.array_equal(gpu_tot, seq) and
                                         np.array_equal(thr, seq))
    return out


def run_layouts(args):
    """The paper's Table 7 on the GPU: {color() 3
    colors, naive_greedy 5 colors} x {none, renumber, reorder, sfc} on c2
    (shuffled tri 708^2, Euler p=2), one SSP-RK3 step each."""
    import torch
    import paper_1601_07613_b200 as P
    from paper_1601_07613_b200.dg import DGOperator
    torch.cuda.set_device(0)
    mesh = P.shuffle_elements(P.gen_tri_rect(708, 708, device="cuda"), 0, device="cuda")
    pal = {"color": P.color(mesh)[0], "naive_greedy": P.naive_greedy(mesh)}
    out = {}
    stream = torch.cuda.current_stream()
    for pname, col in pal.items():
        for ordering in ("none", "renumber", "reorder", "sfc"):
            op = DGOperator(mesh, col, degree=2, physics="euler", ordering=ordering)
            U = torch.from_numpy(op.to_internal(op.initial_state("wave"))).cuda()
            work = op.work_device()
            dt = op.stable_dt(0.2)
            for _ in range(args.warmup):
                op.ssprk3_device(U, work, dt, 1, stream)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            op.ssprk3_device(U, work, dt, args.steps, stream)
            b.record(stream)
            b.synchronize()
            ms = a.elapsed_time(b) / args.steps
            lm, lc = op.layout_mesh, op.layout_coloring
            out[f"{pname}/{ordering}"] = {
                "n_colors": int(col.n_colors), "ms_per_step": ms,
                "edges_per_s": 3 * op.n_surfaces / (ms * 1e-3),
                "plan_fallback": bool(op.plan.used_fallback),
                "coalescing": float(P.coalescing_metric(lm, lc).aggregate)}
            del op, U, work
            torch.cuda.empty_cache()
    print(json.dumps({"layouts": out, "config": CONFIGS["c2"][0], "steps": args.steps,
                      "warmup": args.warmup}))


if __name__ == "__main__":
    main()
