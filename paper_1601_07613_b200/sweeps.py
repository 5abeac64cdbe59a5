"""Algorithm 1 integer harness on the B200 (drop-in for ``meshchroma.sweeps``).

Same names, arguments, return types and errors as
/root/reference/pkg/src/meshchroma/sweeps.py; the accumulation runs in the
sm_100a kernels of ``csrc/sweeps.cu`` through the C ABI:

* ``sweep_colored``   -> one ``k_sweep_color`` launch per color, stream
  order as the inter-color barrier (sweeps.py:114-152);
* ``surface_buffer`` / ``sweep_buffered`` -> fill + gather kernels
  (sweeps.py:155-204);
* ``sweep_atomic``    -> one ``atomicAdd`` launch, no coloring (new; the
  paper's third strategy, absent from the reference);
* ``assert_race_free`` -> device race certificate (sweeps.py:89-105);
* ``sweep_sequential`` -> the reference's oracle order; integers make the
  result order-independent, so it runs as the atomic kernel.

``workers`` is accepted for signature compatibility and ignored: the GPU
grid replaces the thread pool.  There is no CPU fallback — every call needs
the extension and a CUDA device and raises ``NativeLibraryError`` otherwise.
"""

from __future__ import annotations

import weakref
import zlib
from dataclasses import dataclass

import numpy as np

from . import _native
from .coloring import SurfaceColoring
from .errors import WriteConflictError  # noqa: F401  (re-exported semantics)
from .mesh import Mesh

_GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1


@dataclass
class AccumulationState:
    """Per-element integer totals plus the payload that fed them."""

    totals: np.ndarray
    payload: np.ndarray

    def checksum(self) -> int:
        return zlib.crc32(self.totals.astype("<i8").tobytes())


def default_payload(n_surfaces: int, seed: int = 0) -> np.ndarray:
    """Deterministic 20-bit signed payload per surface (splitmix64,
    sweeps.py:55-62).  Host-side input generation; the device twin is
    ``mc_default_payload_dev``."""
    z = np.arange(1, n_surfaces + 1, dtype=np.uint64) * np.uint64(_GOLDEN)
    z += np.uint64((seed * _MIX2) & _MASK)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
    z ^= z >> np.uint64(31)
    return (z >> np.uint64(44)).astype(np.int64) - (1 << 19)


def _payload_for(mesh: Mesh, payload) -> np.ndarray:
    if payload is None:
        return default_payload(mesh.n_surfaces)
    payload = np.ascontiguousarray(payload, dtype=np.int64)
    if payload.shape != (mesh.n_surfaces,):
        raise ValueError("payload must provide one integer per surface")
    return payload


class DeviceLayout:
    """Color-major incidence of one (mesh, coloring) on the device
    (``mc_layout``).  ``coloring=None`` builds the uncolored layout used
    by the buffered and atomic strategies."""

    def __init__(self, mesh: Mesh, coloring: SurfaceColoring | None):
        lib = _native.lib()
        _native.require_device()
        se = np.ascontiguousarray(mesh.surf_elems, dtype=np.int64)
        es = np.ascontiguousarray(mesh.elem_surfs, dtype=np.int64)
        if coloring is None:
            colors = np.ones(mesh.n_surfaces, dtype=np.int32)
            n_colors = 1
        else:
            colors = np.ascontiguousarray(coloring.colors, dtype=np.int32)
            n_colors = int(coloring.n_colors)
        h = _native.C.c_void_p()
        _native.check(lib.mc_layout_create(
            mesh.n_surfaces, mesh.n_elements, _native.ptr(se), _native.ptr(es),
            _native.ptr(colors), n_colors, _native.C.byref(h)))
        self.handle = h
        self.n_surfaces = mesh.n_surfaces
        self.n_elements = mesh.n_elements
        self.n_colors = n_colors
        self._lib = lib
        self.race_checked = False

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.mc_layout_destroy(h)
            self.handle = None

    def color_sizes(self) -> tuple:
        return tuple(int(self._lib.mc_layout_color_size(self.handle, c))
                     for c in range(1, self.n_colors + 1))

    def race_check(self, stream=None) -> None:
        _native.check(self._lib.mc_layout_race_check(
            self.handle, _native.stream_ptr(stream)))
        self.race_checked = True

    # device-pointer entry points (payload/totals are torch CUDA tensors)
    def sweep_colored(self, payload_dev, totals_dev, stream=None) -> None:
        _native.check(self._lib.mc_sweep_colored_i64(
            self.handle, _native.ptr(payload_dev), _native.ptr(totals_dev),
            _native.stream_ptr(stream)))

    def sweep_buffered(self, payload_dev, buffer_dev, totals_dev,
                       stream=None) -> None:
        _native.check(self._lib.mc_sweep_buffered_i64(
            self.handle, _native.ptr(payload_dev), _native.ptr(buffer_dev),
            _native.ptr(totals_dev), _native.stream_ptr(stream)))

    def surface_buffer(self, payload_dev, buffer_dev, stream=None) -> None:
        _native.check(self._lib.mc_surface_buffer_i64(
            self.handle, _native.ptr(payload_dev), _native.ptr(buffer_dev),
            _native.stream_ptr(stream)))

    def sweep_atomic(self, payload_dev, totals_dev, stream=None) -> None:
        _native.check(self._lib.mc_sweep_atomic_i64(
            self.handle, _native.ptr(payload_dev), _native.ptr(totals_dev),
            _native.stream_ptr(stream)))

    def sweep_host(self, strategy: int, payload: np.ndarray) -> np.ndarray:
        """End-to-end through host buffers (``mc_sweep_i64_host``)."""
        payload = np.ascontiguousarray(payload, dtype=np.int64)
        totals = np.empty(self.n_elements, dtype=np.int64)
        _native.check(self._lib.mc_sweep_i64_host(
            self.handle, int(strategy), _native.ptr(payload),
            _native.ptr(totals)))
        return totals


# per-mesh cache, keyed like the reference's incidence cache (identity of the
# immutable Mesh); the mutable coloring is keyed by its current contents
_layouts: "weakref.WeakKeyDictionary[Mesh, dict]" = weakref.WeakKeyDictionary()


def device_layout(mesh: Mesh, coloring: SurfaceColoring | None) -> DeviceLayout:
    per_mesh = _layouts.setdefault(mesh, {})
    if coloring is None:
        key = None
    else:
        colors = np.ascontiguousarray(coloring.colors, dtype=np.int32)
        key = (int(coloring.n_colors), len(colors),
               zlib.crc32(colors.tobytes()), colors.tobytes()[:64])
    lay = per_mesh.get(key)
    if lay is None:
        if len(per_mesh) > 8:
            per_mesh.clear()
        lay = DeviceLayout(mesh, coloring)
        per_mesh[key] = lay
    return lay


def _to_device(a: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", non_blocking=False)


def _empty_i64(n: int):
    import torch
    return torch.empty(max(n, 1), dtype=torch.int64, device="cuda")


def _collect(t, n: int) -> np.ndarray:
    import torch
    torch.cuda.current_stream().synchronize()
    return t[:n].cpu().numpy()


def assert_race_free(mesh: Mesh, coloring: SurfaceColoring) -> None:
    """Raise WriteConflictError if some color writes an element twice."""
    if len(coloring.colors) != mesh.n_surfaces:
        raise ValueError("coloring does not match the mesh")
    if not coloring.is_complete:
        raise ValueError("colored sweep needs a complete coloring")
    device_layout(mesh, coloring).race_check()


def sweep_colored(mesh: Mesh, coloring: SurfaceColoring, payload=None,
                  workers: int = 4, check: bool = True) -> AccumulationState:
    """Color-by-color accumulation on the GPU (sweeps.py:114-152)."""
    if not coloring.is_complete:
        raise ValueError("colored sweep needs a complete coloring")
    if len(coloring.colors) != mesh.n_surfaces:
        raise ValueError("coloring does not match the mesh")
    lay = device_layout(mesh, coloring)
    if check:
        lay.race_check()
    payload = _payload_for(mesh, payload)
    pay_d = _to_device(payload)
    tot_d = _empty_i64(mesh.n_elements)
    lay.sweep_colored(pay_d, tot_d)
    return AccumulationState(_collect(tot_d, mesh.n_elements), payload)


def sweep_sequential(mesh: Mesh, payload=None) -> AccumulationState:
    """Totals in the reference's sequential order; exact integer addition
    makes any order equal, so this runs the single-launch atomic kernel."""
    payload = _payload_for(mesh, payload)
    lay = device_layout(mesh, None)
    pay_d = _to_device(payload)
    tot_d = _empty_i64(mesh.n_elements)
    lay.sweep_atomic(pay_d, tot_d)
    return AccumulationState(_collect(tot_d, mesh.n_elements), payload)


def sweep_atomic(mesh: Mesh, payload=None) -> AccumulationState:
    """The paper's atomics strategy: no coloring, no buffer."""
    return sweep_sequential(mesh, payload)


def surface_buffer(mesh: Mesh, payload=None, workers: int = 4) -> np.ndarray:
    """Phase one of buffer-and-reduce: slot 2k left, 2k+1 right (0 on the
    boundary) (sweeps.py:155-176)."""
    payload = _payload_for(mesh, payload)
    lay = device_layout(mesh, None)
    pay_d = _to_device(payload)
    buf_d = _empty_i64(2 * mesh.n_surfaces)
    lay.surface_buffer(pay_d, buf_d)
    return _collect(buf_d, 2 * mesh.n_surfaces)


def sweep_buffered(mesh: Mesh, payload=None, workers: int = 4) -> AccumulationState:
    """Fill, barrier (stream order), per-element gather (sweeps.py:179-204)."""
    payload = _payload_for(mesh, payload)
    lay = device_layout(mesh, None)
    pay_d = _to_device(payload)
    buf_d = _empty_i64(2 * mesh.n_surfaces)
    tot_d = _empty_i64(mesh.n_elements)
    lay.sweep_buffered(pay_d, buf_d, tot_d)
    return AccumulationState(_collect(tot_d, mesh.n_elements), payload)


def basis_count(p: int, kind: str = "tri") -> int:
    """Modal basis size: P_p on tri/tet, Q_p on quads (sweeps.py:207-217)."""
    if p < 0:
        raise ValueError("degree must be nonnegative")
    if kind == "tri":
        return (p + 1) * (p + 2) // 2
    if kind == "quad":
        return (p + 1) ** 2
    if kind == "tet":
        return (p + 1) * (p + 2) * (p + 3) // 6
    raise ValueError(f"unknown element kind {kind!r}")


@dataclass(frozen=True)
class MemoryEstimate:
    """Bytes of the two surface buffers a buffered solver needs:
    2 * n_basis * n_equations * n_surfaces doubles (sweeps.py:220-239)."""

    n_basis: int
    n_equations: int
    n_surfaces: int
    n_bytes: int

    def __post_init__(self):
        if min(self.n_basis, self.n_equations, self.n_surfaces,
               self.n_bytes) <= 0:
            raise ValueError("estimate fields must be positive")

    @property
    def gb_truncated(self) -> str:
        hundredths = self.n_bytes * 100 // 10 ** 9
        return f"{hundredths // 100}.{hundredths % 100:02d}"


def memory_saved(p: int, n_equations: int, n_surfaces: int,
                 kind: str = "tri") -> MemoryEstimate:
    """Buffer memory the colored sweep avoids (sweeps.py:242-249)."""
    n_basis = basis_count(p, kind)
    if n_equations < 1 or n_surfaces < 1:
        raise ValueError("equation and surface counts must be positive")
    return MemoryEstimate(n_basis, n_equations, n_surfaces,
                          2 * n_basis * n_equations * n_surfaces * 8)
