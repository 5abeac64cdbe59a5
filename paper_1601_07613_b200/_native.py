"""ctypes binding of ``libmeshchroma_b200.so`` (include/meshchroma_b200.h).

This is the same binding a maintainer of the reference would add (see
INTEGRATION.md): plain pointers and sizes, int status codes mapped back to
the reference's exception types.  There is no fallback — if the library is
missing or cannot serve a call, ``NativeLibraryError`` is raised.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import errors

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libmeshchroma_b200.so"

MC_OK, MC_EINVAL, MC_ECONFLICT, MC_ESWAPBUDGET, MC_ERESTARTS = 0, 1, 2, 3, 4
MC_EAUDIT, MC_EINTERNAL, MC_ECUDA, MC_ENOMEM, MC_EUNSUPPORTED = 5, 6, 7, 8, 9
MC_ENONMANIFOLD = 10

_STATUS_TO_EXC = {
    MC_EINVAL: ValueError,
    MC_ECONFLICT: errors.WriteConflictError,
    MC_ESWAPBUDGET: errors.SwapBudgetExceededError,
    MC_ERESTARTS: errors.RestartsExhaustedError,
    MC_EAUDIT: AssertionError,
    MC_EINTERNAL: AssertionError,
    MC_ECUDA: errors.NativeLibraryError,
    MC_ENOMEM: MemoryError,
    MC_EUNSUPPORTED: NotImplementedError,
    MC_ENONMANIFOLD: errors.NonManifoldError,
}


class ColoringStats(C.Structure):
    _fields_ = [("greedy_conflicts", C.c_int64), ("resolutions", C.c_int64),
                ("swaps", C.c_int64), ("loop_breaks", C.c_int64),
                ("no_swap_breaks", C.c_int64), ("forced_reswaps", C.c_int64),
                ("restarts", C.c_int64), ("greedy_seconds", C.c_double),
                ("resolve_seconds", C.c_double), ("total_seconds", C.c_double)]


class DGDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("physics", C.c_int), ("degree", C.c_int),
        ("n_colors", C.c_int),
        ("n_elements", C.c_int64), ("n_ghosts", C.c_int64),
        ("n_surfaces", C.c_int64),
        ("group_bounds", C.c_void_p), ("surf_left", C.c_void_p),
        ("surf_right", C.c_void_p), ("surf_code", C.c_void_p),
        ("surf_geom", C.c_void_p), ("elem_jinv", C.c_void_p),
        ("elem_slot_ptr", C.c_void_p), ("elem_slots", C.c_void_p),
        ("n_face_codes", C.c_int), ("n_face_q", C.c_int),
        ("n_vol_q", C.c_int), ("n_basis", C.c_int),
        ("face_phi", C.c_void_p), ("face_w", C.c_void_p),
        ("vol_phi", C.c_void_p), ("vol_dphi", C.c_void_p),
        ("vol_w", C.c_void_p),
        ("gamma", C.c_double), ("velocity", C.c_double * 3),
        ("farfield", C.c_double * 5),
        ("state_f32", C.c_int),
        ("elem_kind", C.c_void_p),
    ]


_P = C.c_void_p
_I64 = C.c_int64
_SIGS = {
    "mc_last_error": (C.c_char_p, []),
    "mc_abi_version": (C.c_int, []),
    "mc_device_count": (C.c_int, []),
    "mc_color": (C.c_int, [_I64, _I64, _P, _P, C.c_int, _I64, _I64, C.c_int,
                           C.c_int, _P, C.POINTER(ColoringStats)]),
    "mc_modified_greedy": (C.c_int, [_I64, _I64, _P, C.c_int, _I64, _P, _P]),
    "mc_resolve_conflicts": (C.c_int, [_I64, _I64, _P, _P, C.c_int, _I64, _I64,
                                       C.c_int, _P, C.POINTER(ColoringStats)]),
    "mc_naive_greedy": (C.c_int, [_I64, _I64, _P, _P, _P]),
    "mc_layout_create": (C.c_int, [_I64, _I64, _P, _P, _P, C.c_int,
                                   C.POINTER(_P)]),
    "mc_layout_destroy": (C.c_int, [_P]),
    "mc_layout_color_size": (_I64, [_P, C.c_int]),
    "mc_layout_race_check": (C.c_int, [_P, _P]),
    "mc_sweep_colored_i64": (C.c_int, [_P, _P, _P, _P]),
    "mc_surface_buffer_i64": (C.c_int, [_P, _P, _P, _P]),
    "mc_sweep_buffered_i64": (C.c_int, [_P, _P, _P, _P, _P]),
    "mc_sweep_atomic_i64": (C.c_int, [_P, _P, _P, _P]),
    "mc_sweep_i64_host": (C.c_int, [_P, C.c_int, _P, _P]),
    "mc_default_payload_dev": (C.c_int, [_I64, _I64, _P, _P]),
    "mc_dg_create": (C.c_int, [C.POINTER(DGDesc), C.POINTER(_P)]),
    "mc_dg_destroy": (C.c_int, [_P]),
    "mc_dg_block_stride": (_I64, [_P]),
    "mc_dg_buffer_bytes": (_I64, [_P]),
    "mc_dg_rhs": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "mc_dg_rk_stage": (C.c_int, [_P, _P, _P, _P, C.c_double, C.c_double,
                                 C.c_double, _P]),
    "mc_dg_color_pass": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, C.c_double,
                                   C.c_double, C.c_double, _P]),
    "mc_dg_color_range_pass": (C.c_int, [_P, C.c_int, _I64, _I64, _P, _P, _P, C.c_int,
                                         C.c_double, C.c_double, C.c_double, _P]),
    "mc_dg_ssprk3": (C.c_int, [_P, _P, _P, C.c_double, C.c_int, _P]),
    "mc_dg_ssprk3_host": (C.c_int, [_P, _P, C.c_double, C.c_int]),
    "mc_dg_set_grid_cap": (C.c_int, [_P, C.c_int]),
    "mc_dg_set_send_rows": (C.c_int, [_P, _P, _P, _I64]),
    "mc_dg_set_push_rows": (C.c_int, [_P, _P, _P, _I64]),
    "mc_dg_set_ghost_parity": (C.c_int, [_P, C.c_int, C.c_int]),
    "mc_dg_set_user_rows": (C.c_int, [_P, _P, _I64]),
    "mc_dg_user_to_internal": (C.c_int, [_P, _P, _P, _P]),
    "mc_dg_internal_to_user": (C.c_int, [_P, _P, _P, _P]),
    "mc_dg_ssprk3_user_host": (C.c_int, [_P, _P, C.c_double, C.c_int]),
    "mc_dg_rhs_user_host": (C.c_int, [_P, _P, _P, C.c_int]),
    "mc_assemble_create": (C.c_int, [_I64, _I64, _P, _P, C.c_int, C.POINTER(_P),
                                     C.POINTER(_I64)]),
    "mc_assemble_result": (C.c_int, [_P, _P, _P, _P, _P]),
    "mc_assemble_destroy": (C.c_int, [_P]),
    "mc_amr_classify": (C.c_int, [_I64, _P, _I64, _I64, _P, _I64, _P, _P, _P, _P, _P, _P]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def library_path() -> Path:
    return _LIB_PATH


def lib():
    """Load (once) and return the bound library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise errors.NativeLibraryError(
            f"{_LIB_PATH} is missing: run __graft_entry__.build() "
            "(nvcc, sm_100a); there is no CPU fallback")
    try:
        handle = C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    except OSError as exc:
        raise errors.NativeLibraryError(f"cannot load {_LIB_PATH}: {exc}")
    missing = [n for n in _SIGS if not hasattr(handle, n)]
    if missing:
        raise errors.NativeLibraryError(
            f"{_LIB_PATH} is stale (missing {missing}); rebuild it")
    for name, (res, args) in _SIGS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().mc_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    if status == MC_OK:
        return
    exc = _STATUS_TO_EXC.get(status, errors.NativeLibraryError)
    raise exc(last_error())


def ptr(a) -> int | None:
    """Data pointer of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    return a.data_ptr()


def stream_ptr(stream=None) -> int | None:
    """cudaStream_t of a torch stream (current stream when None)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_device() -> None:
    """Fail loudly when there is no GPU: device entry points never fall
    back to the CPU."""
    if lib().mc_device_count() < 1:
        raise errors.NativeLibraryError(
            "no CUDA device visible: the sm_100a sweep/DG kernels need a B200 "
            "(there is no CPU fallback)")
