"""ctypes binding of libhvb.so (C ABI in include/hvb.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the library or a CUDA device is missing, every
device entry point raises :class:`DeviceUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

__all__ = ["lib", "call", "LIB_PATH", "DeviceUnavailable", "HvbError", "ptr", "stream_ptr"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhvb.so")

_P = ctypes.c_void_p
_I = ctypes.c_int
_LL = ctypes.c_longlong
_D = ctypes.c_double

# name -> argtypes (all return int status)
SIGNATURES = {
    "hvb_build_table": [_P, _I, _I, _P, _P, _P],
    "hvb_build_stream": [_P, _I, _P, _D, _P, _P, _LL, _I, _I, _P, _P],
    "hvb_panel_data": [_P, _P, _I, _D, _P, _P, _P, _P],
    "hvb_sweep_geometry": [_P],
    "hvb_assemble_regular": [_P] * 11 + [_I, _I, _P, _I, _I, _P, _P, _P, _P, _P, _LL, _P, _I, _P, _P, _P, _P, _LL, _P],
    "hvb_assemble_singular": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _P],
    "hvb_charge_reduce": [_P, _I, _LL, _I, _P, _I, _P],
    "hvb_fill_float_cols": [_P, _P, _P, _I, _I, _I, _P],
    "hvb_near_pairs": [_P, _LL, _P, _P, _P, _P, _P, _I, _P, _I, _I, _D, _P, _P],
    "hvb_near_apply_rows": [_P, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "hvb_gemv": [_P, _I, _LL, _I, _I, _P, _P, _P, _P],
    "hvb_gather_scale": [_P, _P, _P, _I, _P, _P],
    "hvb_gemv_bcast": [_P, _LL, _I, _I, _P, _P, _P, _I, _LL, _P, _I, ctypes.c_ulonglong, _P, _P],
    "hvb_ipc_alloc": [_LL, _P],
    "hvb_ipc_free": [_P],
    "hvb_ipc_handle": [_P, _P],
    "hvb_ipc_open": [_P, _P],
    "hvb_ipc_close": [_P],
    "hvb_peer_wait": [_P, _I, ctypes.c_ulonglong, _P],
    "hvb_rowmax_diag": [_P, _I, _LL, _I, _I, _P, _P, _P, _P],
    "hvb_mgs": [_P, _LL, _I, _P, _I, _P, _P, _P, _I, _P],
    "hvb_contract": [_P, _I, _I, _P, _P, _P, _P],
    "hvb_field": [_P, _P, _P, _P, _I, _I, _P, _P, _I, _I, _I, _P, _P, _P, _LL, _P],
    "hvb_field_reduce": [_P, _I, _I, _P, _P],
    "hvb_near_apply_points": [_P, _I, _P, _P, _P, _P, _I, _P, _P],
    "hvb_field_singular": [_P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _I, _P, _D, _P, _P, _P],
    "hvb_trace_ctrl": [_P, _I, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P],
    "hvb_trace_summary": [_P, _I, _P, _P, _P],
    "hvb_trace_round": [_P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P,
                        _P, _P, _I, _P, _I, _I, _D, _D, _P, _I, _P],
    "hvb_surface_distance": [_P, _I, _P, _P, _I, _P, _P, _P],
    "hvb_near_coincide": [_P, _LL, _P, _P, _D, _P, _P],
    "hvb_streamer": [_P, _P, _I, _I, _P, _P, _I, _D, _P, _P, _P],
    "hvb_tiling_build": [_P, _I, _P, _I, _I, _I, _I, _P, _P],
    "hvb_tiling_fetch": [_P] * 15,
    "hvb_tiling_free": [_P],
    "hvb_bench_dfma": [_P, _I, _I, _P],
    "hvb_bench_read": [_P, _LL, _P, _I, _P],
}

HVB_EARG = 1
HVB_ECUDA = 2


class DeviceUnavailable(RuntimeError):
    """libhvb.so is not built or no CUDA device is visible."""


class HvbError(RuntimeError):
    """A libhvb.so entry point returned a CUDA error."""


_lock = threading.Lock()
_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceUnavailable(
                    f"{LIB_PATH} is missing; run __graft_entry__.build() (nvcc sm_100a) first"
                )
            h = ctypes.CDLL(LIB_PATH)
            for name, args in SIGNATURES.items():
                fn = getattr(h, name)
                fn.argtypes = args
                fn.restype = _I
            h.hvb_last_error.restype = ctypes.c_char_p
            h.hvb_last_error.argtypes = []
            h.hvb_version.restype = _I
            h.hvb_line_state_bytes.restype = _I
            h.hvb_line_state_bytes.argtypes = []
            h.hvb_mgs_partial_size.restype = _I
            h.hvb_mgs_partial_size.argtypes = []
            h.hvb_ipc_handle_bytes.restype = _I
            h.hvb_ipc_handle_bytes.argtypes = []
            h.hvb_stream_record_doubles.restype = _I
            h.hvb_stream_record_doubles.argtypes = [_I, _I]
            h.hvb_sweep_sched_ints.restype = _LL
            h.hvb_sweep_sched_ints.argtypes = [_I, _I]
            _lib = h
    return _lib


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().hvb_last_error().decode(errors="replace")
        if rc == HVB_EARG:
            raise ValueError(msg)
        raise HvbError(msg)


def ptr(t):
    """Device pointer of a tensor (or None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(device=None):
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def require_device(device=None):
    """Resolve the CUDA device for a device entry point, failing loudly."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceUnavailable("no CUDA device visible; the hvb kernels run on B200 (sm_100a) only")
    lib()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)
