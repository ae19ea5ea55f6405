"""ctypes binding of libpdg_b200.so (C ABI declared in include/pdg_b200.h).

There is no CPU fallback: every entry point needs the sm_100a library and a
CUDA device, and raises ``PdgDeviceError`` loudly when either is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# PDG_LIB_PATH: development override (tools/engine_sweep.sh builds variants)
LIB_PATH = os.environ.get("PDG_LIB_PATH") or os.path.join(_HERE, "libpdg_b200.so")

_lock = threading.Lock()
_lib = None
_checked_device = False


class PdgError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


class PdgDeviceError(PdgError):
    """The CUDA library or an sm_100 device is unavailable."""


class HistRows(C.Structure):
    """Mirror of pdg_hist_rows."""
    _fields_ = [("lo", C.c_void_p), ("width", C.c_void_p), ("est_age", C.c_void_p),
                ("nbins", C.c_void_p), ("nsamp", C.c_void_p), ("counts", C.c_void_p),
                ("stride", C.c_int64)]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_D = C.c_double
_SIG = {
    "pdg_last_error": (C.c_char_p, []),
    "pdg_abi_version": (C.c_int, []),
    "pdg_device_info": (C.c_int, [_P, _P, _P]),
    "pdg_gittins_rank_f64": (C.c_int, [_P, _P, _P, _I64, _I32, _P, _P]),
    "pdg_gittins_rank_f64_host": (C.c_int, [_P, _P, _P, _I64, _I32, _P, _P]),
    "pdg_gittins_score_hist": (C.c_int, [C.POINTER(HistRows), _P, _I64, _D, _P, _P, _P, _P, _P,
                                                  _P]),
    "pdg_bucketize": (C.c_int, [_P, _I64, _I32, _I32, _P, _P, _P, _P, _I64, _P]),
    "pdg_order_temp_bytes": (C.c_size_t, [_I64]),
    "pdg_order": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _P, C.c_size_t, _P]),
    "pdg_policy_keys": (C.c_int, [_I32, _P, _P, _P, _P, _P, _D, _I64, _P, _P, _P, _P]),
    "pdg_dispatch_temp_bytes": (C.c_size_t, [_I64, _I32]),
    "pdg_dispatch_plan": (C.c_int, [_P, _P, _P, _P, _P, _P, _I64, _P, _I32, _D, _I32, _I32, _P,
                                    _P, _P, _P, C.c_size_t, _P]),
    "pdg_dispatch_status": (C.c_int, [_P, _I64, _I32, _P, _P]),
    "pdg_order_update_temp_bytes": (C.c_size_t, [_I64, _I64]),
    "pdg_order_update": (C.c_int, [_P, _P, _P, _I64, _P, _I64, _P, _P, _P, _P, C.c_size_t, _P]),
    "pdg_gittins_rank_samples": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _P]),
    "pdg_gittins_rank_samples_host": (C.c_int, [_P, _I32, C.c_double, _P, _P]),
    "pdg_attained_service": (C.c_int, [_P, _P, _I64, _P, _P, _P, _P, _P, _I64, C.c_double,
                                       _P, _P, C.c_size_t, _P]),
    "pdg_prewarm_triggers_temp_bytes": (C.c_size_t, [_I64, _I32]),
    "pdg_prewarm_triggers": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _I32, C.c_double, _I32,
                                       _P, _P, _P, _P, C.c_size_t, _P]),
    "pdg_rank_allgather_sort_temp_bytes": (C.c_size_t, [_I64, C.c_int32]),
    "pdg_rank_allgather_sort": (C.c_int, [_P, _P, _I64, C.c_int32, _P, _P, C.c_int32, _P,
                                          C.c_size_t, _P]),
    "pdg_prewarm_window_index": (C.c_int, [_P, _I32, _P, _I32, _P, _P]),
    "pdg_pearson_flags": (C.c_int, [_P, _P, _P, _P, _I64, _D, _P, _P, _P]),
    "pdg_mc_grid_warps": (C.c_int, []),
    "pdg_mc_scratch_bytes": (C.c_size_t, [_I32, _I32, _I32]),
    "pdg_mc_remaining_demand": (C.c_int, [_P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _P, _P,
                                          C.c_size_t, _P]),
    "pdg_plan_prewarm": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "pdg_prewarm_need": (C.c_int, [_P, _P, _P, _P, _I64, _P, _I32, _I32, _P, _P, _P]),
}

# Every symbol include/pdg_b200.h declares (tests check the .so exports them).
EXPORTS = tuple(_SIG)


def load():
    """Load the library (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise PdgDeviceError(
                    f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIG.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = load().pdg_last_error().decode(errors="replace")
        raise PdgError(f"{what} failed (status {status}): {msg}")


def lib():
    """Library handle after verifying an sm_100 CUDA device is present."""
    global _checked_device
    L = load()
    if not _checked_device:
        import torch
        if not torch.cuda.is_available():
            raise PdgDeviceError("paper_2506_14851_b200 needs a CUDA device (B200, sm_100a); "
                                 "there is no CPU fallback")
        torch.cuda.init()
        sms, major, minor = C.c_int(), C.c_int(), C.c_int()
        check(L.pdg_device_info(C.byref(sms), C.byref(major), C.byref(minor)),
              "pdg_device_info")
        _checked_device = True
    return L


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())
