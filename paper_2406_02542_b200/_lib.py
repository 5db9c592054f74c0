"""ctypes binding of libloki_b200.so (include/loki_b200.h).

The library is loaded lazily on the first compute call.  There is NO CPU
fallback: if the shared library is missing, or the device is not an sm_100
part, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOKI_LIB_PATH") or os.path.join(PKG_DIR, "libloki_b200.so")  # override: A/B tuning only

LOKI_OK = 0
LOKI_ERR_SHAPE = 1
LOKI_ERR_BUDGET = 2
LOKI_ERR_INDEX = 3
LOKI_ERR_DOMAIN = 4
LOKI_ERR_CUDA = 5
LOKI_ERR_UNSUPPORTED = 6

DTYPE_F32 = 0
DTYPE_BF16 = 1
DTYPE_F64 = 2

ROPE_NONE = 0
ROPE_ROTATE_THEN_PROJECT = 1
ROPE_PROJECT_THEN_ROTATE = 2

SELECT_TOPK = 0
SELECT_ALL = 1
SELECT_INDICES = 2
SELECT_NONE = 3
SELECT_TOPK_SHARED = 4  # opt-in GQA: one selection per KV group on the summed group query

# every symbol include/loki_b200.h declares (checked by tests/test_host.py)
EXPORTED = (
    "loki_last_error", "loki_abi_version", "loki_device_check", "loki_decode",
    "loki_decode_workspace_bytes", "loki_decode_plan", "loki_decode_phase", "loki_append_kv",
    "loki_gathered_scores", "loki_weighted_sum", "loki_weighted_sum_workspace",
    "loki_softmax_rows", "loki_rope", "loki_index_status", "loki_set_phase_trace", "loki_project_rows",
)


class KvGeom(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int32), ("Hq", ctypes.c_int32), ("Hkv", ctypes.c_int32),
        ("D", ctypes.c_int32), ("S_cap", ctypes.c_int32), ("dtype", ctypes.c_int32),
        ("stride_b", ctypes.c_int64), ("stride_h", ctypes.c_int64), ("stride_s", ctypes.c_int64),
    ]


class DecodeArgs(ctypes.Structure):
    _fields_ = [
        ("q_hat", ctypes.c_void_p), ("K", ctypes.c_void_p), ("V", ctypes.c_void_p),
        ("g", KvGeom), ("lens", ctypes.c_void_p), ("S_max", ctypes.c_int32),
        ("d", ctypes.c_int32), ("k_f", ctypes.c_double), ("k_fixed", ctypes.c_int32),
        ("select_mode", ctypes.c_int32), ("ext_scores", ctypes.c_void_p),
        ("ext_idx", ctypes.c_void_p), ("idx_stride", ctypes.c_int64),
        ("out", ctypes.c_void_p), ("idx_out", ctypes.c_void_p), ("approx_out", ctypes.c_void_p),
        ("weights_out", ctypes.c_void_p), ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t), ("cluster_override", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SIGS = {
    "loki_last_error": (ctypes.c_char_p, []),
    "loki_abi_version": (_I32, []),
    "loki_device_check": (_I32, [_I32]),
    "loki_decode": (_I32, [ctypes.POINTER(DecodeArgs), _P]),
    "loki_decode_phase": (_I32, [ctypes.POINTER(DecodeArgs), _I32, _P]),
    "loki_decode_workspace_bytes": (_I32, [ctypes.POINTER(DecodeArgs), ctypes.POINTER(ctypes.c_size_t)]),
    "loki_decode_plan": (_I32, [ctypes.POINTER(DecodeArgs), ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                                ctypes.POINTER(ctypes.c_size_t)]),
    "loki_append_kv": (_I32, [_P, _P, _P, _P, _I64, _P, _P, _I32, _P, _P, KvGeom, _P, _P, _P]),
    "loki_gathered_scores": (_I32, [_P, _I32, _P, _I64, _I32, _I32, _P, _I32, _P, _P]),
    "loki_weighted_sum": (_I32, [_P, _P, _I64, _I32, _I32, _P, _I32, _P, _P, ctypes.c_size_t, _P]),
    "loki_weighted_sum_workspace": (ctypes.c_size_t, [_I32, _I32]),
    "loki_softmax_rows": (_I32, [_P, _I64, _I32, _I64, _P, _P]),
    "loki_rope": (_I32, [_P, _P, _I32, _I64, _I32, _P, _P, _P]),
    "loki_index_status": (_I32, [_P, _I32, _I64, _P, _P]),
    "loki_set_phase_trace": (_I32, [_P, _I32]),
    "loki_project_rows": (_I32, [_P, _I32, _P, _P, _P, _I32, _P, _I32, _I32, _I32, _I32, _I32, _P]),
}

_lock = threading.Lock()
_lib = None
_checked_devices = set()


class LibraryMissing(errors.LokiError, ImportError):
    """libloki_b200.so is not built (run __graft_entry__.build())."""


def load(path: str = LIB_PATH):
    """Load and type the shared library (idempotent)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise LibraryMissing(
                    f"{path} not found: the Loki CUDA extension is not built "
                    "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


_ERRMAP = {
    LOKI_ERR_SHAPE: errors.ShapeError,
    LOKI_ERR_BUDGET: errors.BudgetError,
    LOKI_ERR_INDEX: IndexError,
    LOKI_ERR_DOMAIN: errors.DomainError,
    LOKI_ERR_CUDA: errors.LokiCudaError,
    LOKI_ERR_UNSUPPORTED: errors.UnsupportedShapeError,
}


def check(status: int) -> None:
    if status != LOKI_OK:
        msg = load().loki_last_error().decode("utf-8", "replace")
        raise _ERRMAP.get(status, errors.LokiError)(msg)


def lib_for(device) -> ctypes.CDLL:
    """The library, after checking once that `device` is an sm_100 GPU."""
    lib = load()
    idx = device.index if device.index is not None else 0
    if idx not in _checked_devices:
        check(lib.loki_device_check(idx))
        _checked_devices.add(idx)
    return lib


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
