"""ctypes binding of the in-tree C ABI library lib/libqdot_b200.so.

The library is the only compute path.  If it is missing the import of the
package still works (so CPU-side helpers and tests can run), but every
compute call raises immediately -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import build as _build

KEYS = 4195
KEY_OFFSET = 2148

QDOT_OK, QDOT_ERR_NONFINITE, QDOT_ERR_OVERFLOW, QDOT_ERR_ARG, QDOT_ERR_CUDA, QDOT_ERR_EPS = range(6)
STRATEGY_EXACT, STRATEGY_RANGED, STRATEGY_SPLIT = range(3)


class QdotConfig(ctypes.Structure):
    _fields_ = [("epsilon", ctypes.c_double), ("split", ctypes.c_int32), ("input_mu", ctypes.c_int32),
                ("strategy", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("strategy_param", ctypes.c_int64)]


class QdotBin(ctypes.Structure):
    _fields_ = [("lower", ctypes.c_int64), ("upper", ctypes.c_int64), ("cardinality", ctypes.c_int64),
                ("score", ctypes.c_int64), ("precision", ctypes.c_int32), ("first_key", ctypes.c_int32),
                ("last_key", ctypes.c_int32), ("flags", ctypes.c_int32), ("value", ctypes.c_double)]


class QdotResult(ctypes.Structure):
    _fields_ = [("value", ctypes.c_double), ("eps_eff", ctypes.c_double), ("n", ctypes.c_int64),
                ("nnz", ctypes.c_int64), ("zero_count", ctypes.c_int64), ("counts", ctypes.c_int64 * 4),
                ("status", ctypes.c_int32), ("n_bins", ctypes.c_int32), ("e_min", ctypes.c_int32),
                ("e_max", ctypes.c_int32), ("early_terminated", ctypes.c_int32),
                ("pass2_needed", ctypes.c_int32), ("half_order_sensitive", ctypes.c_int32),
                ("select_ns", ctypes.c_int32), ("compute_ns", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]


class QdotExactResult(ctypes.Structure):
    _fields_ = [("value", ctypes.c_double), ("plain", ctypes.c_double), ("nonfinite", ctypes.c_int64),
                ("status", ctypes.c_int32), ("flexp_e", ctypes.c_int32), ("is_zero", ctypes.c_int32),
                ("fallback", ctypes.c_int32), ("reserved", ctypes.c_int32 * 4)]


class QdotWsLayout(ctypes.Structure):
    _fields_ = [("total_bytes", ctypes.c_int64), ("a_offset", ctypes.c_int64), ("a_len", ctypes.c_int64),
                ("b_offset", ctypes.c_int64), ("b_len", ctypes.c_int64),
                ("result_offset", ctypes.c_int64), ("result_bytes", ctypes.c_int64)]


assert ctypes.sizeof(QdotBin) == 56

# the same header as a numpy record, for bulk parsing of device-recorded iterations
RESULT_DTYPE = np.dtype({"names": ["value", "eps_eff", "n", "nnz", "zero_count", "counts", "status", "n_bins"],
                         "formats": ["<f8", "<f8", "<i8", "<i8", "<i8", ("<i8", (4,)), "<i4", "<i4"],
                         "offsets": [QdotResult.value.offset, QdotResult.eps_eff.offset, QdotResult.n.offset,
                          QdotResult.nnz.offset, QdotResult.zero_count.offset, QdotResult.counts.offset,
                          QdotResult.status.offset, QdotResult.n_bins.offset],
                         "itemsize": ctypes.sizeof(QdotResult)})

_lock = threading.Lock()
_lib = None

# every exported symbol of include/qdot_b200.h: (name, restype, argtypes)
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
SIGNATURES = {
    "qdot_b200_version": (_I, []),
    "qdot_b200_status_string": (ctypes.c_char_p, [_I]),
    "qdot_b200_last_error": (ctypes.c_char_p, []),
    "qdot_b200_workspace_bytes": (ctypes.c_size_t, []),
    "qdot_b200_workspace_layout": (_I, [ctypes.POINTER(QdotWsLayout)]),
    "qdot_b200_device_info": (_I, [ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "qdot_b200_begin": (_I, [_P, _P]),
    "qdot_b200_enqueue": (_I, [_P, _P, _I64, _I, ctypes.POINTER(QdotConfig), _P, _P]),
    "qdot_b200_enqueue_zeroed": (_I, [_P, _P, _I64, _I, ctypes.POINTER(QdotConfig), _P, _P]),
    "qdot_b200_small": (_I, [_P, _P, _I64, _I, ctypes.POINTER(QdotConfig), _P, _P]),
    "qdot_b200_small_max": (_I64, []),
    "qdot_b200_pass1": (_I, [_P, _P, _I64, _I, ctypes.POINTER(QdotConfig), _I64, _P, _P]),
    "qdot_b200_score": (_I, [_P, _I64, ctypes.POINTER(QdotConfig), _P]),
    "qdot_b200_score_finalize": (_I, [_P, _I64, ctypes.POINTER(QdotConfig), _P]),
    "qdot_b200_pass2": (_I, [_P, _P, _I64, _I, _P, _P]),
    "qdot_b200_pass2_finalize": (_I, [_P, _P, _I64, _I, _P, _P]),
    "qdot_b200_finalize": (_I, [_P, _P]),
    "qdot_b200_fetch": (_I, [_P, ctypes.POINTER(QdotResult), ctypes.POINTER(QdotBin), ctypes.c_int32, _P]),
    "qdot_b200_dot": (_I, [_P, _P, _I64, _I, ctypes.POINTER(QdotConfig), _P, ctypes.POINTER(QdotResult),
                           ctypes.POINTER(QdotBin), ctypes.c_int32, _P]),
    "qdot_b200_dot_host": (_I, [_P, _P, _I64, _I, ctypes.POINTER(QdotConfig), ctypes.POINTER(QdotResult),
                                ctypes.POINTER(QdotBin), ctypes.c_int32]),
    "qdot_b200_bin_ids": (_I, [_P, _P, _I64, _I, _P, _P, _P]),
    "qdot_b200_batched": (_I, [_P, _P, _I64, _I64, _I64, _I, ctypes.POINTER(QdotConfig), _P, _P, _P, _P]),
    "qdot_b200_batched_bins": (_I, [_P, _P, _I64, _I64, _I64, _I, ctypes.POINTER(QdotConfig), _P, _P, _P, _P, _P]),
    "qdot_b200_ldexp_rn": (ctypes.c_double, [ctypes.c_double, _I64, ctypes.POINTER(_I)]),
    "qdot_b200_bound_sums": (_I, [_P, ctypes.c_int32, _I64, _P]),
    "qdot_b200_bound_sums2": (_I, [_P, ctypes.c_int32, _I64, _I64, _P]),
    "qdot_b200_csr_spmv": (_I, [_I64, _P, _P, _I, _P, _P, _P, _P]),
    "qdot_b200_read_probe": (_I, [_P, _I64, _P, _P]),
    "qdot_b200_sell_spmv": (_I, [_I64, _P, _P, _P, _P, _P, _P, _P]),
    "qdot_b200_vec_update_dev": (_I, [_I64, _I, _P, _P, _P, _P, _P]),
    "qdot_b200_solver_scalar": (_I, [_I, _P, _P, _P]),
    "qdot_b200_publish_iter": (_I, [_P, _P, _P, _P, _P, _P]),
    "qdot_b200_loop_create": (_I, [_P, ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_ulonglong)]),
    "qdot_b200_loop_finish": (_I, [_P, _P]),
    "qdot_b200_loop_launch": (_I, [_P, _P]),
    "qdot_b200_loop_destroy": (None, [_P]),
    "qdot_b200_acg_check": (_I, [_P, _P, _P, _P, _P, ctypes.c_ulonglong, _P]),
    "qdot_b200_cg_xr": (_I, [_I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "qdot_b200_cg_p_check": (_I, [_I64, _P, _P, _P, _P, _P, _P, _P, ctypes.c_ulonglong, _P, _P]),
    "qdot_b200_pm_div": (_I, [_I64, _P, _P, _P, _P, _P]),
    "qdot_b200_pm_check": (_I, [_I64, _P, _P, _P, _P, _P, _P, _P, ctypes.c_ulonglong, _P]),
    "qdot_b200_exact_workspace_bytes": (ctypes.c_size_t, []),
    "qdot_b200_exact_region_words": (_I64, []),
    "qdot_b200_exact_begin": (_I, [_P, _P]),
    "qdot_b200_exact_accumulate": (_I, [_P, _P, _I64, _I, _P, _P]),
    "qdot_b200_exact_plain": (_I, [_P, _P, _I64, _I, _P, _P]),
    "qdot_b200_exact_finalize": (_I, [_P, _P]),
    "qdot_b200_exact_fetch": (_I, [_P, ctypes.POINTER(QdotExactResult), _P]),
    "qdot_b200_vec_update": (_I, [_I64, _I, _P, ctypes.c_double, _P, _P, _P]),
    "qdot_b200_pass1_host": (_I, [_P, _P, _I64, _I, ctypes.POINTER(QdotConfig), _I64, _P, _P, _P, _P]),
    "qdot_b200_host_copy_threads": (_I, []),
    "qdot_b200_generate": (_I, [_I, ctypes.c_double, ctypes.c_uint64, _I64, _I64, _P, _P, _P]),
    "qdot_b200_order_scratch_bytes": (ctypes.c_size_t, [_I64, ctypes.c_int32]),
    "qdot_b200_bin_order": (_I, [_P, _P, _I64, _I, _P, ctypes.c_int32, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "qdot_b200_half_ordered": (_I, [_P, _P, _I64, _I, _P, ctypes.c_int32, _P, _I64, _P, _P, ctypes.c_size_t,
                                    _I, _P]),
}


class ExtensionMissing(RuntimeError):
    pass


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load lib/libqdot_b200.so (building it with nvcc if absent and possible)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        if not os.path.exists(path) and build_if_missing:
            try:
                _build.build()
            except Exception as exc:  # pragma: no cover - depends on toolchain
                raise ExtensionMissing(f"libqdot_b200.so missing and build failed: {exc}") from exc
        if not os.path.exists(path):
            raise ExtensionMissing(f"CUDA extension not built: {path} (run python -m paper_2105_00115_b200.build)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int, lib=None) -> None:
    """Map a qdot_status to the reference's exception types."""
    if status == QDOT_OK:
        return
    if status == QDOT_ERR_NONFINITE:
        raise ValueError("inputs must be finite")                       # floatbits.py:70-71
    if status == QDOT_ERR_OVERFLOW:
        raise OverflowError("rounded bin product overflowed its format")  # emulate.py:147-148
    if status == QDOT_ERR_EPS:
        raise ValueError("floor_log2 needs a positive finite value")    # scoring.py:84-85
    if status == QDOT_ERR_ARG:
        raise ValueError("invalid qdot argument")
    msg = ""
    if lib is not None:
        msg = (lib.qdot_b200_last_error() or b"").decode()
    raise RuntimeError(f"qdot CUDA failure: {msg or 'CUDA error'}")


def layout() -> QdotWsLayout:
    lay = QdotWsLayout()
    check(load().qdot_b200_workspace_layout(ctypes.byref(lay)))
    return lay
