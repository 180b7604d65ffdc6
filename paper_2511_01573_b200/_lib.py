"""ctypes binding of libhcub_b200.so (include/hcub_b200.h).

The library is the only compute path: if it is missing or cannot find a
CUDA device, calls raise - there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HCUB_B200_LIB", os.path.join(HERE, "libhcub_b200.so"))
MAX_DIM = 13

HCUB_OK, HCUB_E_DIM, HCUB_E_ARG, HCUB_E_CUDA, HCUB_E_PROTOCOL, HCUB_E_OOM, HCUB_E_CAPACITY, HCUB_E_ABORTED = range(8)
KIND = {"f1": 1, "f2": 2, "f3": 3, "f4": 4, "f5": 5, "f6": 6, "f7": 7, "product_peak": 8}
REASONS = ("tolerance", "max_iterations", "max_regions", "width_guard_exhausted")


class hcub_integrand(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32), ("a", C.c_double), ("center", C.c_double * MAX_DIM)]


class hcub_rule(C.Structure):
    _fields_ = [("d", C.c_int32), ("node_count", C.c_int32),
                ("lam2", C.c_double), ("lam3", C.c_double), ("lam4", C.c_double), ("lam5", C.c_double),
                ("w", C.c_double * 5), ("we", C.c_double * 5),
                ("fourth_diff_ratio", C.c_double), ("null_center_weight", C.c_double),
                ("null_axis_weight", C.c_double),
                ("kind", C.c_int32), ("has_axis_pairs", C.c_int32), ("center_index", C.c_int32),
                ("axis_pairs", (C.c_int32 * 4) * MAX_DIM), ("K", C.c_int64),
                ("points", C.POINTER(C.c_double)), ("weights", C.POINTER(C.c_double)),
                ("embedded_weights", C.POINTER(C.c_double))]


class hcub_driver_cfg(C.Structure):
    _fields_ = [("tau_rel", C.c_double), ("abs_floor", C.c_double), ("min_width_ulp_factor", C.c_double),
                ("safety", C.c_double), ("max_iterations", C.c_int64), ("max_regions", C.c_int64)]


class hcub_result(C.Structure):
    _fields_ = [("integral", C.c_double), ("error", C.c_double), ("converged", C.c_int32),
                ("termination_reason", C.c_int32), ("iterations", C.c_int64), ("total_f_evals", C.c_int64),
                ("peak_regions", C.c_int64), ("capacity_limited", C.c_int32), ("pad", C.c_int32),
                ("device_ms", C.c_double), ("k1_ms", C.c_double), ("k2_ms", C.c_double), ("k3_ms", C.c_double),
                ("k1_launches", C.c_int64), ("launches", C.c_int64)]


class hcub_classify_out(C.Structure):
    _fields_ = [("n_split", C.c_int64), ("n_finalized", C.c_int64), ("width_guard_hits", C.c_int64),
                ("finalized_integral", C.c_double), ("finalized_error", C.c_double),
                ("children_integral", C.c_double), ("children_error", C.c_double),
                ("split_done", C.c_int32), ("pad", C.c_int32)]


TRACE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64)

_P = C.POINTER
_D = _P(C.c_double)
_I64 = _P(C.c_int64)
_I32 = _P(C.c_int32)
_W = C.c_void_p

# name -> (restype, argtypes); every symbol include/hcub_b200.h declares
SIGNATURES = {
    "hcub_abi_version": (C.c_int, []),
    "hcub_last_error": (C.c_char_p, []),
    "hcub_device_count": (C.c_int, [_I32]),
    "hcub_set_k1_lanes": (C.c_int, [C.c_int]),
    "hcub_apply_rule_batch": (C.c_int, [C.c_int, _P(hcub_rule), _P(hcub_integrand), _D, _D, C.c_int64, _D, _D, _D,
                                        _I64, _I64]),
    "hcub_eval_points": (C.c_int, [C.c_int, _P(hcub_integrand), _D, C.c_int64, _D]),
    "hcub_exact_sum": (C.c_int, [C.c_int, _D, C.c_int64, C.c_double, _D]),
    "hcub_integrate": (C.c_int, [C.c_int, _P(hcub_rule), _P(hcub_integrand), _D, _D, _D, _D, C.c_int64,
                                 _P(hcub_driver_cfg), C.c_int64, TRACE_FN, C.c_void_p, _P(hcub_result)]),
    "hcub_worker_create": (C.c_int, [C.c_int, _P(hcub_rule), _P(hcub_integrand), _D, _D, C.c_int64, _P(_W)]),
    "hcub_worker_destroy": (None, [_W]),
    "hcub_worker_size": (C.c_int, [_W, _I64, _I64]),
    "hcub_worker_append": (C.c_int, [_W, _D, _D, _D, _D, C.c_int64, C.c_int]),
    "hcub_worker_read": (C.c_int, [_W, _D, _D, _D, _D, _I64]),
    "hcub_worker_set_carry": (C.c_int, [_W, C.c_double, C.c_double]),
    "hcub_worker_get_carry": (C.c_int, [_W, _D, _D]),
    "hcub_worker_evaluate": (C.c_int, [_W, _D, _D, _I64]),
    "hcub_worker_classify": (C.c_int, [_W, C.c_double, _P(hcub_driver_cfg), C.c_int, _P(hcub_classify_out)]),
    "hcub_worker_reserve": (C.c_int, [_W, C.c_int64, C.POINTER(C.c_int32)]),
    "hcub_worker_take_top": (C.c_int, [_W, C.c_int64, _D, _D, _D, _D, C.c_int, _I64]),
    "hcub_worker_exact_partial": (C.c_int, [_W, C.c_int, _I64, _I32]),
    "hcub_worker_timings": (C.c_int, [_W, _D, _D, _D, _I64, _I64]),
    "hcub_worker_evaluate_tail": (C.c_int, [_W, C.c_int64, _I64]),
    "hcub_worker_evaluate_begin": (C.c_int, [_W]),
    "hcub_worker_evaluate_end": (C.c_int, [_W, _D, _D, _I64]),
    "hcub_worker_evaluate_end_async": (C.c_int, [_W, _I64]),
    "hcub_worker_stream": (C.c_int, [_W, _P(C.c_void_p)]),
    "hcub_worker_record_partials": (C.c_int, [_W, C.c_void_p]),
    "hcub_worker_classify_launch": (C.c_int, [_W, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                              _P(hcub_driver_cfg)]),
    "hcub_worker_classify_commit": (C.c_int, [_W, C.c_double, _P(hcub_driver_cfg), _P(hcub_classify_out)]),
    "hcub_worker_classify_discard": (C.c_int, [_W]),
    "hcub_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "hcub_comm_init": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, _P(C.c_void_p)]),
    "hcub_comm_destroy": (None, [C.c_void_p]),
    "hcub_worker_exchange_records": (C.c_int, [_W, C.c_void_p, _D, C.c_int, C.c_int, C.c_int, _P(hcub_driver_cfg),
                                               _D]),
    "hcub_trim": (C.c_int, [C.c_int]),
}

_lib = None
_lock = threading.Lock()


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load (once) and return the CDLL; raises LibraryMissing if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissing(
                    f"{LIB_PATH} not built - run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(no CPU fallback exists)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            if L.hcub_abi_version() != 2:
                raise LibraryMissing("ABI version mismatch")
            _lib = L
    return _lib


def check(rc):
    """Map an HCUB_E_* code onto the reference's exception types."""
    if rc == HCUB_OK:
        return
    msg = lib().hcub_last_error().decode(errors="replace")
    if rc == HCUB_E_DIM:
        from .rules import UnsupportedDimensionError
        raise UnsupportedDimensionError(msg)
    if rc in (HCUB_E_ARG,):
        raise ValueError(msg)
    if rc == HCUB_E_PROTOCOL:
        from .distributed import ProtocolError
        raise ProtocolError(msg)
    if rc == HCUB_E_OOM:
        raise MemoryError(msg)
    if rc == HCUB_E_CAPACITY:
        raise OverflowError(msg)
    if rc == HCUB_E_ABORTED:
        raise RuntimeError(f"hcub: {msg}")
    raise RuntimeError(f"hcub CUDA error: {msg}")


def dptr(a):
    """double* of a C-contiguous float64 ndarray (or None)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def iptr(a):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_I64)


_device = None


def current_device():
    """CUDA device the library targets: set_device(), else LOCAL_RANK, else 0."""
    if _device is not None:
        return _device
    return int(os.environ.get("HCUB_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def set_device(index: int) -> None:
    global _device
    _device = int(index)


def set_k1_lanes(log2_lanes: int) -> None:
    """Force the K1 lanes-per-region choice (-1 = automatic)."""
    check(lib().hcub_set_k1_lanes(int(log2_lanes)))


def device_count() -> int:
    n = C.c_int32(0)
    check(lib().hcub_device_count(C.byref(n)))
    return int(n.value)
