"""ctypes declarations of libbf.so (include/bf.h).  Argument marshalling only.

The library is loaded from this package directory.  There is no fallback: if
libbf.so is missing or fails to load, importing the binding raises.
"""
from __future__ import annotations

import ctypes
import enum
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbf.so")

# every symbol include/bf.h declares (tests check the .so exports all of them)
EXPORTS = ("bf_plan_create", "bf_set_precoders", "bf_apply", "bf_apply_host", "bf_route",
           "bf_apply_routed", "bf_apply_batch",
           "bf_destroy", "bf_plan_set_profiling", "bf_plan_kernel_time",
           "bf_plan_launch_count", "bf_plan_set_host_chunk", "bf_plan_kernel_config",
           "bf_plan_set_variant", "bf_plan_get_variant", "bf_plan_set_sm_share",
           "bf_plan_set_output_exponent",
           "bf_server_create", "bf_server_start", "bf_server_submit", "bf_server_wait",
           "bf_server_slot_time", "bf_server_trace", "bf_server_stop", "bf_server_destroy",
           "bff_plan_create", "bff_set_taps", "bff_apply", "bff_fft", "bff_destroy",
           "bff_plan_set_profiling", "bff_plan_kernel_time", "bff_plan_launch_count",
           "bf_ofdm_plan_create", "bf_ofdm_apply", "bf_ofdm_ifft", "bf_ofdm_plan_set_chunk", "bf_ofdm_plan_set_output",
           "bf_ofdm_destroy", "bf_ofdm_plan_set_profiling", "bf_ofdm_plan_kernel_time",
           "bf_ofdm_plan_launch_count",
           "bf_status_string", "bf_last_error", "bf_version")


class Status(enum.IntEnum):
    OK = 0
    INVALID_VALUE = 1
    UNSUPPORTED = 2
    NO_PRECODERS = 3
    MISALIGNED = 4
    OUT_OF_MEMORY = 5
    CUDA = 6
    NO_DEVICE = 7


class Layout(enum.IntEnum):
    INTERLEAVED = 0
    PLANAR = 1
    INTERLEAVED_F16OUT = 2    # R as fp16 (re, im) pairs
    INTERLEAVED_I16OUT = 3    # R as int16 (re, im) fronthaul samples, x 2^e


class Variant(enum.IntEnum):
    AUTO = 0
    FFMA = 1
    TENSOR = 2


class BatchJob(ctypes.Structure):
    """bf_batch_job (include/bf.h)."""
    _fields_ = [("plan", ctypes.c_void_p), ("S_dev", ctypes.c_void_p),
                ("perm_dev", ctypes.c_void_p), ("offsets_dev", ctypes.c_void_p),
                ("R_dev", ctypes.c_void_p), ("n_blocks", ctypes.c_int64)]


class BfError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = Status(status)
        super().__init__(f"{self.status.name}: {detail}")


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c "
                          f"'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    P = ctypes.POINTER
    sig = {
        "bf_plan_create": (i32, [i32, i32, i32, i32, P(vp)]),
        "bf_set_precoders": (i32, [vp, vp, i32, vp]),
        "bf_apply": (i32, [vp, vp, vp, vp, i64, vp]),
        "bf_apply_host": (i32, [vp, vp, vp, vp, i64, vp]),
        "bf_route": (i32, [vp, vp, i64, vp, vp, vp]),
        "bf_apply_routed": (i32, [vp, vp, vp, vp, vp, i64, vp]),
        "bf_apply_batch": (i32, [P(BatchJob), i32, vp]),
        "bf_destroy": (i32, [vp]),
        "bf_plan_set_profiling": (i32, [vp, i32]),
        "bf_plan_kernel_time": (i32, [vp, P(ctypes.c_double), P(i64)]),
        "bf_plan_launch_count": (i32, [vp, P(i64)]),
        "bf_plan_set_host_chunk": (i32, [vp, i64]),
        "bf_plan_set_variant": (i32, [vp, i32]),
        "bf_plan_set_sm_share": (i32, [vp, i32]),
        "bf_plan_set_output_exponent": (i32, [vp, i32]),
        "bf_plan_get_variant": (i32, [vp, P(i32)]),
        "bf_plan_kernel_config": (i32, [vp, i64, P(i32), P(i32), P(i32), P(i32)]),
        "bf_server_create": (i32, [vp, P(vp)]),
        "bf_server_start": (i32, [vp, vp]),
        "bf_server_submit": (i32, [vp, vp, vp, i64, P(ctypes.c_uint64)]),
        "bf_server_wait": (i32, [vp, ctypes.c_uint64, ctypes.c_double]),
        "bf_server_slot_time": (i32, [vp, ctypes.c_uint64, P(ctypes.c_double)]),
        "bf_server_trace": (i32, [vp, P(ctypes.c_double), i32]),
        "bf_server_stop": (i32, [vp]),
        "bf_server_destroy": (i32, [vp]),
        "bf_status_string": (ctypes.c_char_p, [i32]),
        "bf_last_error": (ctypes.c_char_p, []),
        "bf_version": (i32, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status != 0:
        raise BfError(status, lib().bf_last_error().decode(errors="replace"))
