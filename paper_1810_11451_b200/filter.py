"""Python binding of the filter stage (include/bf_filter.h): y = IFFT(H . FFT(s)).

PAPER.md:67-71: "The filter algorithm computes IFFT(MULT(FFT(s))) where MULT is
the pointwise multiplication by the FFT of the filter sequence and FFT sizes are
all 2048."  Argument marshalling only; the FFTs and the product run in
libbf.so's fused sm_100a kernel.
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import check, lib
from .plan import _ptr, _stream_handle

FILTER_N = 2048


def _sig(L):
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    P = ctypes.POINTER
    for name, args in {
        "bff_plan_create": [i32, P(vp)],
        "bff_set_taps": [vp, vp, vp],
        "bff_apply": [vp, vp, vp, i64, vp],
        "bff_fft": [vp, vp, vp, i64, vp],
        "bff_destroy": [vp],
        "bff_plan_set_profiling": [vp, i32],
        "bff_plan_kernel_time": [vp, P(ctypes.c_double), P(i64)],
        "bff_plan_launch_count": [vp, P(i64)],
    }.items():
        fn = getattr(L, name)
        fn.restype = i32
        fn.argtypes = args
    return L


_L = None


def _lib():
    global _L
    if _L is None:
        _L = _sig(lib())
    return _L


class FilterPlan:
    """Filter of 2048-sample complex signals by a fixed filter sequence h."""

    def __init__(self, n: int = FILTER_N):
        self.n = int(n)
        self._h = ctypes.c_void_p()
        check(_lib().bff_plan_create(self.n, ctypes.byref(self._h)))
        self.device = torch.device("cuda", torch.cuda.current_device())

    def _check(self, t: torch.Tensor, name: str):
        if t.dtype != torch.complex64 or t.dim() != 2 or t.shape[1] != self.n:
            raise ValueError(f"{name} must be complex64 [n_signals][{self.n}]")
        if not t.is_contiguous() or t.device != self.device:
            raise ValueError(f"{name} must be contiguous on {self.device}")

    def set_taps(self, h: torch.Tensor, stream=None) -> "FilterPlan":
        """bff_set_taps: h complex64 [n] on the device (the filter sequence)."""
        h = h.reshape(1, -1)
        self._check(h, "h")
        check(_lib().bff_set_taps(self._h, _ptr(h), _stream_handle(stream)))
        self._h_ref = h
        return self

    def apply(self, s: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """bff_apply: y = IFFT(H . FFT(s)); out may be s itself (in place)."""
        self._check(s, "s")
        if out is None:
            out = torch.empty_like(s)
        self._check(out, "out")
        check(_lib().bff_apply(self._h, _ptr(s), _ptr(out), s.shape[0], _stream_handle(stream)))
        return out

    def fft(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """bff_fft: unnormalised forward DFT of each signal."""
        self._check(x, "x")
        if out is None:
            out = torch.empty_like(x)
        check(_lib().bff_fft(self._h, _ptr(x), _ptr(out), x.shape[0], _stream_handle(stream)))
        return out

    def set_profiling(self, enable: bool = True) -> None:
        check(_lib().bff_plan_set_profiling(self._h, int(bool(enable))))

    def kernel_time(self):
        ms, nl = ctypes.c_double(), ctypes.c_int64()
        check(_lib().bff_plan_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(nl)))
        return ms.value, nl.value

    def launch_count(self) -> int:
        c = ctypes.c_int64()
        check(_lib().bff_plan_launch_count(self._h, ctypes.byref(c)))
        return c.value

    def close(self) -> None:
        if self._h:
            check(_lib().bff_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def filter_plan_create_status(n: int) -> int:
    h = ctypes.c_void_p()
    s = _lib().bff_plan_create(int(n), ctypes.byref(h))
    if s == 0:
        _lib().bff_destroy(h)
    return s
