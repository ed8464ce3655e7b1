"""Python binding of the OFDM output stage (include/bf_ofdm.h): beamforming followed by the
per-antenna OFDM IFFT with cyclic prefix.

y[m][a] = CP(scale * IDFT_unnormalised(map(R[m nb : m nb + nb][a]))), R = W x S
(PAPER.md:84-86 for R; the pipeline stages of PAPER.md:41, 49 and the 2048-point
transforms of PAPER.md:67-71; readings O1-O5 in DESIGN.md §2).  Argument marshalling
only: the product runs in the bf plan's kernels, the IFFT in libbf.so's
bfofdm::ofdm_ifft_kernel.
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import check, lib
from .plan import Plan, _ptr, _stream_handle

OFDM_N = 2048


def _sig(L):
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    P = ctypes.POINTER
    for name, args in {
        "bf_ofdm_plan_create": [vp, i32, i32, i32, ctypes.c_float, P(vp)],
        "bf_ofdm_apply": [vp, vp, vp, i64, vp, vp],
        "bf_ofdm_ifft": [vp, vp, i64, vp, vp],
        "bf_ofdm_plan_set_chunk": [vp, i64],
        "bf_ofdm_plan_set_output": [vp, i32, i32],
        "bf_ofdm_destroy": [vp],
        "bf_ofdm_plan_set_profiling": [vp, i32],
        "bf_ofdm_plan_kernel_time": [vp, P(ctypes.c_double), P(i64)],
        "bf_ofdm_plan_launch_count": [vp, P(i64)],
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


class OfdmPlan:
    """OFDM output of a bf Plan (interleaved layout): nb blocks per symbol, n-point IFFT,
    cp-sample cyclic prefix, output scale."""

    def __init__(self, plan: Plan, nb: int, n: int = OFDM_N, cp: int = 0, scale: float = 1.0):
        self.plan, self.nb, self.n, self.cp = plan, int(nb), int(n), int(cp)
        self.scale = float(torch.tensor(scale, dtype=torch.float32))
        self._h = ctypes.c_void_p()
        check(_lib().bf_ofdm_plan_create(plan._h, self.n, self.cp, self.nb, self.scale,
                                         ctypes.byref(self._h)))
        self.device = plan.device
        self.out16, self.out_exp = False, 12

    def y_shape(self, n_sym: int):
        if self.out16:     # int16 (re, im) pairs
            return (n_sym, self.plan.n_ant, self.cp + self.n, 2)
        return (n_sym, self.plan.n_ant, self.cp + self.n)

    @property
    def y_dtype(self):
        return torch.int16 if self.out16 else torch.complex64

    def set_output(self, fmt: str = "f32", exponent: int = 12) -> None:
        """bf_ofdm_plan_set_output: "f32" (complex64 samples) or "i16" (int16 (re, im) pairs,
        sat(rne(y 2^exponent)))."""
        code = {"f32": 0, "i16": 1}[fmt]
        check(_lib().bf_ofdm_plan_set_output(self._h, code, int(exponent)))
        self.out16, self.out_exp = code == 1, int(exponent)

    def _check(self, t, name, shape, dtype):
        if t.dtype != dtype or tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} must be {dtype} {tuple(shape)}, got {t.dtype} {tuple(t.shape)}")
        if not t.is_contiguous() or t.device != self.device:
            raise ValueError(f"{name} must be contiguous on {self.device}")

    def _out(self, n_sym, out):
        if out is None:
            out = torch.empty(self.y_shape(n_sym), dtype=self.y_dtype, device=self.device)
        self._check(out, "out", self.y_shape(n_sym), self.y_dtype)
        return out

    def apply(self, S: torch.Tensor, tags: torch.Tensor | None = None,
              out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """bf_ofdm_apply: S complex64 [n_sym nb][f][60], tags int32 [n_sym nb] or None."""
        if S.dim() != 3 or S.shape[0] % self.nb:
            raise ValueError("S must be [n_sym * nb][f][b]")
        n_sym = S.shape[0] // self.nb
        self._check(S, "S", self.plan.s_shape(S.shape[0]), torch.complex64)
        if tags is not None:
            self._check(tags, "tags", (S.shape[0],), torch.int32)
        out = self._out(n_sym, out)
        check(_lib().bf_ofdm_apply(self._h, _ptr(S), _ptr(tags), n_sym, _ptr(out),
                                   _stream_handle(stream)))
        return out

    def ifft(self, R: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """bf_ofdm_ifft: the IFFT + cyclic-prefix stage from R complex64 [n_sym nb][64][60]."""
        if R.dim() != 3 or R.shape[0] % self.nb:
            raise ValueError("R must be [n_sym * nb][n_ant][b]")
        n_sym = R.shape[0] // self.nb
        self._check(R, "R", (R.shape[0], self.plan.n_ant, self.plan.b), torch.complex64)
        out = self._out(n_sym, out)
        check(_lib().bf_ofdm_ifft(self._h, _ptr(R), n_sym, _ptr(out), _stream_handle(stream)))
        return out

    def set_chunk(self, symbols: int) -> None:
        check(_lib().bf_ofdm_plan_set_chunk(self._h, int(symbols)))

    def set_profiling(self, enable: bool = True) -> None:
        check(_lib().bf_ofdm_plan_set_profiling(self._h, int(bool(enable))))

    def kernel_time(self):
        ms, nl = ctypes.c_double(), ctypes.c_int64()
        check(_lib().bf_ofdm_plan_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(nl)))
        return ms.value, nl.value

    def launch_count(self) -> int:
        c = ctypes.c_int64()
        check(_lib().bf_ofdm_plan_launch_count(self._h, ctypes.byref(c)))
        return c.value

    def close(self) -> None:
        if self._h:
            check(_lib().bf_ofdm_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ofdm_plan_create_status(plan: Plan, nb: int, n: int = OFDM_N, cp: int = 0,
                            scale: float = 1.0) -> int:
    h = ctypes.c_void_p()
    s = _lib().bf_ofdm_plan_create(plan._h, int(n), int(cp), int(nb), float(scale), ctypes.byref(h))
    if s == 0:
        _lib().bf_ofdm_destroy(h)
    return s
