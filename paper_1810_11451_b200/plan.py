"""Python binding of the beamforming plan (same names as include/bf.h).

Argument marshalling only: shape / dtype / device checks, data_ptr() and the
CUDA stream handle are passed to libbf.so; every step of the computation runs
in the library's sm_100a kernels.  PyTorch supplies device memory and streams.

    plan = Plan(f=36)                       # bf_plan_create(64, 36, 60, INTERLEAVED)
    plan.set_precoders(W)                   # W: cuda complex64 [G][64][36]
    R = plan.apply(S, group_idx=tags)       # S: cuda complex64 [n][36][60] -> [n][64][60]
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import BatchJob, BfError, Layout, Status, Variant, check, lib

N_ANT = 64
N_RE = 60
MAX_F = 36


def _stream_handle(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    if isinstance(stream, torch.cuda.Stream):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(None if t is None else t.data_ptr())


class Plan:
    """A beamforming plan: n_ant x f precoders applied to f x b symbol blocks."""

    def __init__(self, f: int, n_ant: int = N_ANT, b: int = N_RE,
                 layout: Layout | str | int = Layout.INTERLEAVED,
                 variant: Variant | str | int = Variant.AUTO):
        if isinstance(layout, str):
            layout = Layout[layout.upper()]
        self.f, self.n_ant, self.b, self.layout = int(f), int(n_ant), int(b), Layout(layout)
        self.n_groups = 0
        self._h = ctypes.c_void_p()
        check(lib().bf_plan_create(self.n_ant, self.f, self.b, int(self.layout),
                                   ctypes.byref(self._h)))
        self.device = torch.device("cuda", torch.cuda.current_device())
        self._w_ref = None
        self.set_variant(variant)

    # -- shapes ---------------------------------------------------------------
    def s_shape(self, n: int):
        return (n, 2, self.f, self.b) if self.layout == Layout.PLANAR else (n, self.f, self.b)

    def r_shape(self, n: int):
        if self.layout == Layout.PLANAR:
            return (n, 2, self.n_ant, self.b)
        if self.layout in (Layout.INTERLEAVED_F16OUT, Layout.INTERLEAVED_I16OUT):
            return (n, self.n_ant, self.b, 2)
        return (n, self.n_ant, self.b)

    def w_shape(self, g: int):
        return (g, 2, self.n_ant, self.f) if self.layout == Layout.PLANAR else (g, self.n_ant, self.f)

    @property
    def dtype(self):
        """dtype of W and S."""
        return torch.float32 if self.layout == Layout.PLANAR else torch.complex64

    @property
    def r_dtype(self):
        """dtype of R (fp16 / int16 (re, im) pairs for the 16-bit output layouts)."""
        if self.layout == Layout.INTERLEAVED_F16OUT:
            return torch.float16
        if self.layout == Layout.INTERLEAVED_I16OUT:
            return torch.int16
        return self.dtype

    def _check(self, t: torch.Tensor, name: str, shape, device=True, dtype=None):
        dtype = self.dtype if dtype is None else dtype
        if t.dtype != dtype:
            raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if device and t.device != self.device:
            raise ValueError(f"{name} must be on {self.device}, got {t.device}")
        if not device and t.device.type != "cpu":
            raise ValueError(f"{name} must be a host tensor")

    # -- the calls of include/bf.h ------------------------------------------------
    def set_precoders(self, W: torch.Tensor, stream=None) -> "Plan":
        """bf_set_precoders: W [G][64][f] complex64 (interleaved) or [G][2][64][f] float32."""
        if W.dim() == (3 if self.layout == Layout.PLANAR else 2):
            W = W.unsqueeze(0)
        G = W.shape[0]
        self._check(W, "W", self.w_shape(G))
        check(lib().bf_set_precoders(self._h, _ptr(W), G, _stream_handle(stream)))
        self.n_groups = G
        self._w_ref = W          # keep alive until the relayout has run
        return self

    def apply(self, S: torch.Tensor, group_idx: torch.Tensor | None = None,
              out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """bf_apply on device tensors; returns R (allocated if out is None)."""
        n = S.shape[0]
        self._check(S, "S", self.s_shape(n))
        if out is None:
            out = torch.empty(self.r_shape(n), dtype=self.r_dtype, device=self.device)
        self._check(out, "out", self.r_shape(n), dtype=self.r_dtype)
        if group_idx is not None:
            if group_idx.dtype != torch.int32 or tuple(group_idx.shape) != (n,) \
                    or group_idx.device != self.device or not group_idx.is_contiguous():
                raise ValueError("group_idx must be a contiguous int32 [n] tensor on the plan device")
        check(lib().bf_apply(self._h, _ptr(S), _ptr(group_idx), _ptr(out), n,
                             _stream_handle(stream)))
        return out

    def apply_routed(self, S: torch.Tensor, perm: torch.Tensor | None,
                     offsets: torch.Tensor | None, out: torch.Tensor | None = None,
                     stream=None) -> torch.Tensor:
        """bf_apply_routed: apply to blocks routed by route() (perm, offsets)."""
        n = S.shape[0]
        self._check(S, "S", self.s_shape(n))
        if out is None:
            out = torch.empty(self.r_shape(n), dtype=self.r_dtype, device=self.device)
        self._check(out, "out", self.r_shape(n), dtype=self.r_dtype)
        check(lib().bf_apply_routed(self._h, _ptr(S), _ptr(perm), _ptr(offsets), _ptr(out), n,
                                    _stream_handle(stream)))
        return out

    def route_into(self, group_idx: torch.Tensor, perm: torch.Tensor, offsets: torch.Tensor,
                   stream=None):
        """bf_route into caller buffers (int32 [n] and int32 [n_groups + 2])."""
        check(lib().bf_route(self._h, _ptr(group_idx), group_idx.shape[0], _ptr(perm),
                             _ptr(offsets), _stream_handle(stream)))
        return perm, offsets

    def apply_host(self, S: torch.Tensor, group_idx: torch.Tensor | None, out: torch.Tensor,
                   stream=None) -> torch.Tensor:
        """bf_apply_host on host tensors (pinned for full speed)."""
        n = S.shape[0]
        self._check(S, "S", self.s_shape(n), device=False)
        self._check(out, "out", self.r_shape(n), device=False, dtype=self.r_dtype)
        if group_idx is not None and (group_idx.dtype != torch.int32 or
                                      tuple(group_idx.shape) != (n,) or group_idx.is_cuda):
            raise ValueError("group_idx must be a host int32 [n] tensor")
        check(lib().bf_apply_host(self._h, _ptr(S), _ptr(group_idx), _ptr(out), n,
                                  _stream_handle(stream)))
        return out

    def route(self, group_idx: torch.Tensor, stream=None):
        """bf_route: (perm int32 [n], offsets int32 [G + 2]) of the stable sort by tag."""
        n = group_idx.shape[0]
        perm = torch.empty(n, dtype=torch.int32, device=self.device)
        offsets = torch.empty(self.n_groups + 2, dtype=torch.int32, device=self.device)
        check(lib().bf_route(self._h, _ptr(group_idx), n, _ptr(perm), _ptr(offsets),
                             _stream_handle(stream)))
        return perm, offsets

    # -- instrumentation --------------------------------------------------------------
    def set_profiling(self, enable: bool = True) -> None:
        check(lib().bf_plan_set_profiling(self._h, int(bool(enable))))

    def kernel_time(self):
        """(summed ms, launches) of the beamforming kernel since the last call."""
        ms, nl = ctypes.c_double(), ctypes.c_int64()
        check(lib().bf_plan_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(nl)))
        return ms.value, nl.value

    def launch_count(self) -> int:
        c = ctypes.c_int64()
        check(lib().bf_plan_launch_count(self._h, ctypes.byref(c)))
        return c.value

    def set_variant(self, variant: Variant | str | int) -> None:
        """bf_plan_set_variant: AUTO (per-f table), FFMA or TENSOR."""
        if isinstance(variant, str):
            variant = Variant[variant.upper()]
        check(lib().bf_plan_set_variant(self._h, int(variant)))

    @property
    def variant(self) -> Variant:
        """The kernel variant applies of this plan run (AUTO resolved)."""
        v = ctypes.c_int()
        check(lib().bf_plan_get_variant(self._h, ctypes.byref(v)))
        return Variant(v.value)

    def set_output_exponent(self, e: int) -> None:
        """bf_plan_set_output_exponent: int16 output = sat(rne(R x 2^e))."""
        check(lib().bf_plan_set_output_exponent(self._h, int(e)))

    def set_sm_share(self, sms: int) -> None:
        """bf_plan_set_sm_share: spread later applies over `sms` SMs (0 = all)."""
        check(lib().bf_plan_set_sm_share(self._h, int(sms)))

    def set_host_chunk(self, blocks: int) -> None:
        check(lib().bf_plan_set_host_chunk(self._h, int(blocks)))

    def kernel_config(self, n_blocks: int) -> dict:
        g, b, s, c = (ctypes.c_int() for _ in range(4))
        check(lib().bf_plan_kernel_config(self._h, int(n_blocks), ctypes.byref(g), ctypes.byref(b),
                                          ctypes.byref(s), ctypes.byref(c)))
        return {"grid": g.value, "block": b.value, "smem_bytes": s.value, "ctas_per_sm": c.value}

    def close(self) -> None:
        if self._h:
            check(lib().bf_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def plan_create_status(n_ant: int, f: int, b: int, layout: int = 0) -> Status:
    """bf_plan_create's status for the given dimensions (destroys the plan on success)."""
    h = ctypes.c_void_p()
    s = lib().bf_plan_create(n_ant, f, b, layout, ctypes.byref(h))
    if s == 0:
        lib().bf_destroy(h)
    return Status(s)


class Server:
    """bf_server_*: a persistent launch serving untagged applies of `plan` (one precoder
    group) through a mapped-memory mailbox — no launch per slot (include/bf.h)."""

    def __init__(self, plan: Plan):
        self.plan = plan
        self._h = ctypes.c_void_p()
        check(lib().bf_server_create(plan._h, ctypes.byref(self._h)))
        self._keep = {}

    def start(self, stream=None) -> "Server":
        check(lib().bf_server_start(self._h, _stream_handle(stream)))
        return self

    def submit(self, S: torch.Tensor, out: torch.Tensor) -> int:
        """Post R = W x S into `out`; returns the slot's ticket (non-blocking)."""
        n = S.shape[0]
        self.plan._check(S, "S", self.plan.s_shape(n))
        self.plan._check(out, "out", self.plan.r_shape(n), dtype=self.plan.r_dtype)
        t = ctypes.c_uint64()
        check(lib().bf_server_submit(self._h, _ptr(S), _ptr(out), n, ctypes.byref(t)))
        self._keep[t.value % 8] = (S, out)
        return t.value

    def wait(self, ticket: int, timeout_s: float = 30.0) -> None:
        check(lib().bf_server_wait(self._h, ctypes.c_uint64(ticket), float(timeout_s)))

    def slot_time_us(self, ticket: int) -> float:
        """Device time of a done slot (doorbell seen by CTA 0 -> last CTA done), us."""
        v = ctypes.c_double()
        check(lib().bf_server_slot_time(self._h, ctypes.c_uint64(ticket), ctypes.byref(v)))
        return v.value

    def trace_us(self, per_cta: bool = False) -> list:
        """bf_server_trace: CTA 0's timeline of the last done slot (us after its doorbell);
        per_cta: then every CTA's slot start and count (BFTC_SRV_TRACE builds only)."""
        n = 8 + (320 if per_cta else 0)
        arr = (ctypes.c_double * n)()
        check(lib().bf_server_trace(self._h, arr, n))
        return list(arr)

    def stop(self) -> None:
        check(lib().bf_server_stop(self._h))

    def close(self) -> None:
        if self._h:
            check(lib().bf_server_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


__all__ = ["Plan", "Server", "Layout", "Status", "Variant", "BfError", "plan_create_status", "N_ANT", "N_RE",
           "MAX_F"]


def apply_batch(jobs, stream=None) -> None:
    """bf_apply_batch: jobs is a sequence of (plan, S, perm, offsets, out) with perm /
    offsets from Plan.route / route_into or both None; same checks as apply_routed."""
    arr = (BatchJob * max(1, len(jobs)))()
    keep = []
    for i, (plan, S, perm, offsets, out) in enumerate(jobs):
        n = S.shape[0]
        plan._check(S, "S", plan.s_shape(n))
        plan._check(out, "out", plan.r_shape(n), dtype=plan.r_dtype)
        arr[i] = BatchJob(plan._h.value, S.data_ptr(), None if perm is None else perm.data_ptr(),
                          None if offsets is None else offsets.data_ptr(), out.data_ptr(), n)
        keep.append((S, perm, offsets, out))
    check(lib().bf_apply_batch(arr, len(jobs), _stream_handle(stream)))
