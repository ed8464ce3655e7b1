"""Device-side generation of the bf_synth inputs (bench + GPU tests only).

Same counter hash and level tables as bf_synth/__init__.py, so a block drawn
here equals the numpy block bitwise (checked in tests/test_parity_gpu.py).
W is never drawn here: it always comes from the host generator (fp64).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import (KIND_FSIG, KIND_MOD, KIND_S, KIND_TAG, MODULATIONS, Workload, qam_levels,
               stream_key)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbfsynth.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64
        L.bfs_gen_qam.argtypes = [vp, vp, i64, i64, i32, i32, u64, i32, vp, i32, u64, vp]
        L.bfs_gen_tags.argtypes = [vp, vp, i64, i64, u64, i32, vp]
        L.bfs_gen_mods.argtypes = [vp, vp, i64, i64, u64, vp]
        L.bfs_fill_u32.argtypes = [vp, i64, ctypes.c_uint32, vp]
        L.bfs_gen_signals.argtypes = [vp, i64, i64, i32, u64, vp, i32, vp]
        for f in (L.bfs_gen_qam, L.bfs_gen_tags, L.bfs_gen_mods, L.bfs_fill_u32, L.bfs_gen_signals):
            f.restype = i32
        _lib = L
    return _lib


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_LEVELS = np.zeros(24, dtype=np.float32)
for _m, _M in enumerate(MODULATIONS):
    _lv = qam_levels(_M)
    _LEVELS[_m * 8:_m * 8 + len(_lv)] = _lv


def gen_symbols(out: torch.Tensor, seed: int, sub: int, f: int, b: int, M: int,
                first: int = 0, ids: torch.Tensor | None = None, planar: bool = False) -> torch.Tensor:
    """Fill out (cuda; complex64 [n][f][b] or float32 [n][2][f][b]) with QAM symbols.

    M in (4, 16, 64) for all blocks, or 0 to draw the modulation per block (c5).
    Blocks are ids[i] if ids is given (int64 cuda), else first + i.
    """
    n = out.shape[0]
    mod_idx = -1 if M == 0 else MODULATIONS.index(M)
    lv = np.ascontiguousarray(_LEVELS)
    rc = _load().bfs_gen_qam(
        ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(None if ids is None else ids.data_ptr()),
        int(first), int(n), int(f), int(b), stream_key(seed, KIND_S, sub), int(planar),
        lv.ctypes.data_as(ctypes.c_void_p), mod_idx, stream_key(seed, KIND_MOD, 0), _stream())
    if rc:
        raise RuntimeError(f"bfs_gen_qam failed: cudaError {rc}")
    return out


def gen_tags(out: torch.Tensor, seed: int, n_groups: int, first: int = 0,
             ids: torch.Tensor | None = None) -> torch.Tensor:
    rc = _load().bfs_gen_tags(ctypes.c_void_p(out.data_ptr()),
                              ctypes.c_void_p(None if ids is None else ids.data_ptr()),
                              int(first), int(out.shape[0]), stream_key(seed, KIND_TAG, 0),
                              int(n_groups), _stream())
    if rc:
        raise RuntimeError(f"bfs_gen_tags failed: cudaError {rc}")
    return out


def gen_modulations(out: torch.Tensor, seed: int, first: int = 0,
                    ids: torch.Tensor | None = None) -> torch.Tensor:
    rc = _load().bfs_gen_mods(ctypes.c_void_p(out.data_ptr()),
                              ctypes.c_void_p(None if ids is None else ids.data_ptr()),
                              int(first), int(out.shape[0]), stream_key(seed, KIND_MOD, 0),
                              _stream())
    if rc:
        raise RuntimeError(f"bfs_gen_mods failed: cudaError {rc}")
    return out


def fill_u32(buf: torch.Tensor, value: int = 0) -> None:
    """Overwrite a buffer (L2 flush between timed iterations)."""
    n = buf.numel() * buf.element_size() // 4
    rc = _load().bfs_fill_u32(ctypes.c_void_p(buf.data_ptr()), int(n), value & 0xFFFFFFFF,
                              _stream())
    if rc:
        raise RuntimeError(f"bfs_fill_u32 failed: cudaError {rc}")


def workload_device(wl: Workload, device, first: int = 0, n: int | None = None,
                    ids: torch.Tensor | None = None, planar: bool = False):
    """Device S (and tags) of a single-f workload for blocks [first, first+n) or ids."""
    if n is None:
        n = wl.n_blocks if ids is None else ids.shape[0]
    if planar:
        S = torch.empty((n, 2, wl.f, wl.b), dtype=torch.float32, device=device)
    else:
        S = torch.empty((n, wl.f, wl.b), dtype=torch.complex64, device=device)
    if wl.f > 0 and n > 0:
        gen_symbols(S, wl.seed, wl.sub, wl.f, wl.b, wl.M, first=first, ids=ids, planar=planar)
    tags = None
    if wl.tagged:
        tags = torch.empty(n, dtype=torch.int32, device=device)
        if n > 0:
            gen_tags(tags, wl.seed, wl.n_groups, first=first, ids=ids)
    return S, tags


def gen_filter_signals(out: torch.Tensor, seed: int, sub: int = 0, first: int = 0,
                       M: int = 64) -> torch.Tensor:
    """Fill out (cuda complex64 [n_sig][n]) with bf_synth.filter_signals(seed, sub, first + i)."""
    n_sig, n = out.shape
    lv = np.ascontiguousarray(_LEVELS)
    rc = _load().bfs_gen_signals(ctypes.c_void_p(out.data_ptr()), int(first), int(n_sig), int(n),
                                 stream_key(seed, KIND_FSIG, sub), lv.ctypes.data_as(ctypes.c_void_p),
                                 MODULATIONS.index(M), _stream())
    if rc:
        raise RuntimeError(f"bfs_gen_signals failed: cudaError {rc}")
    return out
