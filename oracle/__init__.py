"""CPU oracle for the beamforming hot path (§III equation).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package.  The product package ``paper_1810_11451_b200`` never imports it and
shares no code with it; the only shared module is the input generator
``bf_synth`` (no arithmetic of the method).

The arithmetic lives in ``bf_oracle.c`` (beamforming),
``filter_oracle.c`` (the filter stage IFFT(MULT(FFT(s)))) and
``ofdm_oracle.c`` (beamforming followed by the per-antenna OFDM IFFT, SURVEY.md
§8(f) row 4): plain C, fp64, one rounding to fp32; see their headers for the passage-by-passage
reading.  This file only builds the C library with gcc and marshals numpy arrays.

Pins (tests/test_oracle_pins.py, ``-m "not gpu"``): hand-expanded golden
fixture (tests/golden/), f = 0 closed form, identity / selection / permutation
special cases, Gaussian-integer inputs against exact integer arithmetic,
numpy complex128 matmul (zgemm) cross-check, exact-rational rounding bound,
linearity, conjugation symmetry, T closed form, FLOP-count closed form and
group indexing.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import tempfile

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "bf_oracle.c"), os.path.join(_HERE, "filter_oracle.c"),
         os.path.join(_HERE, "ofdm_oracle.c")]
_LIB = os.path.join(_HERE, "libbforacle.so")
_CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
           "-pthread"]
_lib = None


def build(force: bool = False) -> str:
    """Compile bf_oracle.c with gcc into oracle/libbforacle.so (atomic rename)."""
    if (not force and os.path.exists(_LIB)
            and all(os.path.getmtime(_LIB) >= os.path.getmtime(src) for src in _SRCS)):
        return _LIB
    fd, tmp = tempfile.mkstemp(suffix=".so", dir=_HERE)
    os.close(fd)
    try:
        subprocess.run(["gcc", *_CFLAGS, "-o", tmp, *_SRCS, "-lm"], check=True)
        os.replace(tmp, _LIB)
    finally:
        if os.path.exists(tmp):
            os.unlink(tmp)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.bfo_beamform.restype = ctypes.c_int
        lib.bfo_beamform.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]
        lib.fo_dft.restype = ctypes.c_int
        lib.fo_dft.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                               ctypes.c_int]
        lib.fo_filter.restype = ctypes.c_int
        lib.fo_filter.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_int]
        lib.fm_ofdm.restype = ctypes.c_int
        lib.fm_ofdm.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def beamform(W: np.ndarray, S: np.ndarray, group_idx: np.ndarray | None = None,
             n_threads: int = 1, bound: bool = True):
    """Oracle R = W[g(n)] x S[n] for every block n.

    W: complex64 [G][n_ant][f] (or [n_ant][f] for one group);
    S: complex64 [n][f][b];  group_idx: int32 [n] in [0, G) or None (group 0).
    Returns (R complex64 [n][n_ant][b], T float64 [n][n_ant][b] or None, flops int).
    Raises ValueError on invalid input (the C side returns -1).
    """
    W = np.ascontiguousarray(W, dtype=np.complex64)
    if W.ndim == 2:
        W = W[None]
    S = np.ascontiguousarray(S, dtype=np.complex64)
    G, A, F = W.shape
    n, F2, B = S.shape
    if F2 != F:
        raise ValueError(f"W has f={F} but S has f={F2}")
    gi = None
    if group_idx is not None:
        gi = np.ascontiguousarray(group_idx, dtype=np.int32)
        if gi.shape != (n,):
            raise ValueError("group_idx must have one entry per block")
    R = np.empty((n, A, B), dtype=np.complex64)
    T = np.empty((n, A, B), dtype=np.float64) if bound else None
    flops = ctypes.c_int64(0)
    rc = _load().bfo_beamform(A, F, B, G, n, _ptr(W), _ptr(S), _ptr(gi), _ptr(R), _ptr(T),
                              int(n_threads), ctypes.byref(flops))
    if rc != 0:
        raise ValueError("oracle rejected the arguments (sizes or group index)")
    return R, T, int(flops.value)


def max_threads() -> int:
    """Host threads available to this process (for the cpu_baseline leg)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# Filter stage: IFFT(MULT(FFT(s))), n = 2048
# ---------------------------------------------------------------------------
def dft(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Direct O(n^2) DFT of the last axis in fp64 (unnormalised forward, 1/n inverse)."""
    x = np.ascontiguousarray(x, dtype=np.complex64)
    flat = x.reshape(-1, x.shape[-1])
    out = np.empty_like(flat)
    rc = _load().fo_dft(_ptr(flat), _ptr(out), flat.shape[-1], flat.shape[0], int(inverse))
    if rc != 0:
        raise ValueError("oracle rejected the arguments")
    return out.reshape(x.shape)


def filter_apply(s: np.ndarray, h: np.ndarray, n_threads: int = 1, direct: bool = False):
    """y = IDFT(DFT(h) . DFT(s)) per signal (direct=True: circular convolution s (*) h).

    s: complex64 [n_sig][n]; h: complex64 [n] (the filter sequence).
    Returns (y complex64 [n_sig][n], bound float64 [n_sig] = ||s||_2 max|DFT(h)|).
    """
    s = np.ascontiguousarray(s, dtype=np.complex64)
    if s.ndim == 1:
        s = s[None]
    h = np.ascontiguousarray(h, dtype=np.complex64).reshape(-1)
    n_sig, n = s.shape
    if h.shape[0] != n:
        raise ValueError("h must have the signal length")
    y = np.empty_like(s)
    bound = np.empty(n_sig, dtype=np.float64)
    rc = _load().fo_filter(_ptr(s), _ptr(h), _ptr(y), _ptr(bound), n, n_sig, 1 if direct else 0,
                           int(n_threads))
    if rc != 0:
        raise ValueError("oracle rejected the arguments")
    return y, bound


# ---------------------------------------------------------------------------
# OFDM output: per-antenna IFFT of the beamformed symbol
# ---------------------------------------------------------------------------
def ofdm(W: np.ndarray, S: np.ndarray, nb: int, n: int = 2048, cp: int = 0, scale: float = 1.0,
         group_idx: np.ndarray | None = None, n_threads: int = 1):
    """y[m][a] = CP(scale * IDFT_unnormalised(map(R[m*nb : m*nb+nb][a]))) from fp64 R = W x S.

    W: complex64 [G][A][F] (or [A][F]); S: complex64 [n_sym*nb][F][b]; group_idx int32
    [n_sym*nb] or None.  Subcarrier q of a symbol (block q // b, element q % b) sits in bin
    (q - nb*b/2) mod n.  Returns (y complex64 [n_sym][A][cp + n], bound float64 [n_sym][A]).
    """
    W = np.ascontiguousarray(W, dtype=np.complex64)
    if W.ndim == 2:
        W = W[None]
    S = np.ascontiguousarray(S, dtype=np.complex64)
    G, A, F = W.shape
    nblk, F2, B = S.shape
    if F2 != F or nblk % nb != 0:
        raise ValueError("S must be [n_sym*nb][f][b] with W's f")
    n_sym = nblk // nb
    gi = None
    if group_idx is not None:
        gi = np.ascontiguousarray(group_idx, dtype=np.int32)
        if gi.shape != (nblk,):
            raise ValueError("group_idx must have one entry per block")
    y = np.empty((n_sym, A, cp + n), dtype=np.complex64)
    bound = np.empty((n_sym, A), dtype=np.float64)
    rc = _load().fm_ofdm(A, F, B, G, n_sym, int(nb), int(n), int(cp), float(scale), _ptr(W),
                         _ptr(S), _ptr(gi), _ptr(y), _ptr(bound), int(n_threads))
    if rc != 0:
        raise ValueError("oracle rejected the arguments (sizes or group index)")
    return y, bound
