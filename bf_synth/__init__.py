"""bf_synth — seeded, counter-based synthetic inputs for the beamforming path.

This module is the ONLY code shared between the oracle side (``oracle/``,
``tests/``, ``bench.py``'s cpu_baseline leg) and the CUDA side (bench and
parity tests).  It holds none of the method's arithmetic: it never forms a
product of W and S.  It only draws

* W   — complex-Gaussian precoders (BASELINE.json configs: "entries i.i.d.
        complex Gaussian", optionally "columns normalised to unit norm" or
        "scaled by 1/sqrt(8)"),
* S   — square M-QAM symbols normalised to unit average power (QPSK, 16-QAM,
        64-QAM per BASELINE.json configs),
* subband tags (which W a block uses), per-block modulation, per-cell f.

Every value is a pure function of (seed, stream, element index) through a
SplitMix64 counter hash, so any block can be regenerated independently of
chunking, rank count or device (DESIGN.md §"Input recipe").  The CUDA
generator in ``bf_synth/csrc/synth.cu`` implements the SAME hash for S, tags and
modulations (integer ops + a host-computed level table), and is checked
bitwise against this file by the GPU tests.  W is always drawn here, on the
host, in fp64 (it is small: at most 8 cells x 55 x 64 x 36 complex values).

Index spaces (fixed strides, independent of f and b so that a block's symbols
do not depend on how many blocks or which f the caller asks for):
    W element (g, i, k)  ->  e = (g * 256 + i) * 64 + k        (n_ant <= 256, f <= 64)
    S element (n, k, j)  ->  e = (n * 64 + k) * 256 + j         (f <= 64, b <= 256)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15          # SplitMix64 increment (golden ratio)
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB

# stream kinds (high 32 bits of the stream id); low 32 bits are a sub-stream
KIND_W = 1
KIND_S = 2
KIND_TAG = 3
KIND_MOD = 4
KIND_CELLF = 5
KIND_FSIG = 6     # filter-stage input signals

W_STRIDE_I = 256
W_STRIDE_K = 64
S_STRIDE_K = 64
S_STRIDE_J = 256


# --------------------------------------------------------------------------
# SplitMix64 counter hash
# --------------------------------------------------------------------------
def mix64_int(z: int) -> int:
    """SplitMix64 output function on a Python int (mod 2^64)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * M1) & MASK64
    z = ((z ^ (z >> 27)) * M2) & MASK64
    return z ^ (z >> 31)


def splitmix64_sequence(seed: int, count: int) -> list[int]:
    """The textbook SplitMix64 generator: state += GAMMA; output mix64(state)."""
    out, s = [], seed & MASK64
    for _ in range(count):
        s = (s + GAMMA) & MASK64
        out.append(mix64_int(s))
    return out


def stream_key(seed: int, kind: int, sub: int = 0) -> int:
    """64-bit key of one (seed, stream) pair."""
    stream = ((kind & 0xFFFFFFFF) << 32) | (sub & 0xFFFFFFFF)
    k = mix64_int((seed * GAMMA + 0x632BE59BD9B4E019) & MASK64)
    k ^= (stream * 0xD1B54A32D192ED03) & MASK64
    return mix64_int((k + GAMMA) & MASK64)


def counter_hash(key: int, idx: np.ndarray) -> np.ndarray:
    """h(idx) = mix64(key + (idx + 1) * GAMMA) for a uint64 index array.

    This is element ``idx`` of the SplitMix64 sequence seeded with ``key``.
    """
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (idx + np.uint64(1)) * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
        z = z ^ (z >> np.uint64(31))
    return z


def _unit53(h: np.ndarray) -> np.ndarray:
    """[0, 1) double from the top 53 bits."""
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _bounded(h: np.ndarray, n: int) -> np.ndarray:
    """Map a hash to [0, n) with the multiply-shift (Lemire) reduction on 32 bits."""
    hi = (h >> np.uint64(32)).astype(np.uint64)
    return ((hi * np.uint64(n)) >> np.uint64(32)).astype(np.int64)


# --------------------------------------------------------------------------
# W: complex Gaussian precoders (host, fp64 -> complex64)
# --------------------------------------------------------------------------
def complex_gaussian(seed: int, sub: int, n_groups: int, n_ant: int, f: int) -> np.ndarray:
    """fp64 CN(0,1) draws (re, im i.i.d. N(0, 1/2)) via Box-Muller, shape [G][A][f]."""
    if n_ant > W_STRIDE_I or f > W_STRIDE_K:
        raise ValueError("n_ant <= 256 and f <= 64 in the W index space")
    g, i, k = np.meshgrid(np.arange(n_groups), np.arange(n_ant), np.arange(f), indexing="ij")
    e = ((g.astype(np.uint64) * W_STRIDE_I + i.astype(np.uint64)) * W_STRIDE_K
         + k.astype(np.uint64))
    key = stream_key(seed, KIND_W, sub)
    h1 = counter_hash(key, e * np.uint64(2))
    h2 = counter_hash(key, e * np.uint64(2) + np.uint64(1))
    u1 = ((h1 >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)   # (0, 1]
    u2 = _unit53(h2)
    r = np.sqrt(-np.log(u1))
    return r * np.cos(2.0 * np.pi * u2) + 1j * (r * np.sin(2.0 * np.pi * u2))


def precoders(seed: int, sub: int, n_groups: int, n_ant: int, f: int,
              norm: str = "unit_columns") -> np.ndarray:
    """complex64 [G][A][f] precoders.

    norm: "unit_columns" (sum_i |w_ik|^2 = 1 per group and column, in fp64),
          "scale_inv_sqrt8" (c1: CN(0,1) / sqrt(8)), or "none" (plain CN(0,1)).
    """
    w = complex_gaussian(seed, sub, n_groups, n_ant, f)
    if norm == "unit_columns":
        if f:
            w = w / np.sqrt(np.sum(np.abs(w) ** 2, axis=1, keepdims=True))
    elif norm == "scale_inv_sqrt8":
        w = w / math.sqrt(8.0)
    elif norm != "none":
        raise ValueError(norm)
    return w.astype(np.complex64)


# --------------------------------------------------------------------------
# S: QAM symbols
# --------------------------------------------------------------------------
def qam_levels(M: int, normalised: bool = True) -> np.ndarray:
    """Per-axis levels of square M-QAM: (2 i - (L - 1)) / sqrt(2 (M - 1) / 3), as float32.

    i in [0, L), L = sqrt(M).  Unit average power when normalised.  The table
    is computed in fp64 and rounded once to fp32; the CUDA generator receives
    this same table.
    """
    L = int(round(math.sqrt(M)))
    if L * L != M or L & (L - 1):
        raise ValueError("square M-QAM with power-of-two sqrt(M) only")
    lv = np.array([2 * i - (L - 1) for i in range(L)], dtype=np.float64)
    if normalised:
        lv = lv / math.sqrt(2.0 * (M - 1) / 3.0)
    return lv.astype(np.float32)


MODULATIONS = (4, 16, 64)   # QPSK, 16-QAM, 64-QAM


def block_modulations(seed: int, block_ids: np.ndarray) -> np.ndarray:
    """Per-block M drawn uniformly from (4, 16, 64) (config c5)."""
    h = counter_hash(stream_key(seed, KIND_MOD, 0), np.asarray(block_ids, dtype=np.uint64))
    return np.asarray(MODULATIONS, dtype=np.int64)[_bounded(h, 3)]


def symbol_indices(seed: int, sub: int, block_ids: np.ndarray, f: int, b: int):
    """Raw per-element hashes of S, shape [n][f][b] (uint64)."""
    if f > S_STRIDE_K or b > S_STRIDE_J:
        raise ValueError("f <= 64 and b <= 256 in the S index space")
    n = np.asarray(block_ids, dtype=np.uint64).reshape(-1, 1, 1)
    k = np.arange(f, dtype=np.uint64).reshape(1, -1, 1)
    j = np.arange(b, dtype=np.uint64).reshape(1, 1, -1)
    e = (n * np.uint64(S_STRIDE_K) + k) * np.uint64(S_STRIDE_J) + j
    return counter_hash(stream_key(seed, KIND_S, sub), e)


def qam_symbols(seed: int, sub: int, block_ids, f: int, b: int, M,
                normalised: bool = True) -> np.ndarray:
    """complex64 S blocks [n][f][b].  M is an int or a per-block int array.

    Re level index = h & (L-1), Im level index = (h >> 8) & (L-1).
    """
    block_ids = np.asarray(block_ids, dtype=np.int64).reshape(-1)
    h = symbol_indices(seed, sub, block_ids, f, b)
    Ms = np.broadcast_to(np.asarray(M, dtype=np.int64), block_ids.shape)
    out = np.empty(h.shape, dtype=np.complex64)
    for m in np.unique(Ms):
        sel = Ms == m
        L = int(round(math.sqrt(int(m))))
        lv = qam_levels(int(m), normalised)
        hs = h[sel]
        ire = (hs & np.uint64(L - 1)).astype(np.int64)
        iim = ((hs >> np.uint64(8)) & np.uint64(L - 1)).astype(np.int64)
        o = np.empty(hs.shape, dtype=np.complex64)
        o.real = lv[ire]
        o.imag = lv[iim]
        out[sel] = o
    return out


KIND_GS = 7       # Gaussian S (accuracy tests: continuous values instead of QAM levels)


def gaussian_symbols(seed: int, sub: int, block_ids, f: int, b: int,
                     exp_spread: int = 0) -> np.ndarray:
    """complex64 S blocks [n][f][b] of fp32 CN(0,1) draws (Box-Muller in fp64, one rounding),
    for accuracy tests whose inputs must exercise every significand bit (QAM levels exercise
    only a handful).  exp_spread > 0 multiplies each element by 2^u, u uniform in
    [-exp_spread, exp_spread] (wide dynamic range inside a block)."""
    block_ids = np.asarray(block_ids, dtype=np.int64).reshape(-1)
    if f > S_STRIDE_K or b > S_STRIDE_J:
        raise ValueError("f <= 64 and b <= 256 in the S index space")
    n = block_ids.astype(np.uint64).reshape(-1, 1, 1)
    k = np.arange(f, dtype=np.uint64).reshape(1, -1, 1)
    j = np.arange(b, dtype=np.uint64).reshape(1, 1, -1)
    e = (n * np.uint64(S_STRIDE_K) + k) * np.uint64(S_STRIDE_J) + j
    key = stream_key(seed, KIND_GS, sub)
    h1 = counter_hash(key, e * np.uint64(3))
    h2 = counter_hash(key, e * np.uint64(3) + np.uint64(1))
    u1 = ((h1 >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)   # (0, 1]
    u2 = _unit53(h2)
    r = np.sqrt(-np.log(u1))
    z = r * np.cos(2.0 * np.pi * u2) + 1j * (r * np.sin(2.0 * np.pi * u2))
    if exp_spread > 0:
        h3 = counter_hash(key, e * np.uint64(3) + np.uint64(2))
        u = _bounded(h3, 2 * exp_spread + 1) - exp_spread
        z = z * np.ldexp(1.0, u)
    return z.astype(np.complex64)


def subband_tags(seed: int, block_ids, n_groups: int) -> np.ndarray:
    """int32 tag in [0, n_groups) per block, uniform (configs c4, c5)."""
    h = counter_hash(stream_key(seed, KIND_TAG, 0), np.asarray(block_ids, dtype=np.uint64))
    return _bounded(h, n_groups).astype(np.int32)


def cell_flows(seed: int, n_cells: int, f_max: int = 36) -> np.ndarray:
    """Per-cell flow count f_c ~ U{1..f_max} (config c5)."""
    h = counter_hash(stream_key(seed, KIND_CELLF, 0), np.arange(n_cells, dtype=np.uint64))
    return (_bounded(h, f_max) + 1).astype(np.int64)


# --------------------------------------------------------------------------
# Layout helpers (pure data movement; no arithmetic of the method)
# --------------------------------------------------------------------------
def to_planar(x: np.ndarray) -> np.ndarray:
    """complex64 [..., r, c] -> float32 [..., 2, r, c] (re plane, then im plane)."""
    return np.ascontiguousarray(np.stack([x.real, x.imag], axis=-3).astype(np.float32))


def from_planar(p: np.ndarray) -> np.ndarray:
    """float32 [..., 2, r, c] -> complex64 [..., r, c]."""
    out = np.empty(p.shape[:-3] + p.shape[-2:], dtype=np.complex64)
    out.real = p[..., 0, :, :]
    out.imag = p[..., 1, :, :]
    return out


# --------------------------------------------------------------------------
# The five BASELINE.json workloads
# --------------------------------------------------------------------------
C3_FLOWS = (0, 1, 2, 3, 4, 7, 8, 12, 16, 17, 24, 31, 32, 36)


@dataclass(frozen=True)
class Workload:
    name: str
    n_ant: int
    f: int                      # -1 for mixed (c5)
    b: int
    n_blocks: int
    n_groups: int
    M: int                      # 0 for mixed per block (c5)
    seed: int
    w_norm: str
    sub: int = 0                # stream sub-id (c3: f)
    tagged: bool = False        # per-block subband tags
    desc: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def block_bytes(self) -> int:
        """Algorithmic bytes per block: S read + R write."""
        return 8 * self.b * (self.f + self.n_ant)

    @property
    def block_flops(self) -> int:
        """8 real FLOPs per complex MAC x n_ant x b x f."""
        return 8 * self.n_ant * self.b * self.f


def workload(name: str, f: int | None = None) -> Workload:
    """BASELINE.json configs[0..4] as concrete workloads (DESIGN.md §Input recipe)."""
    if name == "c1":
        return Workload("c1", 64, 8, 60, 16, 1, 4, 0, "scale_inv_sqrt8",
                        desc="BASELINE.json configs[0]: 1 W 64x8, 16 QPSK blocks, seed 0")
    if name == "c2":
        return Workload("c2", 64, 36, 60, 770, 1, 64, 1, "unit_columns",
                        desc="BASELINE.json configs[1]: 1 W 64x36, 770 64-QAM blocks "
                             "(55 subbands x 14 symbols), seed 1")
    if name == "c3":
        if f is None:
            raise ValueError("c3 needs f")
        if f not in C3_FLOWS:
            raise ValueError(f"c3 f must be one of {C3_FLOWS}")
        return Workload(f"c3_f{f}", 64, f, 60, 100_000, 1, 16, 2, "none", sub=f,
                        desc=f"BASELINE.json configs[2]: f={f}, 100000 16-QAM blocks, seed 2")
    if name == "c4":
        return Workload("c4", 64, 36, 60, 1 << 20, 55, 64, 3, "unit_columns", tagged=True,
                        desc="BASELINE.json configs[3]: 55 W 64x36, 2^20 64-QAM blocks "
                             "tagged U{0..54}, seed 3")
    if name == "c5":
        return Workload("c5", 64, -1, 60, 1 << 23, 55, 0, 4, "none", tagged=True,
                        desc="BASELINE.json configs[4]: 8 cells x 55 W 64xf_c, 2^23 blocks "
                             "of mixed QPSK/16/64-QAM in 4096-block chunks, seed 4",
                        extra={"n_cells": 8, "chunk": 4096})
    raise ValueError(name)


def c5_cell_of_block(block_ids) -> np.ndarray:
    """c5: chunk c = n // 4096 belongs to cell c mod 8 (reading R13)."""
    return (np.asarray(block_ids, dtype=np.int64) // 4096) % 8


def workload_inputs(wl: Workload, block_ids=None):
    """Host (numpy) inputs of a single-f workload for the given blocks.

    Returns (W complex64 [G][A][f], S complex64 [n][f][b], tags int32 [n] or None).
    """
    if wl.f < 0:
        raise ValueError("use c5 helpers for mixed-f workloads")
    if block_ids is None:
        block_ids = np.arange(wl.n_blocks, dtype=np.int64)
    W = precoders(wl.seed, wl.sub, wl.n_groups, wl.n_ant, wl.f, wl.w_norm)
    S = qam_symbols(wl.seed, wl.sub, block_ids, wl.f, wl.b, wl.M)
    tags = subband_tags(wl.seed, block_ids, wl.n_groups) if wl.tagged else None
    return W, S, tags


# --------------------------------------------------------------------------
# Filter stage: signals and the filter sequence
# --------------------------------------------------------------------------
FILTER_N = 2048      # "FFT sizes are all 2048"


def filter_signals(seed: int, sub: int, sig_ids, n: int = FILTER_N, M: int = 64) -> np.ndarray:
    """complex64 [n_sig][n] synthetic time samples: square M-QAM points, index e = sig*n + k."""
    ids = np.asarray(sig_ids, dtype=np.uint64).reshape(-1, 1)
    e = ids * np.uint64(n) + np.arange(n, dtype=np.uint64).reshape(1, -1)
    h = counter_hash(stream_key(seed, KIND_FSIG, sub), e)
    L = int(round(math.sqrt(M)))
    lv = qam_levels(M)
    out = np.empty(h.shape, dtype=np.complex64)
    out.real = lv[(h & np.uint64(L - 1)).astype(np.int64)]
    out.imag = lv[((h >> np.uint64(8)) & np.uint64(L - 1)).astype(np.int64)]
    return out


def filter_taps(n: int = FILTER_N, taps: int = 64, cutoff: float = 0.25) -> np.ndarray:
    """The filter sequence h (complex64 [n]): a Hann-windowed sinc low-pass FIR of
    `taps` real taps (normalised cutoff in cycles/sample, DC gain 1), zero-padded to n.
    Computed in fp64, rounded once to fp32."""
    k = np.arange(taps, dtype=np.float64) - (taps - 1) / 2.0
    h = 2.0 * cutoff * np.sinc(2.0 * cutoff * k) * (0.5 - 0.5 * np.cos(2 * np.pi * np.arange(taps) / (taps - 1)))
    h /= h.sum()
    out = np.zeros(n, dtype=np.complex64)
    out[:taps] = h.astype(np.float32)
    return out


@dataclass(frozen=True)
class FilterWorkload:
    name: str
    n: int
    n_signals: int
    M: int
    seed: int
    desc: str = ""

    @property
    def signal_bytes(self) -> int:
        """Algorithmic bytes per signal: read s + write y (complex fp32)."""
        return 2 * 8 * self.n


def filter_workload(name: str) -> FilterWorkload:
    if name == "fl0":
        return FilterWorkload("fl0", FILTER_N, 16, 64, 5, "16 signals of 2048 64-QAM samples, seed 5")
    if name == "fl1":
        return FilterWorkload("fl1", FILTER_N, 1 << 18, 64, 6,
                              "2^18 signals of 2048 64-QAM samples (4.3 GB in + out), seed 6")
    raise ValueError(name)


# --------------------------------------------------------------------------
# OFDM output stage: symbols of nb consecutive blocks
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class OfdmWorkload:
    name: str
    n_sym: int          # OFDM symbols (each nb consecutive blocks of 60 REs)
    nb: int             # blocks (subbands) per symbol: nb * 60 active subcarriers
    f: int
    n: int              # IFFT size
    cp: int             # cyclic prefix samples
    M: int
    seed: int
    desc: str = ""
    n_ant: int = 64
    b: int = 60

    @property
    def n_blocks(self) -> int:
        return self.n_sym * self.nb

    def symbol_bytes(self, out_bytes: int = 8, fused: bool = True) -> int:
        """Algorithmic HBM bytes per symbol: S read + output write (+ R write and read when
        the beamformed symbol goes through HBM between the two stages, fused=False)."""
        s = self.nb * 8 * self.b * self.f
        y = self.n_ant * (self.cp + self.n) * out_bytes
        r = 0 if fused else 2 * self.nb * 8 * self.b * self.n_ant
        return s + y + r


def ofdm_workload(name: str) -> OfdmWorkload:
    """of0 (tests), of1 (bench): 26 subbands x 60 REs = 1560 active subcarriers in a
    2048-point IFFT (a 50 MHz carrier at 30 kHz spacing), normal cyclic prefix 144,
    f = 36 flows, one unit-column precoder per subband (tag = block mod nb)."""
    if name == "of0":
        return OfdmWorkload("of0", 6, 26, 36, 2048, 144, 64, 7,
                            "6 symbols x 26 subbands, f = 36, 64-QAM, seed 7")
    if name == "of1":
        return OfdmWorkload("of1", 1 << 15, 26, 36, 2048, 144, 64, 8,
                            "2^15 symbols x 26 subbands (851 968 blocks), f = 36, 64-QAM, seed 8")
    raise ValueError(name)


def ofdm_tags(block_ids, nb: int) -> np.ndarray:
    """Subband of each block: blocks of a symbol are its subbands in order (block mod nb)."""
    return (np.asarray(block_ids, dtype=np.int64) % nb).astype(np.int32)


def ofdm_inputs(wl: OfdmWorkload, sym_ids=None):
    """(W complex64 [nb][64][f], S complex64 [len(sym_ids) * nb][f][60], tags int32) for the
    given symbols (default: all)."""
    if sym_ids is None:
        sym_ids = np.arange(wl.n_sym, dtype=np.int64)
    sym_ids = np.asarray(sym_ids, dtype=np.int64).reshape(-1)
    ids = (sym_ids[:, None] * wl.nb + np.arange(wl.nb)[None, :]).reshape(-1)
    W = precoders(wl.seed, 0, wl.nb, wl.n_ant, wl.f, "unit_columns")
    S = qam_symbols(wl.seed, 0, ids, wl.f, wl.b, wl.M)
    return W, S, ofdm_tags(ids, wl.nb)
