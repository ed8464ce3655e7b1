"""Pins of the filter-stage oracle (oracle/filter_oracle.c).

The paper prints no filter numbers (Fig. 4 is lost, its timings are machine-
specific), so the oracle is pinned to hand-expanded examples
(tests/golden/filter_hand_examples.txt), closed forms of the DFT, Parseval,
the convolution theorem (two independent formulas must agree), shifts, and a
library routine (numpy.fft).
"""
import os

import numpy as np
import pytest

import bf_synth as syn
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "filter_hand_examples.txt")


def _golden():
    cases, cur = {}, None
    for line in open(GOLDEN):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        if tok[0] in ("dft", "filter"):
            n = int(tok[2])
            cur = {"kind": tok[0], "n": n}
            cases[tok[1]] = cur
        else:
            arr = cur.setdefault(tok[0], np.zeros(cur["n"], np.complex64))
            arr[int(tok[1])] = complex(float(tok[2]), float(tok[3]))
    return cases


def test_golden_dft_hand_expanded():
    c = _golden()["A"]
    assert np.allclose(oracle.dft(c["x"]), c["X"], atol=1e-6)   # cos(pi/2) != 0 in fp64
    assert np.allclose(oracle.dft(c["X"], inverse=True), c["x"], atol=1e-6)


@pytest.mark.parametrize("name", ["B", "C"])
def test_golden_filter_hand_expanded(name):
    c = _golden()[name]
    for direct in (False, True):
        y, _ = oracle.filter_apply(c["s"], c["h"], direct=direct)
        assert np.allclose(y[0], c["y"], atol=1e-6), (name, direct, y[0], c["y"])


def test_dft_closed_forms():
    n = 2048
    d = np.zeros(n, np.complex64); d[0] = 1
    assert np.allclose(oracle.dft(d), 1.0, atol=1e-12)                     # delta -> ones
    c = np.full(n, 0.5 - 0.25j, np.complex64)
    X = oracle.dft(c)
    assert abs(X[0] - n * (0.5 - 0.25j)) < 1e-9 and np.abs(X[1:]).max() < 1e-9   # const -> delta
    m = 37
    tone = np.exp(2j * np.pi * m * np.arange(n) / n).astype(np.complex64)
    X = oracle.dft(tone)
    assert abs(X[m] - n) < 1e-3 and np.abs(np.delete(X, m)).max() < 1e-3      # tone -> n delta_m


def test_dft_parseval_roundtrip_and_numpy():
    rng = np.random.default_rng(0)
    x = (rng.standard_normal((3, 2048)) + 1j * rng.standard_normal((3, 2048))).astype(np.complex64)
    X = oracle.dft(x)
    e_t = np.sum(np.abs(x.astype(np.complex128)) ** 2, axis=1)
    e_f = np.sum(np.abs(X.astype(np.complex128)) ** 2, axis=1) / 2048
    assert np.allclose(e_t, e_f, rtol=1e-6)
    assert np.allclose(oracle.dft(X, inverse=True), x, atol=1e-5)
    ref = np.fft.fft(x.astype(np.complex128), axis=1)
    assert np.abs(X - ref).max() <= 2e-7 * np.abs(ref).max()


def test_convolution_theorem_two_formulas_agree():
    """IDFT(DFT(h) . DFT(s)) (mode 0) against the direct circular convolution (mode 1)."""
    s = syn.filter_signals(1, 0, np.arange(3))
    h = syn.filter_taps()
    y0, b = oracle.filter_apply(s, h, n_threads=3)
    y1, _ = oracle.filter_apply(s, h, n_threads=3, direct=True)
    assert (np.abs(y0 - y1).max(axis=1) <= 1e-7 * b).all()


def test_filter_identity_shift_linearity():
    n = 2048
    s = syn.filter_signals(2, 0, np.arange(2))
    d = np.zeros(n, np.complex64); d[0] = 1
    y, b = oracle.filter_apply(s, d)
    assert (np.abs(y - s).max(axis=1) <= 1e-12 * b + 2 ** -23).all()          # identity filter
    d1 = np.zeros(n, np.complex64); d1[5] = 1
    y, _ = oracle.filter_apply(s, d1, direct=True)
    assert np.array_equal(y, np.roll(s, 5, axis=1))                          # cyclic delay
    h = syn.filter_taps()
    s2 = syn.filter_signals(3, 0, np.arange(2))
    ya, ba = oracle.filter_apply(s + s2, h)
    yb, _ = oracle.filter_apply(s, h)
    yc, _ = oracle.filter_apply(s2, h)
    assert (np.abs(ya - (yb + yc)).max(axis=1) <= 1e-6 * ba).all()           # linearity


def test_filter_bound_and_workloads():
    h = syn.filter_taps()
    assert abs(np.sum(h.astype(np.complex128)) - 1) < 1e-6                    # DC gain 1
    s = syn.filter_signals(4, 0, np.arange(2))
    _, b = oracle.filter_apply(s, h)
    H = np.fft.fft(h.astype(np.complex128))
    assert np.allclose(b, np.linalg.norm(s.astype(np.complex128), axis=1) * np.abs(H).max())
    assert set(np.unique(s.real).tolist()) <= set(syn.qam_levels(64).tolist())
    wl = syn.filter_workload("fl1")
    assert wl.n == 2048 and wl.signal_bytes == 32768
