"""Pins of the OFDM-output oracle (oracle/ofdm_oracle.c; SURVEY.md §8(f) row 4:
beamforming, followed by the per-antenna OFDM IFFT; readings O1-O5
in DESIGN.md §2).

The paper prints no numbers for this stage, so the oracle is pinned to
hand-expanded examples (tests/golden/ofdm_hand_examples.txt, n = 4: every value
exact), the closed form of a single active subcarrier (a complex exponential),
Parseval, the cyclic-prefix identity, linearity, the bound's closed form, and a
library routine (numpy einsum + numpy.fft.ifft) on a realistic size — each
chosen so a plausible mistake (exponent sign, bin offset, CP on the wrong end,
transposed W, dropped scale) fails one of them.
"""
import os

import numpy as np
import pytest

import bf_synth as syn
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ofdm_hand_examples.txt")


def _golden():
    cases, cur = {}, None
    for line in open(GOLDEN):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        t = line.split()
        if t[0] == "case":
            n, b, nb, A, F, G, cp = map(int, t[2:9])
            scale, n_sym = float(t[9]), int(t[10])
            cur = dict(n=n, nb=nb, cp=cp, scale=scale,
                       W=np.zeros((G, A, F), np.complex64),
                       S=np.zeros((n_sym * nb, F, b), np.complex64),
                       tags=None, y=np.full((n_sym, A, cp + n), np.nan, np.complex64))
            cases[t[1]] = cur
        elif t[0] == "W":
            g, a, k = map(int, t[1:4])
            cur["W"][g, a, k] = complex(float(t[4]), float(t[5]))
        elif t[0] == "S":
            blk, k, j = map(int, t[1:4])
            cur["S"][blk, k, j] = complex(float(t[4]), float(t[5]))
        elif t[0] == "tag":
            if cur["tags"] is None:
                cur["tags"] = np.zeros(cur["S"].shape[0], np.int32)
            cur["tags"][int(t[1])] = int(t[2])
        elif t[0] == "y":
            m, a, u = map(int, t[1:4])
            cur["y"][m, a, u] = complex(float(t[4]), float(t[5]))
    return cases


@pytest.mark.parametrize("name", ["A", "B", "C"])
def test_golden_hand_expanded(name):
    c = _golden()[name]
    assert not np.isnan(c["y"]).any()
    y, _ = oracle.ofdm(c["W"], c["S"], c["nb"], n=c["n"], cp=c["cp"], scale=c["scale"],
                       group_idx=c["tags"])
    # cos(pi/2) is 6e-17 in fp64, so "exact" means within a few ulps of the largest value
    assert np.allclose(y, c["y"], rtol=0, atol=1e-6), (name, y, c["y"])


def _rand(seed, G, A, F, nblk, b=60):
    W = syn.precoders(seed, 0, G, A, F, "unit_columns")
    S = syn.gaussian_symbols(seed, 0, np.arange(nblk), F, b)
    return W, S


@pytest.mark.parametrize("nb,q0", [(26, 0), (26, 779), (26, 780), (26, 1559), (3, 91)])
def test_single_subcarrier_is_a_complex_exponential(nb, q0):
    """Only subcarrier q0 nonzero: x[t] = scale R e^{+2 pi i bin t / n}, bin = (q0 - Nsc/2) mod n,
    evaluated here from numpy's exp of the reduced angle (and R from numpy's fp64 matmul)."""
    n, cp, scale, b = 2048, 144, 0.25, 60
    W, _ = _rand(3, 1, 2, 4, 1)
    S = np.zeros((nb, 4, b), np.complex64)
    blk, j = divmod(q0, b)
    S[blk, :, j] = np.array([1 + 2j, -0.5j, 0.75, -1 + 1j], np.complex64)
    y, _ = oracle.ofdm(W, S, nb, n=n, cp=cp, scale=scale)
    R = W[0].astype(np.complex128) @ S[blk, :, j].astype(np.complex128)   # [A]
    binq = (q0 - nb * b // 2) % n
    t = np.arange(n)
    e = np.exp(2j * np.pi * ((binq * t) % n) / n)
    for a in range(2):
        x = scale * R[a] * e
        ref = np.concatenate([x[n - cp:], x])
        assert np.abs(y[0, a] - ref).max() <= 1e-6 * np.abs(R[a]) * scale + 1e-30


def test_matches_numpy_ifft_at_the_workload_shape():
    """Library routine: R = einsum in fp64, X mapped by index arithmetic, numpy.fft.ifft * n."""
    wl = syn.ofdm_workload("of0")
    W, S, tags = syn.ofdm_inputs(wl, np.arange(2))
    y, bound = oracle.ofdm(W, S, wl.nb, n=wl.n, cp=wl.cp, scale=1.0, group_idx=tags, n_threads=8)
    R = np.einsum("nak,nkj->naj", W[tags].astype(np.complex128), S.astype(np.complex128))
    nsc = wl.nb * wl.b
    for m in range(2):
        for a in (0, 17, 63):
            X = np.zeros(wl.n, np.complex128)
            sc = R[m * wl.nb:(m + 1) * wl.nb, a, :].reshape(-1)          # q = blk * 60 + j
            X[(np.arange(nsc) - nsc // 2) % wl.n] = sc
            x = np.fft.ifft(X) * wl.n
            ref = np.concatenate([x[wl.n - wl.cp:], x])
            err = np.abs(y[m, a] - ref).max()
            assert err <= 1e-6 * np.abs(ref).max(), (m, a, err)
            # bound closed form: sum_q T_q + sqrt(n) ||X||_2
            Tq = sum((np.abs(W[tags[m * wl.nb + k], a].astype(np.complex128))
                      @ np.abs(S[m * wl.nb + k].astype(np.complex128))).sum() for k in range(wl.nb))
            assert bound[m, a] == pytest.approx(Tq + np.sqrt(wl.n) * np.linalg.norm(sc), rel=1e-12)


def test_parseval_and_cyclic_prefix():
    W, S = _rand(5, 1, 4, 6, 10)
    n, cp, nb = 2048, 160, 5
    y, _ = oracle.ofdm(W, S, nb, n=n, cp=cp, n_threads=4)
    R = np.einsum("ak,nkj->naj", W[0].astype(np.complex128), S.astype(np.complex128))
    for m in range(2):
        for a in range(4):
            X2 = (np.abs(R[m * nb:(m + 1) * nb, a, :]) ** 2).sum()
            x = y[m, a, cp:].astype(np.complex128)
            assert (np.abs(x) ** 2).sum() == pytest.approx(n * X2, rel=1e-6)
            # the prefix is the tail, value for value
            assert np.array_equal(y[m, a, :cp], y[m, a, n:n + cp])


def test_linearity_and_scale():
    W, S1 = _rand(6, 1, 2, 3, 4)
    S2 = syn.gaussian_symbols(9, 0, np.arange(4), 3, 60)
    ya, _ = oracle.ofdm(W, S1, 2, cp=8)
    yb, _ = oracle.ofdm(W, S2, 2, cp=8)
    yc, _ = oracle.ofdm(W, (S1 + 2 * S2).astype(np.complex64), 2, cp=8, scale=0.5)
    ref = 0.5 * (ya.astype(np.complex128) + 2 * yb.astype(np.complex128))
    assert np.abs(yc - ref).max() <= 1e-5 * np.abs(ref).max()


def test_f0_and_rejections():
    W = np.zeros((1, 64, 0), np.complex64)
    S = np.zeros((4, 0, 60), np.complex64)
    y, bound = oracle.ofdm(W, S, 2, cp=4)
    assert not y.any() and not bound.any()
    W, S = _rand(1, 1, 2, 2, 4)
    with pytest.raises(ValueError):
        oracle.ofdm(W, S, 3)                         # blocks not a multiple of nb
    with pytest.raises(ValueError):
        oracle.ofdm(W, S, 2, n=64)                   # 120 subcarriers > n
    with pytest.raises(ValueError):
        oracle.ofdm(W, S, 2, group_idx=np.array([0, 1, 0, 0], np.int32))   # tag out of range
