"""Pins of the CPU oracle (oracle/bf_oracle.c) against things other than itself.

Each test pins the oracle to something the paper or mathematics fixes, chosen so
that a plausible mistake (a dropped term, a wrong sign, a conjugation, a
transposed operand, a wrong group or block index, a wrong rounding) fails one
of them.  The paper prints no numeric beamforming example (its
Fig. 5 is lost), so the pins are: hand-expanded fixtures (tests/golden/),
closed forms, special cases, exact integer arithmetic, a library routine
(numpy complex128 matmul = BLAS zgemm) and exact rational arithmetic.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import bf_synth as syn
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "bf_hand_examples.txt")


def _parse_golden():
    cases, cur = {}, None
    for line in open(GOLDEN):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        if tok[0] == "case":
            A, F, B, G, N = map(int, tok[2:7])
            cur = dict(W=np.zeros((G, A, F), np.complex64), S=np.zeros((N, F, B), np.complex64),
                       G=None, R={}, T={})
            cases[tok[1]] = cur
        elif tok[0] == "W":
            g, i, k = map(int, tok[1:4])
            cur["W"][g, i, k] = complex(float(tok[4]), float(tok[5]))
        elif tok[0] == "S":
            n, k, j = map(int, tok[1:4])
            cur["S"][n, k, j] = complex(float(tok[4]), float(tok[5]))
        elif tok[0] == "G":
            if cur["G"] is None:
                cur["G"] = np.zeros(cur["S"].shape[0], np.int32)
            cur["G"][int(tok[1])] = int(tok[2])
        elif tok[0] == "R":
            cur["R"][tuple(map(int, tok[1:4]))] = complex(float(tok[4]), float(tok[5]))
        elif tok[0] == "T":
            cur["T"][tuple(map(int, tok[1:4]))] = eval(tok[4], {"__builtins__": {}},
                                                       {"sqrt": math.sqrt})
    return cases


@pytest.mark.parametrize("name", ["A", "B", "C"])
def test_golden_hand_expanded(name):
    """PAPER.md:84-86 equation expanded by hand (tests/golden/bf_hand_examples.txt)."""
    c = _parse_golden()[name]
    R, T, _ = oracle.beamform(c["W"], c["S"], c["G"])
    assert len(c["R"]) == R.size
    for (n, i, j), v in c["R"].items():
        assert R[n, i, j] == np.complex64(v), (name, n, i, j, R[n, i, j], v)
    for (n, i, j), t in c["T"].items():
        assert T[n, i, j] == pytest.approx(t, rel=1e-14)


def test_f0_is_positive_zero_bitwise():
    """f = 0: the empty sum, +0.0 exactly ("f can vary from 0")."""
    W = np.zeros((1, 64, 0), np.complex64)
    S = np.zeros((5, 0, 60), np.complex64)
    R, T, flops = oracle.beamform(W, S)
    assert R.shape == (5, 64, 60)
    assert not R.view(np.uint32).any()          # +0.0 bit patterns only
    assert not T.any() and flops == 0


@pytest.mark.parametrize("A,F,B,N", [(64, 36, 60, 3), (64, 1, 60, 2), (7, 5, 3, 4), (1, 1, 1, 1)])
def test_flop_counter_closed_form(A, F, B, N):
    """Counted FLOPs == 8 * n_ant * b * f per block."""
    rng = np.random.default_rng(0)
    W = (rng.standard_normal((1, A, F)) + 1j * rng.standard_normal((1, A, F))).astype(np.complex64)
    S = (rng.standard_normal((N, F, B)) + 1j * rng.standard_normal((N, F, B))).astype(np.complex64)
    _, _, flops = oracle.beamform(W, S, n_threads=3)
    assert flops == 8 * A * B * F * N


def _qam(seed, n, f, b=60, M=64):
    return syn.qam_symbols(seed, 0, np.arange(n), f, b, M)


@pytest.mark.parametrize("f", [1, 8, 17, 36])
def test_identity_reproduces_rows_bitwise(f):
    """W = [I_f ; 0] (R7): rows i < f of R are rows of S, rows >= f are +0."""
    W = np.zeros((1, 64, f), np.complex64)
    W[0, np.arange(f), np.arange(f)] = 1
    S = _qam(5, 3, f)
    R, _, _ = oracle.beamform(W, S)
    assert np.array_equal(R[:, :f].view(np.uint32), S.view(np.uint32))
    assert not R[:, f:].view(np.uint32).any()


def test_selection_permutation_bitwise():
    """W[i][k] = 1 iff k = sigma(i): R row i is S row sigma(i), bitwise."""
    f = 36
    rng = np.random.default_rng(1)
    sigma = rng.integers(0, f, size=64)
    sigma[:f] = rng.permutation(f)
    W = np.zeros((1, 64, f), np.complex64)
    W[0, np.arange(64), sigma] = 1
    S = _qam(7, 4, f)
    R, _, _ = oracle.beamform(W, S)
    assert np.array_equal(R.view(np.uint32), S[:, sigma].view(np.uint32))


def test_one_real_nonzero_per_row_correctly_rounded():
    """One real nonzero c per row: R = c * s rounded once (exact product in fp64)."""
    f = 12
    rng = np.random.default_rng(2)
    sigma = rng.integers(0, f, size=64)
    c = rng.standard_normal(64).astype(np.float32)
    W = np.zeros((1, 64, f), np.complex64)
    W[0, np.arange(64), sigma] = c
    S = _qam(9, 2, f).astype(np.complex64)
    R, _, _ = oracle.beamform(W, S)
    exp_re = (c.astype(np.float64)[None, :, None] * S[:, sigma].real.astype(np.float64)).astype(np.float32)
    exp_im = (c.astype(np.float64)[None, :, None] * S[:, sigma].imag.astype(np.float64)).astype(np.float32)
    assert np.array_equal(R.real, exp_re) and np.array_equal(R.imag, exp_im)


def test_gaussian_integers_exact_against_integer_arithmetic():
    """Gaussian-integer inputs: every partial sum is an integer < 2^24, so the
    oracle must equal exact int64 arithmetic bitwise (SURVEY.md §8(c) P-c),
    at full c4 shape with several groups and tags."""
    rng = np.random.default_rng(3)
    G, A, F, B, N = 5, 64, 36, 60, 6
    Wr = rng.integers(-3, 4, (G, A, F)); Wi = rng.integers(-3, 4, (G, A, F))
    S = syn.qam_symbols(11, 0, np.arange(N), F, B, 64, normalised=False)
    Sr = S.real.astype(np.int64); Si = S.imag.astype(np.int64)
    tags = rng.integers(0, G, N).astype(np.int32)
    W = (Wr + 1j * Wi).astype(np.complex64)
    R, _, _ = oracle.beamform(W, S, tags, n_threads=2)
    Er = np.einsum("nik,nkj->nij", Wr[tags], Sr) - np.einsum("nik,nkj->nij", Wi[tags], Si)
    Ei = np.einsum("nik,nkj->nij", Wr[tags], Si) + np.einsum("nik,nkj->nij", Wi[tags], Sr)
    assert np.abs(Er).max() < 2 ** 24
    assert np.array_equal(R.real, Er.astype(np.float32))
    assert np.array_equal(R.imag, Ei.astype(np.float32))


def test_against_numpy_zgemm():
    """Library cross-check (SURVEY.md P-d): numpy complex128 W @ S (BLAS zgemm).

    The oracle is the exact product rounded once to fp32 (up to its own fp64
    error <= ~2f 2^-53 T); so per component |R - Z| <= 2^-24 |Z| + 1e-13 T.
    """
    wl = syn.workload("c2")
    W, S, _ = syn.workload_inputs(wl, np.arange(0, 770, 97))
    R, T, _ = oracle.beamform(W, S, n_threads=4)
    Z = np.stack([W[0].astype(np.complex128) @ S[n].astype(np.complex128) for n in range(len(S))])
    lim = 2.0 ** -24 * np.abs(Z.real) + 1e-13 * T
    assert (np.abs(R.real - Z.real) <= lim).all()
    lim = 2.0 ** -24 * np.abs(Z.imag) + 1e-13 * T
    assert (np.abs(R.imag - Z.imag) <= lim).all()
    # and most elements are exactly the correctly rounded zgemm value
    assert np.mean(R == Z.astype(np.complex64)) > 0.999


def test_exact_rational_rounding_bound():
    """Against exact rational arithmetic (fractions.Fraction): |R - X| <= 2^-24 |X| + 2^-40 T."""
    rng = np.random.default_rng(4)
    A, F, B = 3, 9, 4
    W = (rng.standard_normal((1, A, F)) + 1j * rng.standard_normal((1, A, F))).astype(np.complex64)
    S = (rng.standard_normal((1, F, B)) + 1j * rng.standard_normal((1, F, B))).astype(np.complex64)
    R, T, _ = oracle.beamform(W, S)
    for i in range(A):
        for j in range(B):
            xr = sum(Fraction(float(W[0, i, k].real)) * Fraction(float(S[0, k, j].real))
                     - Fraction(float(W[0, i, k].imag)) * Fraction(float(S[0, k, j].imag))
                     for k in range(F))
            xi = sum(Fraction(float(W[0, i, k].real)) * Fraction(float(S[0, k, j].imag))
                     + Fraction(float(W[0, i, k].imag)) * Fraction(float(S[0, k, j].real))
                     for k in range(F))
            t = T[0, i, j]
            for got, x in ((R[0, i, j].real, xr), (R[0, i, j].imag, xi)):
                err = abs(Fraction(float(got)) - x)
                assert err <= Fraction(2.0 ** -24) * abs(x) + Fraction(2.0 ** -40) * Fraction(t)


def test_linearity_exact_on_integers():
    """R is linear in S and in W (SURVEY.md P-f); exact on Gaussian-integer inputs."""
    rng = np.random.default_rng(5)
    A, F, B, N = 64, 16, 60, 2
    W1 = (rng.integers(-3, 4, (1, A, F)) + 1j * rng.integers(-3, 4, (1, A, F))).astype(np.complex64)
    W2 = (rng.integers(-3, 4, (1, A, F)) + 1j * rng.integers(-3, 4, (1, A, F))).astype(np.complex64)
    S1 = syn.qam_symbols(1, 0, np.arange(N), F, B, 16, normalised=False)
    S2 = syn.qam_symbols(2, 0, np.arange(N), F, B, 64, normalised=False)
    f = lambda W, S: oracle.beamform(W, S)[0]
    assert np.array_equal(f(W1, S1 + S2), f(W1, S1) + f(W1, S2))
    assert np.array_equal(f(W1 + W2, S1), f(W1, S1) + f(W2, S1))
    assert np.array_equal(f(W1, 3 * S1), 3 * f(W1, S1))


def test_power_of_two_scaling_bitwise():
    """Scaling W by 2^e scales R by 2^e exactly (no over/underflow)."""
    wl = syn.workload("c2")
    W, S, _ = syn.workload_inputs(wl, np.arange(3))
    R1 = oracle.beamform(W, S)[0]
    R2 = oracle.beamform((W * np.float32(8.0)).astype(np.complex64), S)[0]
    R3 = oracle.beamform((W * np.float32(0.25)).astype(np.complex64), S)[0]
    assert np.array_equal(R2, R1 * np.float32(8.0))
    assert np.array_equal(R3, R1 * np.float32(0.25))


def test_conjugation_symmetry_bitwise():
    """R(conj W, conj S) = conj R(W, S): the expansion is sign-symmetric (SURVEY.md P-i).
    A conjugation or swapped re/im term in the oracle breaks this or the golden file."""
    wl = syn.workload("c2")
    W, S, _ = syn.workload_inputs(wl, np.arange(2))
    R = oracle.beamform(W, S)[0]
    Rc = oracle.beamform(np.conj(W), np.conj(S))[0]
    assert np.array_equal(Rc.view(np.uint32), np.conj(R).view(np.uint32))


def test_bound_T_closed_form_and_dominance():
    """Positive real inputs: |w||s| = w s so T equals R (up to rounding); in general |R| <= T."""
    rng = np.random.default_rng(6)
    W = rng.uniform(0.5, 2, (1, 8, 10)).astype(np.complex64)
    S = rng.uniform(0.5, 2, (2, 10, 7)).astype(np.complex64)
    R, T, _ = oracle.beamform(W, S)
    assert np.array_equal(R.real, T.astype(np.float32))
    assert not R.imag.any()
    wl = syn.workload("c2")
    W, S, _ = syn.workload_inputs(wl, np.arange(2))
    R, T, _ = oracle.beamform(W, S)
    assert (np.abs(R.astype(np.complex128)) <= T * (1 + 1e-6)).all()


def test_group_index_selects_precoder():
    """Tagged blocks use W[tag] (BASELINE.json configs[3]): equals per-group calls."""
    wl = syn.workload("c4")
    ids = np.arange(0, 1 << 20, (1 << 20) // 12)
    W, S, tags = syn.workload_inputs(wl, ids)
    R, _, _ = oracle.beamform(W, S, tags, n_threads=4)
    for n in range(len(ids)):
        Rn, _, _ = oracle.beamform(W[tags[n]], S[n:n + 1])
        assert np.array_equal(R[n], Rn[0])
    bad = tags.copy(); bad[0] = 55
    with pytest.raises(ValueError):
        oracle.beamform(W, S, bad)


def test_thread_count_independence():
    wl = syn.workload("c3", 17)
    W, S, _ = syn.workload_inputs(wl, np.arange(9))
    a = oracle.beamform(W, S, n_threads=1)
    b = oracle.beamform(W, S, n_threads=5)
    assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
    assert np.array_equal(a[1], b[1]) and a[2] == b[2]


def test_shape_mismatch_rejected():
    with pytest.raises(ValueError):
        oracle.beamform(np.zeros((1, 4, 3), np.complex64), np.zeros((1, 2, 5), np.complex64))
