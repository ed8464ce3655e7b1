"""Numpy model of the tensor kernel's split-precision arithmetic, used to
search for adversarial inputs and to check the dropped-term part of the error bound.

It models the operand splits exactly (tc_ptx.cuh tf32_round / cvt.rna.tf32: round to 11
significant bits, ties away from zero) and sums the products that the kernel multiplies
(general W: S2 W1 + S1 W2 + S1 W1; tf32-exact W: S2 W1 + S3 W1 + S1 W1), either exactly
(real_product / complex_error: the dropped terms alone) or MMA by MMA with the tensor
core's accumulation in the bit-exact model that tools/tc_acc_probe measured
(kernel_element).

    python tools/tc_emulate.py search [--n 20000] [--out tests/golden/tc_adversarial.txt]

`search` looks for complex (s, w) pairs with the largest |dR| / (|s| |w|) when every k of a
block holds the same pair (errors then add coherently over k) and writes them as a test
fixture of inputs; expected values always come from the oracle at test time.
Not part of the product; not imported by the tests.
"""
from __future__ import annotations

import argparse
import sys

import numpy as np


def tf32(x: np.ndarray) -> np.ndarray:
    """Round fp32 to 11 significant bits, ties away (bit add 0x1000, mask), as the kernel."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x1000) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)


def split_s(s):
    s = np.asarray(s, np.float32)
    s1 = tf32(s)
    r1 = (s.astype(np.float64) - s1).astype(np.float32)       # exact
    s2 = tf32(r1)
    s3 = (r1.astype(np.float64) - s2).astype(np.float32)      # exact
    return s1, s2, s3


def split_w(w):
    w = np.asarray(w, np.float32)
    w1 = tf32(w)
    w2 = tf32((w.astype(np.float64) - w1).astype(np.float32))
    return w1, w2


def real_product(s, w):
    """What the kernel's MMAs sum for one real product s*w (exact accumulation)."""
    s1, s2, s3 = split_s(s)
    w1, w2 = split_w(w)
    d = lambda a: np.asarray(a, np.float64)  # noqa: E731
    exact_w = d(w2) == 0
    general = d(s2) * d(w1) + d(s1) * d(w2) + d(s1) * d(w1)
    exactw = d(s2) * d(w1) + d(s3) * d(w1) + d(s1) * d(w1)
    return np.where(exact_w, exactw, general)


def complex_error(sr, si, wr, wi):
    """Per-k complex error of the embedding (re: wr sr - wi si, im: wi sr + wr si) and T."""
    d = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    re = real_product(sr, wr) - real_product(si, wi)
    im = real_product(sr, wi) + real_product(si, wr)
    ere = re - (d(wr) * d(sr) - d(wi) * d(si))
    eim = im - (d(wi) * d(sr) + d(wr) * d(si))
    T = np.hypot(d(wr), d(wi)) * np.hypot(d(sr), d(si))
    return np.hypot(ere, eim), T


def mma_step(D, a, b):
    """One kind::tf32 MMA on the accumulator values D [..] with operand rows a, b [.., 8],
    using the bit-exact model measured by tools/tc_acc_probe: alignment
    exponent E = max(e(D), e(a_k) + e(b_k)), every addend truncated toward zero to a
    multiple of 2^(E - 25), exact sum, result rounded toward zero to fp32."""
    expo = lambda x: np.floor(np.log2(np.where(x != 0, np.abs(x), 1.0)))  # noqa: E731
    a64, b64 = np.asarray(a, np.float64), np.asarray(b, np.float64)
    P = a64 * b64
    D64 = np.asarray(D, np.float32).astype(np.float64)
    ep = np.where(P != 0, expo(a64) + expo(b64), -1e9)
    ec = np.where(D64 != 0, expo(D64), -1e9)
    E = np.maximum(ec, ep.max(axis=-1))
    E = np.where(E < -1e8, 0.0, E)
    terms = np.concatenate([D64[..., None], P], axis=-1)
    q = np.trunc(np.ldexp(terms, (25 - E).astype(np.int64)[..., None]))
    sm = np.ldexp(q.sum(axis=-1), (E - 25).astype(np.int64))
    rn = sm.astype(np.float32)
    over = np.abs(rn.astype(np.float64)) > np.abs(sm)
    return np.where(over, np.nextafter(rn, np.float32(0)), rn).astype(np.float32)


def kernel_element(sr, si, wr, wi, exact_w=None):
    """The tensor kernel's re and im output for one (antenna, RE) element: sr, si [.., f]
    (S[k][j]) and wr, wi [.., f] (W[i][k]), emulated MMA by MMA in the kernel's order
    (general W: S2 W1, S1 W2, S1 W1; tf32-exact W: S2 W1, S3 W1, S1 W1), K = 8 real
    columns (4 flows) per MMA, padded with zeros to KP = 8 ceil(2 f / 8).  exact_w: whether
    the group's W is exactly tf32 (the kernel's per-group flag; None: derived from the
    given w values, which must then be the whole group)."""
    sr, si, wr, wi = (np.asarray(x, np.float32) for x in (sr, si, wr, wi))
    f = sr.shape[-1]
    kp = (2 * f + 7) // 8 * 8
    Aa = np.zeros(sr.shape[:-1] + (kp,), np.float32)
    Aa[..., 0:2 * f:2], Aa[..., 1:2 * f:2] = sr, si
    Bre = np.zeros(Aa.shape, np.float32)
    Bim = np.zeros(Aa.shape, np.float32)
    Bre[..., 0:2 * f:2], Bre[..., 1:2 * f:2] = wr, -wi
    Bim[..., 0:2 * f:2], Bim[..., 1:2 * f:2] = wi, wr
    a1, a2, a3 = split_s(Aa)
    if exact_w is None:
        exact_w = not (np.any(split_w(Bre)[1]) or np.any(split_w(Bim)[1]))
    out = []
    for B in (Bre, Bim):
        b1, b2 = split_w(B)
        groups = [(a2, b1), (a3, b1) if exact_w else (a1, b2), (a1, b1)]
        D = np.zeros(Aa.shape[:-1], np.float32)
        for ga, gb in groups:
            for kb in range(kp // 8):
                D = mma_step(D, ga[..., 8 * kb:8 * kb + 8], gb[..., 8 * kb:8 * kb + 8])
        out.append(D)
    return out[0], out[1]


def search(n: int, seed: int = 0, keep: int = 8, f: int = 36):
    """Worst |dR| / T of the emulated kernel (model accumulation) for blocks whose every k
    holds the same (s, w) pair: random pairs, then the best ones perturbed bit by bit."""
    rng = np.random.default_rng(seed)

    def score(c):          # c [m][4] = sr, si, wr, wi
        rep = lambda x: np.repeat(x[:, None], f, axis=1)  # noqa: E731
        re, im = kernel_element(rep(c[:, 0]), rep(c[:, 1]), rep(c[:, 2]), rep(c[:, 3]), False)
        d = c.astype(np.float64)
        ere = re - f * (d[:, 2] * d[:, 0] - d[:, 3] * d[:, 1])
        eim = im - f * (d[:, 3] * d[:, 0] + d[:, 2] * d[:, 1])
        T = f * np.hypot(d[:, 2], d[:, 3]) * np.hypot(d[:, 0], d[:, 1])
        return np.hypot(ere, eim) / T

    sign = rng.choice(np.array([-1.0, 1.0]), (n, 4))
    mag = rng.uniform(1.0, 2.0, (n, 4)) * 2.0 ** rng.integers(-1, 2, (n, 4))
    cand = (sign * mag).astype(np.float32)
    r = score(cand)
    best = cand[np.argsort(r)[::-1][:64]]
    for _ in range(6):                        # perturb the low mantissa bits of the best
        rep = np.repeat(best, 64, axis=0)
        bits = rep.view(np.uint32) ^ rng.integers(0, 1 << 12, rep.shape).astype(np.uint32)
        rep = bits.view(np.float32)
        allc = np.concatenate([best, rep])
        rr = score(allc)
        order = np.argsort(rr)[::-1]
        best = allc[order[:64]]
    rb = score(best)
    rows, seen = [], set()
    for i in np.argsort(rb)[::-1]:
        key = tuple(best[i].tolist())
        if key not in seen:
            seen.add(key)
            rows.append((float(rb[i]),) + tuple(float(x) for x in best[i]))
        if len(rows) == keep:
            break
    return rows


def search_structured(n: int, seed: int = 1, keep: int = 4, f: int = 36):
    """Worst |dR| / T over blocks with per-k values: the first 4 flows (the first main MMA)
    of magnitude ~1, the rest 2^-1..2^-4 smaller, random signs and mantissas, then the
    best perturbed in their low mantissa bits (the truncating accumulator loses most when
    a large partial sum meets many small addends whose low bits it cuts off)."""
    rng = np.random.default_rng(seed)

    def score(c):          # c [m][4][f] = sr, si, wr, wi
        re, im = kernel_element(c[:, 0], c[:, 1], c[:, 2], c[:, 3], False)
        d = c.astype(np.float64)
        ere = re - (d[:, 2] * d[:, 0] - d[:, 3] * d[:, 1]).sum(-1)
        eim = im - (d[:, 3] * d[:, 0] + d[:, 2] * d[:, 1]).sum(-1)
        T = (np.hypot(d[:, 2], d[:, 3]) * np.hypot(d[:, 0], d[:, 1])).sum(-1)
        return np.hypot(ere, eim) / T

    def gen(m):
        sign = rng.choice(np.array([-1.0, 1.0]), (m, 4, f))
        sc = np.ones((m, 1, f))
        sc[:, :, 4:] = 2.0 ** -rng.integers(2, 9, (m, 1, 1))
        return (sign * rng.uniform(1, 2, (m, 4, f)) * np.sqrt(sc)).astype(np.float32)

    best = None
    for _ in range(max(1, n // 2000)):
        c = gen(2000)
        allc = c if best is None else np.concatenate([best, c])
        best = allc[np.argsort(score(allc))[::-1][:32]]
    for _ in range(10):
        rep = np.repeat(best, 32, axis=0)
        bits = rep.view(np.uint32) ^ rng.integers(0, 1 << 10, rep.shape).astype(np.uint32)
        allc = np.concatenate([best, bits.view(np.float32)])
        best = allc[np.argsort(score(allc))[::-1][:32]]
    rb = score(best)
    return [(float(rb[i]), best[i]) for i in range(keep)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["search"])
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rows = search(a.n)
    lines = ["# Adversarial inputs for the tensor kernel's split precision (DESIGN.md §7).",
             "# Written by tools/tc_emulate.py search: a numpy emulation of the kernel (its operand",
             "# splits and MMA order, with the tensor core's accumulation in the bit-exact model",
             "# measured by tools/tc_acc_probe) searched for the (s, w) pairs with the largest",
             "# |dR| / T when EVERY k of a block holds the same pair (the per-k errors then add",
             "# coherently over f = 36).  Inputs only: expected values come from the oracle",
             "# (oracle/bf_oracle.c) at test time.",
             "# kind  emulated|dR|/T  sr si wr wi  (fp32 values, repr)"]
    for r, sr, si, wr, wi in rows:
        lines.append(f"complex {r:.6e} {sr!r} {si!r} {wr!r} {wi!r}")
    lines.append("# kind  emulated|dR|/T, then 4 lines of f = 36 values: sr[k], si[k], wr[k], wi[k]")
    for r, c in search_structured(a.n):
        lines.append(f"vector {r:.6e}")
        for row in c:
            lines.append(" ".join(repr(float(x)) for x in row))
    text = "\n".join(lines) + "\n"
    if a.out:
        open(a.out, "w").write(text)
    sys.stdout.write(text)


if __name__ == "__main__":
    main()
