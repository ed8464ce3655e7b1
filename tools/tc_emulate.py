"""Numpy model of the tensor kernel's split-precision arithmetic, used to
search for adversarial inputs, to check the dropped-term part of the error bound and (tests)
to check the kernel bit for bit.

The kernel scales every row of S (one RE: all k) by 2^sg and every precoder group by 2^tau
(powers of two placing the largest component in [2^14, 2^15)), splits the scaled values into
terms of 11 significant bits (tc_ptx.cuh tf32_round / cvt.rna.tf32: round to nearest, ties
away from zero), rounds every term to fp16 (round to nearest even; exact in fp16's normal
range), and sums the products it multiplies (general W: S2 W1 + S1 W2 + S1 W1; exact W:
S2 W1 + S3 W1 + S1 W1) with kind::f16 MMAs of K = 16, MMA by MMA with the tensor core's
accumulation in the bit-exact model that tools/tc_acc_probe measured (kernel_element); the
result is scaled back by 2^-(sg + tau) (one fp32 multiply).

    python tools/tc_emulate.py search [--n 20000] [--out tests/golden/tc_adversarial.txt]

`search` looks for complex (s, w) pairs with the largest |dR| / (|s| |w|) when every k of a
block holds the same pair (errors then add coherently over k) and writes them as a test
fixture of inputs; expected values always come from the oracle at test time.
Not part of the product; the GPU accuracy test uses kernel_element.
"""
from __future__ import annotations

import argparse
import sys

import numpy as np

REL_RANGE = 14          # bf_tc.cuh kRelRange
DOM_LO, DOM_HI = 0x2B800000, 0x53800000


def tf32(x: np.ndarray) -> np.ndarray:
    """Round fp32 to 11 significant bits, ties away (bit add 0x1000, mask), as the kernel."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x1000) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)


def h16(x: np.ndarray) -> np.ndarray:
    """fp32 -> fp16 (round to nearest even, cvt.rn.f16x2.f32) -> the exact value as fp64."""
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float64)


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


def scale_exp(comp_max_bits: np.ndarray) -> np.ndarray:
    """2^e placing the largest component (its fp32 bits) in [2^14, 2^15): e = 141 - biased."""
    e = (np.asarray(comp_max_bits, np.uint32) >> 23).astype(np.int64)
    return np.where(e != 0, 141 - e, 0)


def real_product(s, w):
    """What the kernel's MMAs sum for one real product s*w (exact accumulation; the split of
    the unscaled values — scaling by powers of two does not change the relative terms)."""
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


def mma_step(D, a, b, fp16=True):
    """One MMA on the accumulator values D [..] with operand rows a, b [.., K] (fp16 or tf32
    values), using the bit-exact model measured by tools/tc_acc_probe:
    alignment exponent E = max(e(D), e(a_k) + e(b_k)) — operand exponents clamped at fp16's
    subnormal exponent -14 for kind::f16 —, every addend truncated toward zero to a multiple
    of 2^(E - 25), exact sum, result rounded toward zero to fp32."""
    lo = -14.0 if fp16 else -1e9
    expo = lambda x: np.floor(np.log2(np.where(x != 0, np.abs(x), 1.0)))  # noqa: E731
    a64, b64 = np.asarray(a, np.float64), np.asarray(b, np.float64)
    P = a64 * b64
    D64 = np.asarray(D, np.float32).astype(np.float64)
    ep = np.where(P != 0, np.maximum(expo(a64), lo) + np.maximum(expo(b64), lo), -1e9)
    ec = np.where(D64 != 0, expo(D64), -1e9)
    E = np.maximum(ec, ep.max(axis=-1))
    E = np.where(E < -1e8, 0.0, E)
    terms = np.concatenate([D64[..., None], P], axis=-1)
    q = np.trunc(np.ldexp(terms, (25 - E).astype(np.int64)[..., None]))
    sm = np.ldexp(q.sum(axis=-1), (E - 25).astype(np.int64))
    rn = sm.astype(np.float32)
    over = np.abs(rn.astype(np.float64)) > np.abs(sm)
    return np.where(over, np.nextafter(rn, np.float32(0)), rn).astype(np.float32)


def group_scale(wr, wi):
    """The kernel's per-group W flags from the whole group's components: (tau, exact, in
    domain) — bf_api.cu bf_tc_build_wimg."""
    ur = np.abs(np.asarray(wr, np.float32)).view(np.uint32)
    ui = np.abs(np.asarray(wi, np.float32)).view(np.uint32)
    el = np.maximum(ur, ui)
    emax = int(el.max() >> 23)
    ok = bool(np.all(((ur == 0) | ((ur >= DOM_LO) & (ur < DOM_HI))) & ((ui == 0) | ((ui >= DOM_LO) & (ui < DOM_HI)))))
    ok &= emax == 0 or bool(np.all((el == 0) | ((el >> 23).astype(np.int64) >= emax - REL_RANGE)))
    tau = int(scale_exp(np.uint32(el.max()))) if ok else 0
    sc = np.float32(2.0 ** tau)
    exact = True
    for x in (wr, wi):
        v = np.asarray(x, np.float32) * sc
        b1, b2 = split_w(v)
        exact &= not np.any(b2) and np.array_equal(h16(b1), b1.astype(np.float64))
    return tau, exact, ok


def row_in_domain(sr, si, exact_w):
    """The split warps' test per row (last axis = k): largest element max(|re|, |im|) in
    [2^-40, 2^40), no NaN, every nonzero element within REL_RANGE binades of it, for exact W
    every nonzero scaled component >= 2^-1."""
    ur = np.abs(np.asarray(sr, np.float32)).view(np.uint32).astype(np.int64)
    ui = np.abs(np.asarray(si, np.float32)).view(np.uint32).astype(np.int64)
    el = np.maximum(ur, ui)
    emax = el.max(axis=-1) >> 23
    nan = np.any(np.isnan(sr) | np.isnan(si), axis=-1)
    ok = ~nan & (emax < (DOM_HI >> 23)) & ((emax == 0) | (emax >= (DOM_LO >> 23)))
    ok &= np.all((el == 0) | ((el >> 23) >= (emax - REL_RANGE)[..., None]), axis=-1)
    if exact_w:
        sg = np.where(emax != 0, 141 - emax, 0)
        for u in (ur, ui):
            ok &= np.all((u == 0) | ((u >> 23) + sg[..., None] >= 126), axis=-1)
    return ok


def kernel_element(sr, si, wr, wi, tau=None, exact_w=None):
    """The tensor kernel's re and im output for (antenna, RE) elements: sr, si [.., f]
    (S[k][j], the whole row) and wr, wi [.., f] (W[i][k]), emulated MMA by MMA in the
    kernel's order (general W: S2 W1, S1 W2, S1 W1; exact W: S2 W1, S3 W1, S1 W1), K = 16
    real columns (8 flows) per MMA, padded with zeros to KP = 16 ceil(2 f / 16).  tau, exact_w:
    the group's W scale and exact flag (group_scale of the whole group; None: every row of the
    given w values is its own group, as in the searches).  Rows outside the domain (see
    row_in_domain) are the FFMA fix-up's business; their values here are meaningless."""
    sr, si, wr, wi = (np.asarray(x, np.float32) for x in (sr, si, wr, wi))
    if tau is None or exact_w is None:      # every row (last axis) its own group
        wel = np.maximum(np.abs(wr).view(np.uint32), np.abs(wi).view(np.uint32)).max(axis=-1)
        tau = scale_exp(wel)
        wsc_r = np.ldexp(np.float32(1), tau).astype(np.float32)[..., None]
        exact_w = np.ones(wr.shape[:-1], bool)
        for x in (wr, wi):
            b1, b2 = split_w(x * wsc_r)
            exact_w &= ~np.any(b2 != 0, axis=-1) & np.all(h16(b1) == b1.astype(np.float64), axis=-1)
    tau = np.asarray(tau)
    exact_w = np.asarray(exact_w, bool)
    f = sr.shape[-1]
    kp = (2 * f + 15) // 16 * 16
    ur = np.abs(sr).view(np.uint32)
    ui = np.abs(si).view(np.uint32)
    sg = scale_exp(np.maximum(ur, ui).max(axis=-1))
    ssc = np.ldexp(np.float32(1), sg).astype(np.float32)[..., None]
    Aa = np.zeros(sr.shape[:-1] + (kp,), np.float32)
    Aa[..., 0:2 * f:2], Aa[..., 1:2 * f:2] = sr * ssc, si * ssc
    wsc = np.ldexp(np.float32(1), tau).astype(np.float32)[..., None]
    Bre = np.zeros(Aa.shape, np.float32)
    Bim = np.zeros(Aa.shape, np.float32)
    Bre[..., 0:2 * f:2], Bre[..., 1:2 * f:2] = wr * wsc, -wi * wsc
    Bim[..., 0:2 * f:2], Bim[..., 1:2 * f:2] = wi * wsc, wr * wsc
    a1, a2, a3 = (h16(x) for x in split_s(Aa))
    us = np.ldexp(np.float32(1), -(sg + tau)).astype(np.float32)
    out = []
    for B in (Bre, Bim):
        b1, b2 = (h16(x) for x in split_w(B))
        groups = [(a2, b1), (np.where(exact_w[..., None], a3, a1), np.where(exact_w[..., None], b1, b2)),
                  (a1, b1)]
        D = np.zeros(Aa.shape[:-1], np.float32)
        for ga, gb in groups:
            for kb in range(kp // 16):
                D = mma_step(D, ga[..., 16 * kb:16 * kb + 16], gb[..., 16 * kb:16 * kb + 16])
        out.append((D * us).astype(np.float32))
    return out[0], out[1]


def search(n: int, seed: int = 0, keep: int = 8, f: int = 36):
    """Worst |dR| / T of the emulated kernel (model accumulation) for blocks whose every k
    holds the same (s, w) pair: random pairs, then the best ones perturbed bit by bit."""
    rng = np.random.default_rng(seed)

    def score(c):          # c [m][4] = sr, si, wr, wi
        rep = lambda x: np.repeat(x[:, None], f, axis=1)  # noqa: E731
        re, im = kernel_element(rep(c[:, 0]), rep(c[:, 1]), rep(c[:, 2]), rep(c[:, 3]))
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
        re, im = kernel_element(c[:, 0], c[:, 1], c[:, 2], c[:, 3])
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
