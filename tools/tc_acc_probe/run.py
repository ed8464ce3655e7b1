"""Measures the tcgen05 kind::tf32 accumulation model used by DESIGN.md §7 (run on a B200).

Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
            -o tools/tc_acc_probe/libtcacc.so tools/tc_acc_probe/tc_acc_probe.cu
Run:    python tools/tc_acc_probe/run.py [--np 64] [--out gpurun_out/tc_acc.json]

Every case runs `np` independent 128 x 128 problems D = C + sum_m A_m B_m^T (K = 8 per
MMA, tf32-exact operands) and compares D with the exact sum (products exact in fp64,
the terms summed in extended precision, smallest magnitude first).  For one MMA the
error is reported in units of u23(M) = 2^-23 * M with M = max(|C|, max_k |a_k b_k|)
(the largest addend) and of ulp(M); for chains, in units of 2^-23 * sum |terms|.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def lib():
    L = ctypes.CDLL(os.path.join(HERE, "libtcacc.so"))
    L.acc_run.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int] * 3
    L.acc_run_kind.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int] * 4
    return L


def h16(x):
    """fp16-exact values (round to nearest fp16), as fp32."""
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float32)


def tf32(x):
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x1000) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)


def run(L, A, B, C, c_mode=1, kind=0):
    npb, nmma = A.shape[0], A.shape[1]
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    C = np.ascontiguousarray(C, np.float32)
    D = np.empty((npb, 128, 128), np.float32)
    rc = L.acc_run_kind(A.ctypes.data, B.ctypes.data, C.ctypes.data, D.ctypes.data, npb, nmma, c_mode,
                        kind)
    assert rc == 0, rc
    return D


def exact(A, B, C, c_mode=1):
    """Exact D (extended precision): terms [np][128][128][nmma*8 (+1)], summed by magnitude."""
    npb, nmma, K = A.shape[0], A.shape[1], A.shape[3]
    A64 = A.astype(np.float64).transpose(0, 2, 1, 3).reshape(npb, 128, nmma * K)
    B64 = B.astype(np.float64).transpose(0, 2, 1, 3).reshape(npb, 128, nmma * K)
    out = np.empty((npb, 128, 128), np.longdouble)
    absum = np.empty((npb, 128, 128), np.float64)
    amax = np.empty((npb, 128, 128), np.float64)
    for p in range(npb):
        terms = A64[p][:, None, :] * B64[p][None, :, :]          # exact (22-bit products)
        if c_mode:
            terms = np.concatenate([terms, C[p].astype(np.float64)[..., None]], axis=-1)
        order = np.argsort(np.abs(terms), axis=-1)
        t = np.take_along_axis(terms, order, axis=-1).astype(np.longdouble)
        out[p] = t.sum(axis=-1)
        absum[p] = np.abs(terms).sum(axis=-1)
        amax[p] = np.abs(terms).max(axis=-1)
    return out, absum, amax


def stats(D, ex, absum, amax, nmma):
    err = (D.astype(np.longdouble) - ex).astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        u_max = np.where(amax > 0, np.abs(err) / (2.0 ** -23 * amax), 0.0)
        ulp_m = np.where(amax > 0, 2.0 ** (np.floor(np.log2(np.where(amax > 0, amax, 1))) - 23), 1)
        in_ulp = np.abs(err) / ulp_m
        u_sum = np.where(absum > 0, np.abs(err) / (2.0 ** -23 * absum), 0.0)
        signed = np.where(amax > 0, err / ulp_m, 0.0)
    return {"max_err_over_u23_maxaddend": float(u_max.max()),
            "max_err_in_ulp_of_maxaddend": float(in_ulp.max()),
            "max_err_over_u23_sumabs": float(u_sum.max()),
            "mean_signed_err_ulp_maxaddend": float(signed.mean()),
            "frac_exact": float((err == 0).mean()), "n": int(err.size), "nmma": nmma}


def cases(rng, npb):
    g = lambda *s: rng.standard_normal(s)  # noqa: E731
    sh = (npb, 1, 128, 8)
    yield "gauss_c0", tf32(g(*sh)), tf32(g(*sh)), np.zeros((npb, 128, 128)), 0
    u = rng.integers(-20, 21, (npb, 128, 128))
    yield "gauss_c_scaled", tf32(g(*sh)), tf32(g(*sh)), g(npb, 128, 128) * 2.0 ** u, 1
    yield ("positive", tf32(rng.uniform(0.5, 1, sh)), tf32(rng.uniform(0.5, 1, sh)),
           rng.uniform(0.5, 1, (npb, 128, 128)) * 2.0 ** rng.integers(-3, 4, (npb, 128, 128)), 1)
    v = rng.integers(-30, 31, sh)
    w = rng.integers(-30, 31, sh)
    yield "spread_exponents", tf32(g(*sh) * 2.0 ** v), tf32(g(*sh) * 2.0 ** w), g(npb, 128, 128), 1
    # large accumulator, small same-sign addends whose bits fall below its ulp
    a = tf32(rng.uniform(1, 2, sh) * 2.0 ** rng.integers(-32, -20, sh))
    b = tf32(rng.uniform(1, 2, sh))
    yield "trunc_below_acc_pos", a, b, np.ones((npb, 128, 128)) * rng.uniform(1, 2, (npb, 128, 128)), 1
    yield "trunc_below_acc_neg", -a, b, np.ones((npb, 128, 128)) * rng.uniform(1, 2, (npb, 128, 128)), 1
    # one large product, the other addends small, mixed signs
    a2 = tf32(g(*sh) * 2.0 ** rng.integers(-26, -10, sh))
    a2[..., 0] = tf32(rng.uniform(1, 2, (npb, 1, 128)))
    yield "one_large_product", a2, tf32(g(*sh)), g(npb, 128, 128) * 2.0 ** -12, 1
    # cancellation: C = -(fp32 sum of the products) + perturbation
    A3, B3 = tf32(g(*sh)), tf32(g(*sh))
    s = np.einsum("pmik,pmjk->pij", A3.astype(np.float64), B3.astype(np.float64))
    yield "cancellation", A3, B3, (-s).astype(np.float32) * (1 + 2.0 ** -20 * g(npb, 128, 128)), 1
    # alternating-sign addends of equal magnitude around a large C
    a4 = tf32(np.ones(sh) * rng.uniform(1, 2, sh))
    a4[..., 1::2] *= -1
    yield "alternating", a4, tf32(rng.uniform(1, 2, sh)), rng.uniform(1, 2, (npb, 128, 128)) * 16, 1


def chain_cases(rng, npb):
    """The product kernel's chain at f = 36: 9 MMAs of S2 W1, 9 of S1 W2 (both ~2^-11 of the
    main product), then 9 of S1 W1; and the same with everything positive (no cancellation)."""
    sh = (npb, 9, 128, 8)
    for name, gen in (("kernel_chain_gauss", lambda: rng.standard_normal(sh)),
                      ("kernel_chain_positive", lambda: rng.uniform(0.5, 1.0, sh))):
        s, w = gen().astype(np.float32), gen().astype(np.float32)
        s1, w1 = tf32(s), tf32(w)
        s2, w2 = tf32(s - s1), tf32(w - w1)
        A = np.concatenate([s2, s1, s1], axis=1)
        B = np.concatenate([w1, w2, w1], axis=1)
        yield name, A, B, np.zeros((npb, 128, 128)), 0


def cases16(rng, npb):
    """kind::f16 (fp16 operands, K = 16): the same families within fp16's range."""
    g = lambda *s: rng.standard_normal(s)  # noqa: E731
    sh = (npb, 1, 128, 16)
    yield "f16_gauss_c0", h16(g(*sh)), h16(g(*sh)), np.zeros((npb, 128, 128)), 0
    u = rng.integers(-20, 21, (npb, 128, 128))
    yield "f16_gauss_c_scaled", h16(g(*sh)), h16(g(*sh)), g(npb, 128, 128) * 2.0 ** u, 1
    yield ("f16_positive", h16(rng.uniform(0.5, 1, sh)), h16(rng.uniform(0.5, 1, sh)),
           rng.uniform(0.5, 1, (npb, 128, 128)) * 2.0 ** rng.integers(-3, 4, (npb, 128, 128)), 1)
    v = rng.integers(-12, 13, sh)
    w = rng.integers(-12, 13, sh)
    yield "f16_spread_exponents", h16(g(*sh) * 2.0 ** v), h16(g(*sh) * 2.0 ** w), g(npb, 128, 128), 1
    a = h16(rng.uniform(1, 2, sh) * 2.0 ** rng.integers(-14, -4, sh))
    b = h16(rng.uniform(1, 2, sh) * 2.0 ** rng.integers(-14, -4, sh))
    yield "f16_trunc_below_acc_pos", a, b, np.ones((npb, 128, 128)) * rng.uniform(1, 2, (npb, 128, 128)), 1
    yield "f16_trunc_below_acc_neg", -a, b, np.ones((npb, 128, 128)) * rng.uniform(1, 2, (npb, 128, 128)), 1
    a2 = h16(g(*sh) * 2.0 ** rng.integers(-14, -2, sh))
    a2[..., 0] = h16(rng.uniform(1, 2, (npb, 1, 128)) * 2.0 ** 10)
    yield "f16_one_large_product", a2, h16(g(*sh)), g(npb, 128, 128) * 2.0 ** -2, 1
    A3, B3 = h16(g(*sh) * 64), h16(g(*sh) * 64)
    s = np.einsum("pmik,pmjk->pij", A3.astype(np.float64), B3.astype(np.float64))
    yield "f16_cancellation", A3, B3, (-s).astype(np.float32) * (1 + 2.0 ** -20 * g(npb, 128, 128)), 1
    a4 = h16(np.ones(sh) * rng.uniform(1, 2, sh))
    a4[..., 1::2] *= -1
    yield "f16_alternating", a4, h16(rng.uniform(1, 2, sh)), rng.uniform(1, 2, (npb, 128, 128)) * 16, 1
    # fp16 subnormal operands (exact in fp16) and products near fp16's range ends
    sub = h16(rng.integers(1, 1024, sh) * 2.0 ** -24)
    yield "f16_subnormal_operands", sub, h16(g(*sh) * 2.0 ** 14), g(npb, 128, 128), 1
    yield "f16_large", h16(rng.uniform(1, 2, sh) * 2.0 ** 15), h16(rng.uniform(-2, 2, sh) * 2.0 ** 15), \
        g(npb, 128, 128) * 2.0 ** 30, 1


def chain_cases16(rng, npb):
    """The f16 kernel's chain at f = 36 (K padded to 80: 5 MMAs per group), operands scaled
    so the row / group maximum sits in [2^14, 2^15): S2 W1, S1 W2, then S1 W1."""
    sh = (npb, 5, 128, 16)
    for name, gen in (("f16_kernel_chain_gauss", lambda: rng.standard_normal(sh)),
                      ("f16_kernel_chain_positive", lambda: rng.uniform(0.5, 1.0, sh))):
        s, w = gen().astype(np.float32) * 2.0 ** 12, gen().astype(np.float32) * 2.0 ** 12
        s[:, 4, :, 8:] = 0                       # K = 72 of 80
        w[:, 4, :, 8:] = 0
        s1, w1 = tf32(s), tf32(w)
        s2, w2 = h16(tf32(s - s1)), h16(tf32(w - w1))
        s1, w1 = h16(s1), h16(w1)
        A = np.concatenate([s2, s1, s1], axis=1)
        B = np.concatenate([w1, w2, w1], axis=1)
        yield name, A, B, np.zeros((npb, 128, 128)), 0


def subnormal_checks(L):
    out = {}
    A = np.zeros((1, 1, 128, 8), np.float32)
    B = np.zeros((1, 1, 128, 8), np.float32)
    C = np.zeros((1, 128, 128), np.float32)
    # subnormal input times 1: tf32-representable subnormal 2^-130 * 1.5
    A[..., 0] = np.float32(1.5 * 2.0 ** -130)
    B[..., 0] = 1.0
    D = run(L, A, B, C, 0)
    out["subnormal_input_x1"] = {"want": float(np.float32(1.5 * 2.0 ** -130)), "got": float(D[0, 0, 0])}
    # normal x normal with a subnormal product
    A[..., 0] = np.float32(2.0 ** -70)
    B[..., 0] = np.float32(2.0 ** -70)
    D = run(L, A, B, C, 0)
    out["subnormal_product"] = {"want": 2.0 ** -140, "got": float(D[0, 0, 0])}
    # subnormal accumulator plus zero products
    A[..., 0] = 0
    C[:] = np.float32(3 * 2.0 ** -140)
    D = run(L, A, B, C, 1)
    out["subnormal_accumulator"] = {"want": float(np.float32(3 * 2.0 ** -140)), "got": float(D[0, 0, 0])}
    # normal + product -> subnormal result by cancellation
    A[..., 0] = np.float32(2.0 ** -60)
    B[..., 0] = np.float32(-(2.0 ** -63) * (1 + 2.0 ** -10))
    C[:] = np.float32(2.0 ** -123)
    D = run(L, A, B, C, 1)
    out["cancellation_to_subnormal"] = {"want": float(2.0 ** -123 - 2.0 ** -123 * (1 + 2.0 ** -10)),
                                        "got": float(D[0, 0, 0])}
    # huge: products near FLT_MAX
    A[..., 0] = np.float32(2.0 ** 64)
    B[..., 0] = np.float32(2.0 ** 63)
    C[:] = 0
    D = run(L, A, B, C, 1)
    out["product_2^127"] = {"want": 2.0 ** 127, "got": float(D[0, 0, 0])}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--np", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--save", default="", help="npz of every case's A, B, C, D (model fitting)")
    ap.add_argument("--kind", default="tf32", choices=["tf32", "f16"])
    args = ap.parse_args()
    L = lib()
    rng = np.random.default_rng(args.seed)
    res = {}
    raw = {}
    kind = 1 if args.kind == "f16" else 0
    gen = (list(cases16(rng, args.np)) + list(chain_cases16(rng, max(4, args.np // 4)))) if kind else \
        (list(cases(rng, args.np)) + list(chain_cases(rng, max(4, args.np // 4))))
    for name, A, B, C, cm in gen:
        A, B = (h16(A), h16(B)) if kind else (tf32(A), tf32(B))
        C = np.asarray(C, np.float32)
        D = run(L, A, B, C, cm, kind)
        if args.save:
            raw.update({f"{name}/A": A, f"{name}/B": B, f"{name}/C": C, f"{name}/D": D,
                        f"{name}/cmode": np.int32(cm)})
        ex, absum, amax = exact(A, B, C, cm)
        res[name] = stats(D, ex, absum, amax, A.shape[1])
        print(name, json.dumps(res[name]), flush=True)
    if not kind:
        res["subnormals"] = subnormal_checks(L)
        print("subnormals", json.dumps(res["subnormals"]))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)
    if args.save:
        np.savez_compressed(args.save, **raw)


if __name__ == "__main__":
    main()
