#!/usr/bin/env python3
"""Randomised cross-check of the tensor kernel against the FFMA kernel (both libbf.so, both
on the GPU): random f, layout, block count, group count, SM share, tags (a few out of
range), CUDA streams — so every shared-memory configuration, ragged tiles, single-W-buffer
reloads and the staged / direct epilogues meet many shapes the fixed tests do not.

    python tools/stress_tc.py [--trials 200] [--seed 1]

Per trial: fp32 layouts must agree within 2e-5 * T (T = sum |w||s|, both kernels are
inside 1e-5 * T of the exact result), blocks with invalid tags must be left untouched by
both, and the 16-bit layouts must equal the tensor kernel's own fp32 result rounded (fp16
RN; int16 sat(rne(R * 2^12))).  Then random bf_apply_batch job lists (any f, one layout,
tagged or not) against the jobs' own apply_routed calls, bitwise.  Not a test of the oracle
(tests/ does that); a bug hunt.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1810_11451_b200 import Layout, Plan, Variant  # noqa: E402

DEV = torch.device("cuda", 0)
SENT = -12345.0


def run(layout, variant, f, W, S, tags, share, R0):
    p = Plan(f=f, layout=layout, variant=variant)
    if share:
        p.set_sm_share(share)
    p.set_precoders(W)
    R = R0.clone()
    p.apply(S, tags, out=R)
    torch.cuda.synchronize()
    p.close()
    return R


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    torch.manual_seed(a.seed)             # (the Gaussian inputs come from torch's generator)
    t0 = time.time()
    bad = 0
    for trial in range(a.trials):
        f = int(rng.integers(1, 37))
        n = int(rng.choice([1, 2, 3, 7, 64, 299, 1000, 4097, 20000]))
        G = int(rng.choice([1, 2, 13, 55, 300]))
        share = int(rng.choice([0, 0, 1, 2, 7, 100]))
        W = (torch.randn(G, 64, f, dtype=torch.complex64, device=DEV) / f ** 0.5)
        S = torch.randn(n, f, 60, dtype=torch.complex64, device=DEV)
        tags = torch.from_numpy(rng.integers(0, G, n).astype(np.int32)).to(DEV)
        n_bad = int(rng.integers(0, 3)) if n > 4 else 0
        bad_idx = rng.choice(n, n_bad, replace=False) if n_bad else np.zeros(0, np.int64)
        if n_bad:
            tags[torch.from_numpy(bad_idx).to(DEV)] = G + 5
        valid = torch.ones(n, dtype=torch.bool, device=DEV)
        valid[torch.from_numpy(bad_idx).to(DEV)] = False
        # fp32 interleaved: tensor vs FFMA
        R0 = torch.full((n, 64, 60), complex(SENT, SENT), dtype=torch.complex64, device=DEV)
        Rt = run(Layout.INTERLEAVED, Variant.TENSOR, f, W, S, tags, share, R0)
        Rf = run(Layout.INTERLEAVED, Variant.FFMA, f, W, S, tags, 0, R0)
        T = torch.einsum("gik,nkj->nij", W.abs().double(), S.abs().double()) if G == 1 else \
            torch.einsum("nik,nkj->nij", W.abs().double()[tags.long().clamp(max=G - 1)], S.abs().double())
        err = (Rt.to(torch.complex128) - Rf.to(torch.complex128)).abs()
        ok = bool((err[valid] <= 2e-5 * T[valid] + 1e-30).all())
        untouched = bool((Rt[~valid] == complex(SENT, SENT)).all() and (Rf[~valid] == complex(SENT, SENT)).all())
        # planar: the same numbers (tensor), bitwise, after the layout change
        Sp = torch.stack([S.real, S.imag], 1).contiguous()
        Wp = torch.stack([W.real, W.imag], 1).contiguous()
        Rp0 = torch.full((n, 2, 64, 60), SENT, dtype=torch.float32, device=DEV)
        Rp = run(Layout.PLANAR, Variant.TENSOR, f, Wp, Sp, tags, share, Rp0)
        planar_eq = bool(torch.equal(torch.complex(Rp[:, 0], Rp[:, 1])[valid], Rt[valid]))
        # 16-bit outputs vs the tensor fp32 result
        R16 = run(Layout.INTERLEAVED_F16OUT, Variant.TENSOR, f, W, S, tags, share,
                  torch.zeros((n, 64, 60, 2), dtype=torch.float16, device=DEV))
        exp16 = torch.stack([Rt.real, Rt.imag], -1).half()
        f16_eq = bool(torch.equal(R16[valid], exp16[valid]))
        Ri = run(Layout.INTERLEAVED_I16OUT, Variant.TENSOR, f, W, S, tags, share,
                 torch.zeros((n, 64, 60, 2), dtype=torch.int16, device=DEV))
        x = torch.stack([Rt.real, Rt.imag], -1).double() * 4096.0
        expi = torch.round(x).clamp(-32768, 32767).to(torch.int16)   # torch.round: half to even
        i16_eq = bool(torch.equal(Ri[valid], expi[valid]))
        good = ok and untouched and planar_eq and f16_eq and i16_eq
        if not good:
            bad += 1
        print(json.dumps({"trial": trial, "f": f, "n": n, "G": G, "share": share, "bad_tags": n_bad,
                          "max_err_over_T": float((err[valid] / (T[valid] + 1e-30)).max()) if n_bad < n else 0.0,
                          "ok": ok, "untouched": untouched, "planar_eq": planar_eq, "f16_eq": f16_eq,
                          "i16_eq": i16_eq}), flush=True)
    # bf_apply_batch: random job lists (any f, one layout, some untagged) must equal the
    # jobs' own apply_routed calls on the tensor kernel, bitwise
    from paper_1810_11451_b200 import apply_batch
    bbad = 0
    for trial in range(a.trials // 4):
        layout = [Layout.INTERLEAVED, Layout.PLANAR, Layout.INTERLEAVED_F16OUT,
                  Layout.INTERLEAVED_I16OUT][int(rng.integers(0, 4))]
        jobs, refs, keep = [], [], []
        for _ in range(int(rng.integers(1, 17))):
            f = int(rng.integers(1, 37))
            n = int(rng.choice([1, 3, 64, 777, 4096]))
            G = int(rng.choice([1, 7, 55]))
            p = Plan(f=f, layout=layout, variant=Variant.AUTO)
            Wc = torch.randn(G, 64, f, dtype=torch.complex64, device=DEV) / f ** 0.5
            Sc = torch.randn(n, f, 60, dtype=torch.complex64, device=DEV)
            if layout == Layout.PLANAR:
                Wc = torch.stack([Wc.real, Wc.imag], 1).contiguous()
                Sc = torch.stack([Sc.real, Sc.imag], 1).contiguous()
            p.set_precoders(Wc)
            if rng.random() < 0.3:
                perm = offs = None
            else:
                tags = torch.from_numpy(rng.integers(0, G, n).astype(np.int32)).to(DEV)
                perm, offs = p.route(tags)
            out = torch.zeros(p.r_shape(n), dtype=p.r_dtype, device=DEV)
            jobs.append((p, Sc, perm, offs, out))
            # the contract (bf.h): bitwise equal to the job's apply_routed with the tensor
            # variant — or, for an AUTO plan whose precoders leave the tensor domain (which
            # bf_apply_batch runs on its own, i.e. FFMA), to the plan's own apply_routed
            q = Plan(f=f, layout=layout, variant=Variant.TENSOR)
            q.set_precoders(Wc)
            ref_t = torch.zeros_like(out)
            q.apply_routed(Sc, perm, offs, out=ref_t)
            ref_o = torch.zeros_like(out)
            p.apply_routed(Sc, perm, offs, out=ref_o)
            refs.append((ref_t, ref_o))
            keep += [p, q]
        apply_batch(jobs)
        torch.cuda.synchronize()
        eq = all(torch.equal(j[4], r[0]) or torch.equal(j[4], r[1]) for j, r in zip(jobs, refs))
        bbad += 0 if eq else 1
        diff = []
        if not eq:                      # which jobs, blocks and how far
            for ji, (j, rr) in enumerate(zip(jobs, refs)):
                r = rr[0]
                if not (torch.equal(j[4], rr[0]) or torch.equal(j[4], rr[1])):
                    a32 = j[4].float() if j[4].dtype != torch.complex64 else torch.view_as_real(j[4])
                    b32 = r.float() if r.dtype != torch.complex64 else torch.view_as_real(r)
                    d = (a32 - b32).abs().reshape(a32.shape[0], -1)
                    blocks = torch.nonzero(d.amax(1) > 0).flatten().tolist()
                    diff.append({"job": ji, "f": j[0].f, "n": int(a32.shape[0]), "tagged": j[2] is not None,
                                 "blocks": blocks[:8], "n_blocks": len(blocks), "max_abs": float(d.max())})
        print(json.dumps({"batch_trial": trial, "layout": layout.name, "jobs": len(jobs),
                          "f": [j[0].f for j in jobs], "equal": eq, "diff": diff}), flush=True)
        for p in keep:
            p.close()
    print(json.dumps({"trials": a.trials, "failed": bad, "batch_trials": a.trials // 4,
                      "batch_failed": bbad, "seconds": time.time() - t0}))
    return 1 if bad or bbad else 0


if __name__ == "__main__":
    sys.exit(main())
