#!/usr/bin/env python3
"""Cost of group routing inside short launches (not part of the product).

Back-to-back bf_apply_routed launches on one stream over one 4096-block chunk at
f = 32, with the blocks routed into G groups (G = 1 is the untagged layout with a
routing pass), timed with CUDA events; prints us per launch and GB/s.

    python tools/route_cost.py [--f 32] [--n 4096] [--reps 200]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bf_synth as syn  # noqa: E402
import bf_synth.cuda as sync  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--f", type=int, default=32)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--only", default="", help="G:tags, e.g. 300:random (one config, for ncu)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    f, n = a.f, a.n
    S = torch.empty((n, f, 60), dtype=torch.complex64, device=dev)
    sync.gen_symbols(S, 4, 0, f, 60, 0, first=0)
    R = torch.empty((n, 64, 60), dtype=torch.complex64, device=dev)
    cases = [(1, "untagged"), (1, "one-group"), (8, "random"), (55, "random"),
             (55, "sorted-input"), (300, "random")]
    if a.only:
        cases = [(int(a.only.split(":")[0]), a.only.split(":")[1])]
    for G, tagmode in cases:
        W = syn.precoders(4, 0, G, 64, f, "none")
        plan = bf.Plan(f=f)
        plan.set_precoders(torch.from_numpy(W).to(dev))
        tags = syn.subband_tags(4, np.arange(n), G)
        if tagmode == "one-group":
            tags[:] = 0
        if tagmode == "sorted-input":
            tags = np.sort(tags)
        td = torch.from_numpy(tags.astype(np.int32)).to(dev)
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        offs = torch.empty(G + 2, dtype=torch.int32, device=dev)
        if tagmode != "untagged":
            plan.route_into(td, perm, offs)
        args = (None, None) if tagmode == "untagged" else (perm, offs)
        for share in (148, 146):
            plan.set_sm_share(share)
            for _ in range(10):
                plan.apply_routed(S, *args, out=R)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                plan.apply_routed(S, *args, out=R)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / a.reps
            print(json.dumps({"G": G, "tags": tagmode, "share": share, "us_per_launch": round(us, 2),
                              "GBps": round(n * 480 * (64 + f) / us / 1e3, 1)}), flush=True)
        # the routing kernel alone
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            plan.route_into(td, perm, offs)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"G": G, "tags": tagmode, "route_us": round(e0.elapsed_time(e1) * 1e3 / a.reps, 2)}),
              flush=True)
        plan.close()


if __name__ == "__main__":
    main()
