#!/usr/bin/env python3
"""Experiment: effect of the block order produced by routing on the tensor kernel.

Same S, same 55 precoders, 2^20 blocks at f = 36; tags (a) uniformly random
(config c4), (b) already sorted (block i -> group 55 i / n), (c) untagged.
Prints kernel ms and HBM GB/s for each.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bf_synth as syn  # noqa: E402
import bf_synth.cuda as sync  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402


def timeit(plan, S, tags, R, reps=10):
    for _ in range(3):
        plan.apply(S, tags, out=R)
    torch.cuda.synchronize()
    plan.set_profiling(True)
    plan.kernel_time()
    for _ in range(reps):
        plan.apply(S, tags, out=R)
    ms, n = plan.kernel_time()
    plan.set_profiling(False)
    return ms / n


def main():
    dev = torch.device("cuda", 0)
    wl = syn.workload("c4")
    n = int(sys.argv[1]) if len(sys.argv) > 1 else wl.n_blocks
    S, tags = sync.workload_device(wl, dev, n=n)
    W = syn.precoders(wl.seed, wl.sub, wl.n_groups, 64, 36, wl.w_norm)
    R = torch.empty((n, 64, 60), dtype=torch.complex64, device=dev)
    sorted_tags = (torch.arange(n, device=dev, dtype=torch.int64) * 55 // n).to(torch.int32)
    for variant in ("tensor", "ffma"):
        plan = bf.Plan(f=36, variant=variant)
        plan.set_precoders(torch.from_numpy(W).to(dev))
        for name, t in (("random", tags), ("sorted", sorted_tags), ("untagged", None)):
            ms = timeit(plan, S, t, R)
            print(json.dumps({"variant": variant, "order": name, "blocks": n, "kernel_ms": ms,
                              "GBps": wl.block_bytes * n / ms / 1e6}), flush=True)
        plan.close()


if __name__ == "__main__":
    main()
