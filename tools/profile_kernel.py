#!/usr/bin/env python3
"""Small driver for ncu captures: one workload, a few bf_apply calls.

    python tools/profile_kernel.py --config c4 --blocks 131072 --reps 3

Runs the same kernel instantiation and launch shape (grid = SMs x resident
CTAs) as bench.py on a prefix of the workload, so `ncu --set full` replays a
launch that fits the replay buffers.  Prints the per-block algorithmic bytes and
FLOPs so the captured dram bytes can be compared per block.
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
    ap.add_argument("--config", default="c4")
    ap.add_argument("--f", type=int, default=36)
    ap.add_argument("--blocks", type=int, default=131072)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--layout", default="interleaved")
    ap.add_argument("--variant", default="auto")
    a = ap.parse_args()
    wl = syn.workload("c3", a.f) if a.config == "c3" else syn.workload(a.config)
    dev = torch.device("cuda", 0)
    n = min(a.blocks, wl.n_blocks)
    planar = a.layout == "planar"
    S, tags = sync.workload_device(wl, dev, n=n, planar=planar)
    W = syn.precoders(wl.seed, wl.sub, wl.n_groups, wl.n_ant, wl.f, wl.w_norm)
    plan = bf.Plan(f=wl.f, layout=a.layout, variant=a.variant)
    plan.set_precoders(torch.from_numpy(syn.to_planar(W) if planar else W).to(dev))
    R = torch.empty(plan.r_shape(n), dtype=plan.dtype, device=dev)
    for _ in range(a.reps):
        plan.apply(S, tags, out=R)
    torch.cuda.synchronize()
    print(json.dumps({"workload": wl.name, "blocks": n, "layout": a.layout,
                      "bytes_per_block": wl.block_bytes, "flops_per_block": wl.block_flops,
                      "variant": plan.variant.name, "kernel": plan.kernel_config(n)}))


if __name__ == "__main__":
    main()
