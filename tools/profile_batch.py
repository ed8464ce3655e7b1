#!/usr/bin/env python3
"""One c5 window (8 consecutive 4096-block chunks, one per cell) through bf_apply_batch,
a few times — for ncu captures of the batch kernel (bf_tc_kernel<0,0>).

    python tools/profile_batch.py [--window 0] [--reps 3] [--chunks 8]
Prints the window's algorithmic bytes so a capture's DRAM bytes can be compared.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bf_synth as syn  # noqa: E402
import bf_synth.cuda as sync  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--window", type=int, default=0)
    ap.add_argument("--chunks", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    wl = syn.workload("c5")
    fc = syn.cell_flows(wl.seed, 8)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    plans = []
    for cell in range(8):
        pl = bf.Plan(f=int(fc[cell]))
        pl.set_precoders(torch.from_numpy(syn.precoders(wl.seed, cell, 55, 64, int(fc[cell]), "none")).to(dev))
        pl.set_sm_share(sms - 2)
        plans.append(pl)
    jobs, nbytes = [], 0
    for c in range(a.window * a.chunks, (a.window + 1) * a.chunks):
        f = int(fc[c % 8])
        S = torch.empty((4096, f, 60), dtype=torch.complex64, device=dev)
        sync.gen_symbols(S, wl.seed, 0, f, 60, 0, first=c * 4096)
        T = torch.empty(4096, dtype=torch.int32, device=dev)
        sync.gen_tags(T, wl.seed, 55, first=c * 4096)
        perm, offs = plans[c % 8].route(T)
        jobs.append((plans[c % 8], S, perm, offs, torch.empty((4096, 64, 60), dtype=torch.complex64, device=dev)))
        nbytes += 4096 * 480 * (64 + f)
    for _ in range(a.reps):
        bf.apply_batch(jobs)
    torch.cuda.synchronize()
    print(json.dumps({"window": a.window, "chunks": a.chunks, "algorithmic_bytes": nbytes}))


if __name__ == "__main__":
    main()
