#!/usr/bin/env python3
"""Where the c5 batch kernel loses time (not part of the product): one bf_apply_batch
launch over a window of 8 chunks (one per cell, BASELINE.json configs[4]), timed with CUDA
events over many windows, with the chunks' real tags, with every tag 0 (one group per
chunk: no group changes inside a job), and untagged (no routing arrays at all).

    python tools/batch_exp.py [--windows 16] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import benchkit  # noqa: E402
import bf_synth as syn  # noqa: E402
import bf_synth.cuda as sync  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--windows", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--share", type=int, default=0)
    ap.add_argument("--per-launch", type=int, default=8, help="chunks per bf_apply_batch launch (<= 16)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    wl = syn.workload("c5")
    fc = syn.cell_flows(wl.seed, 8)
    plans = []
    for cell in range(8):
        pl = bf.Plan(f=int(fc[cell]))
        pl.set_precoders(torch.from_numpy(syn.precoders(wl.seed, cell, 55, 64, int(fc[cell]), "none")).to(dev))
        if a.share:
            pl.set_sm_share(a.share)
        plans.append(pl)
    wins = []
    nbytes = 0
    B = a.per_launch
    for w in range(a.windows * 8 // B):
        jobs = {"tagged": [], "one_group": [], "untagged": []}
        for c in range(B * w, B * w + B):
            f = int(fc[c % 8])
            S = torch.empty((4096, f, 60), dtype=torch.complex64, device=dev)
            sync.gen_symbols(S, wl.seed, 0, f, 60, 0, first=c * 4096)
            T = torch.empty(4096, dtype=torch.int32, device=dev)
            sync.gen_tags(T, wl.seed, 55, first=c * 4096)
            R = torch.empty((4096, 64, 60), dtype=torch.complex64, device=dev)
            perm, offs = plans[c % 8].route(T)
            perm0, offs0 = plans[c % 8].route(torch.zeros_like(T))
            jobs["tagged"].append((plans[c % 8], S, perm, offs, R))
            jobs["one_group"].append((plans[c % 8], S, perm0, offs0, R))
            jobs["untagged"].append((plans[c % 8], S, None, None, R))
            nbytes += 4096 * 480 * (64 + f)
        wins.append(jobs)
    torch.cuda.synchronize()
    hbm = benchkit.measured_peaks()["hbm_gbs"]
    for mode in ("tagged", "one_group", "untagged"):
        for w in wins:
            bf.apply_batch(w[mode])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            for w in wins:
                bf.apply_batch(w[mode])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(json.dumps({"mode": mode, "per_launch": B, "windows": a.windows, "us_per_window": 1e3 * ms / a.windows,
                          "GBps": nbytes / (ms * 1e-3) / 1e9, "frac": nbytes / (ms * 1e-3) / 1e9 / hbm}),
              flush=True)


if __name__ == "__main__":
    main()
