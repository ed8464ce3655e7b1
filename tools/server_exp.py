#!/usr/bin/env python3
"""Slot-server latency against the slot size (not part of the product): device time per
slot (bf_server_slot_time) for n blocks, so latency = fixed + per-tile cost can be read
off.  f = 36, one W, 16 S / R buffers in rotation (cold L2).

    python tools/server_exp.py [--slots 100]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bf_synth as syn  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slots", type=int, default=100)
    ap.add_argument("--f", type=int, default=36)
    ap.add_argument("--per-cta", action="store_true", help="per-CTA start / count (BFTC_SRV_TRACE build)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    f = a.f
    W = syn.precoders(1, 0, 1, 64, f, "unit_columns")
    plan = bf.Plan(f=f, variant=bf.Variant.TENSOR)
    plan.set_precoders(torch.from_numpy(W).to(dev))
    sizes = [1, 148, 296, 592, 770, 1184, 2368, 4736]
    nbuf = 16
    bufs = {}
    for n in sizes:
        S = torch.from_numpy(syn.qam_symbols(1, 0, np.arange(n), f, 60, 64)).to(dev)
        bufs[n] = [(S.clone(), torch.empty((n, 64, 60), dtype=torch.complex64, device=dev)) for _ in range(nbuf)]
    torch.cuda.synchronize()
    srv = bf.Server(plan).start(torch.cuda.Stream(dev))
    try:
        for n in sizes:
            d, tr = [], []
            for i in range(10 + a.slots):
                S, R = bufs[n][i % nbuf]
                t = srv.submit(S, R)
                srv.wait(t, timeout_s=30)
                if i >= 10:
                    d.append(srv.slot_time_us(t))
                    tr.append(srv.trace_us(per_cta=a.per_cta))
            tiles = (n + 1) // 2
            if a.per_cta:
                seen = [statistics.median(x[8 + c] for x in tr) for c in range(148)]
                done = [statistics.median(x[168 + c] for x in tr) for c in range(148)]
                print(json.dumps({"n": n, "cta_seen_us": [round(v, 2) for v in seen],
                                  "cta_done_us": [round(v, 2) for v in done]}), flush=True)
            print(json.dumps({"n": n, "tiles_per_cta": tiles / 148, "device_us_median": statistics.median(d),
                              "device_us_min": min(d), "bytes_us_at_6.5TBps": n * 48000 / 6.5e6,
                              "cta0_trace_us_median": [statistics.median(x[j] for x in tr) for j in range(7)]}),
                  flush=True)
    finally:
        srv.close()


if __name__ == "__main__":
    main()
