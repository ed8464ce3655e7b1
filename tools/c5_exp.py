#!/usr/bin/env python3
"""Scheduling experiments for the c5 streaming config (not part of the product).

    python tools/c5_exp.py --chunks 512 --mode cells|full [--cells 0,1,..] [--inline-route]

mode "cells": cell k's chunks on stream k with an SM share proportional to 64 + f_k;
mode "full" : every chunk on the full grid, chunk c on stream c % 2 (the old bench).
Prints the CUDA-graph step time, the sum of per-kernel times of one eager step and the
mixed-f HBM roofline time of the same chunks.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import benchkit  # noqa: E402
import bf_synth as syn  # noqa: E402
import bf_synth.cuda as sync  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=512)
    ap.add_argument("--mode", default="cells")
    ap.add_argument("--cells", default="")
    ap.add_argument("--inline-route", action="store_true")
    ap.add_argument("--route-sms", type=int, default=2)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--full-share", type=int, default=0, help="mode full: SM share of every plan")
    ap.add_argument("--no-route", action="store_true", help="untagged applies (group 0)")
    ap.add_argument("--pslots", type=int, default=0, help="deep perm ring on one route stream")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    wl = syn.workload("c5")
    fc = syn.cell_flows(wl.seed, 8)
    cells = [int(x) for x in a.cells.split(",")] if a.cells else list(range(8))
    chunks = [c for c in range(a.chunks) if c % 8 in cells]
    plans = {}
    for k in cells:
        pl = bf.Plan(f=int(fc[k]))
        pl.set_precoders(torch.from_numpy(syn.precoders(wl.seed, k, 55, 64, int(fc[k]), "none")).to(dev))
        plans[k] = pl
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    if a.mode == "cells":
        w = np.array([64.0 + fc[k] for k in cells])
        avail = sms - a.route_sms
        sh = np.maximum(1, np.floor(w / w.sum() * avail)).astype(int)
        while sh.sum() < avail:
            sh[np.argmax(w / w.sum() * avail - sh)] += 1
        for k, s in zip(cells, sh):
            plans[k].set_sm_share(int(s))
    elif a.full_share:
        for pl in plans.values():
            pl.set_sm_share(a.full_share)
    S, T, P, O, R = {}, {}, {}, {}, {}
    for c in chunks:
        f = int(fc[c % 8])
        S[c] = torch.empty((4096, f, 60), dtype=torch.complex64, device=dev)
        sync.gen_symbols(S[c], wl.seed, 0, f, 60, 0, first=c * 4096)
        T[c] = torch.empty(4096, dtype=torch.int32, device=dev)
        sync.gen_tags(T[c], wl.seed, 55, first=c * 4096)
    nstr = len(cells) if a.mode == "cells" else 2
    for i in range(nstr):
        for s in range(2):
            P[i, s] = torch.empty(4096, dtype=torch.int32, device=dev)
            O[i, s] = torch.empty(57, dtype=torch.int32, device=dev)
            R[i, s] = torch.empty((4096, 64, 60), dtype=torch.complex64, device=dev)
    PS = a.pslots
    PP = [torch.empty(4096, dtype=torch.int32, device=dev) for _ in range(PS)]
    PO = [torch.empty(57, dtype=torch.int32, device=dev) for _ in range(PS)]
    ev_prt = [torch.cuda.Event() for _ in range(PS)]
    ev_puse = [torch.cuda.Event() for _ in range(PS)]
    a_st = [torch.cuda.Stream() for _ in range(nstr)]
    r_st = [torch.cuda.Stream() for _ in range(nstr)]
    ev_rt = {(i, s): torch.cuda.Event() for i in range(nstr) for s in range(2)}
    ev_use = {(i, s): torch.cuda.Event() for i in range(nstr) for s in range(2)}
    fork = torch.cuda.Event()
    joins = [torch.cuda.Event() for _ in range(2 * nstr)]
    state = {"main": torch.cuda.current_stream()}

    def step():
        main = state["main"]
        fork.record(main)
        for st in a_st + r_st:
            st.wait_event(fork)
        for i in range(nstr):
            for s in range(2):
                ev_use[i, s].record(a_st[i])
        for q in range(PS):
            ev_puse[q].record(main)
        for j, c in enumerate(chunks):
            k = c % 8
            i = cells.index(k) if a.mode == "cells" else j % 2
            s = (j // nstr) % 2
            pl = plans[k]
            if PS:
                q = j % PS
                r_st[0].wait_event(ev_puse[q])
                pl.route_into(T[c], PP[q], PO[q], stream=r_st[0])
                ev_prt[q].record(r_st[0])
                a_st[i].wait_event(ev_prt[q])
                pl.apply_routed(S[c], PP[q], PO[q], out=R[i, s], stream=a_st[i])
                ev_puse[q].record(a_st[i])
            elif a.no_route:
                pl.apply_routed(S[c], None, None, out=R[i, s], stream=a_st[i])
            elif a.inline_route:
                pl.route_into(T[c], P[i, s], O[i, s], stream=a_st[i])
                pl.apply_routed(S[c], P[i, s], O[i, s], out=R[i, s], stream=a_st[i])
            else:
                r_st[i].wait_event(ev_use[i, s])
                pl.route_into(T[c], P[i, s], O[i, s], stream=r_st[i])
                ev_rt[i, s].record(r_st[i])
                a_st[i].wait_event(ev_rt[i, s])
                pl.apply_routed(S[c], P[i, s], O[i, s], out=R[i, s], stream=a_st[i])
                ev_use[i, s].record(a_st[i])
        for n_, st in enumerate(a_st + r_st):
            joins[n_].record(st)
            main.wait_event(joins[n_])

    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        state["main"] = torch.cuda.current_stream()
        step()
    state["main"] = torch.cuda.current_stream()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = benchkit.ClockSampler(0, period_ms=50).start()
    e0.record()
    for _ in range(a.reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    c_ = clk.stop()
    ms = e0.elapsed_time(e1) / a.reps
    for pl in plans.values():
        pl.set_profiling(True)
        pl.kernel_time()
    step()
    torch.cuda.synchronize()
    per_cell = {k: plans[k].kernel_time() for k in cells}
    byt = sum(4096 * 480 * (64 + int(fc[c % 8])) for c in chunks)
    hbm = benchkit.measured_peaks()["hbm_gbs"]
    print(json.dumps({"mode": a.mode, "cells": cells, "chunks": len(chunks),
                      "inline_route": a.inline_route, "no_route": a.no_route,
                      "graph_ms": ms, "roof_ms": byt / hbm / 1e6, "frac": byt / hbm / 1e6 / ms,
                      "per_cell_kernel_ms": {k: round(v[0], 3) for k, v in per_cell.items()},
                      "per_kernel_us": {k: round(1e3 * v[0] / max(v[1], 1), 1) for k, v in per_cell.items()},
                      "clocks": c_}), flush=True)


if __name__ == "__main__":
    main()
