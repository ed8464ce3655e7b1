#!/usr/bin/env python3
"""Steady-state behaviour of one variant on config c4: back-to-back bf_apply calls
for a few seconds with nvidia-smi sampling (clock, power, throttle reasons).

    python tools/steady_state.py [--variant tensor] [--seconds 6]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import benchkit  # noqa: E402
import bf_synth as syn  # noqa: E402
import bf_synth.cuda as sync  # noqa: E402
import paper_1810_11451_b200 as bf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="tensor")
    ap.add_argument("--seconds", type=float, default=6.0)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--f", type=int, default=36)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    wl = syn.workload("c3", a.f) if a.config == "c3" else syn.workload(a.config)
    S, tags = sync.workload_device(wl, dev)
    W = syn.precoders(wl.seed, wl.sub, wl.n_groups, 64, wl.f, wl.w_norm)
    plan = bf.Plan(f=wl.f, variant=a.variant)
    plan.set_precoders(torch.from_numpy(W).to(dev))
    R = torch.empty(plan.r_shape(wl.n_blocks), dtype=plan.dtype, device=dev)
    for _ in range(3):
        plan.apply(S, tags, out=R)
    torch.cuda.synchronize()
    clk = benchkit.ClockSampler(0, period_ms=50).start()
    plan.set_profiling(True)
    t0 = time.time()
    times = []
    while time.time() - t0 < a.seconds:
        for _ in range(10):
            plan.apply(S, tags, out=R)
        ms, n = plan.kernel_time()
        times.append(ms / n)
    c = clk.stop()
    sms = [float(r[0]) for r in clk.rows if r[0].replace('.', '').isdigit()]
    pw = [float(r[2]) for r in clk.rows if r[2].replace('.', '').isdigit()]
    gbs = [wl.block_bytes * wl.n_blocks / t / 1e6 for t in times]
    print(json.dumps({"variant": a.variant, "workload": wl.name, "batches": len(times),
                      "kernel_ms_first": times[0], "kernel_ms_last": times[-1],
                      "kernel_ms_median": statistics.median(times),
                      "GBps_median": statistics.median(gbs), "GBps_max": max(gbs),
                      "sm_mhz_series": sms[::4], "power_series": pw[::4], "clocks": c}))


if __name__ == "__main__":
    main()
