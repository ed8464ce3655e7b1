#!/usr/bin/env python3
"""Sustained (power-capped) throughput of the per-f kernel (bf_apply) against the runtime-f
batch kernel (bf_apply_batch, one job) on the same untagged blocks (not part of the
product): each mode runs back to back for --seconds with nvidia-smi sampling of SM clock
and power, after a cool-down, so the two are compared at the clocks the power cap leaves.

    python tools/sustained_exp.py [--f 35] [--seconds 6] [--modes per_f batch]
"""
import argparse
import json
import os
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
    ap.add_argument("--f", type=int, nargs="*", default=[35])
    ap.add_argument("--modes", nargs="*", default=["per_f", "batch"])
    ap.add_argument("--seconds", type=float, default=6.0)
    ap.add_argument("--cool", type=float, default=15.0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    hbm = benchkit.measured_peaks()["hbm_gbs"]
    n = 65536
    for f in a.f:
        W = syn.precoders(1, f, 1, 64, f, "none")
        p = bf.Plan(f=f, variant=bf.Variant.TENSOR)
        p.set_precoders(torch.from_numpy(W).to(dev))
        S = torch.empty((n, f, 60), dtype=torch.complex64, device=dev)
        sync.gen_symbols(S, 1, 0, f, 60, 64, first=0)
        R = torch.empty((n, 64, 60), dtype=torch.complex64, device=dev)
        for mode in a.modes:
            run = (lambda: p.apply(S, out=R)) if mode == "per_f" else \
                (lambda: bf.apply_batch([(p, S, None, None, R)]))
            time.sleep(a.cool)
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            mon = benchkit.ClockSampler().start()
            fr = []
            t_end = time.perf_counter() + a.seconds
            while time.perf_counter() < t_end:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    run()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 20
                fr.append(n * 480 * (f + 64) / (ms * 1e-3) / 1e9 / hbm)
            clk = mon.stop()
            fr_s = sorted(fr[len(fr) // 2:])           # second half: settled under the cap
            print(json.dumps({"f": f, "mode": mode, "first": round(fr[0], 4),
                              "settled_median": round(fr_s[len(fr_s) // 2], 4), "n": len(fr),
                              "sm_mhz": clk.get("sm_mhz"), "power_w_median": clk.get("power_w_median"),
                              "reasons": clk.get("reasons")}), flush=True)
        p.close()


if __name__ == "__main__":
    main()
