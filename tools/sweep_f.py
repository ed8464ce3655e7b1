#!/usr/bin/env python3
"""Per-f, per-variant kernel timing on config c3 (BASELINE.json configs[2]):
the data behind libbf's AUTO variant table.

    python tools/sweep_f.py [--blocks 100000] [--reps 10] [--layout interleaved]

Prints one JSON line per (f, variant): kernel ms (CUDA events inside libbf),
GB/s of algorithmic bytes, TFLOP/s of algorithmic FLOPs, fractions of the HBM
and derived FP32 peaks.
"""
import argparse
import dataclasses
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
    ap.add_argument("--blocks", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--layout", default="interleaved")
    ap.add_argument("--flows", default=",".join(str(f) for f in syn.C3_FLOWS))
    ap.add_argument("--variants", default="ffma,tensor")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    peaks = benchkit.measured_peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    p32 = benchkit.fp32_peak_tflops(sms, peaks.get("sm_max_mhz", 1965.0))
    planar = a.layout == "planar"
    for f in [int(x) for x in a.flows.split(",")]:
        # off-sweep f (the AUTO table needs every f): c3's recipe with that f
        wl = syn.workload("c3", f) if f in syn.C3_FLOWS else \
            dataclasses.replace(syn.workload("c3", 1), name=f"c3like_f{f}", f=f, sub=f)
        n = min(a.blocks, wl.n_blocks)
        S, _ = sync.workload_device(wl, dev, n=n, planar=planar)
        W = syn.precoders(wl.seed, wl.sub, 1, 64, f, wl.w_norm)
        for variant in (a.variants.split(",") if f > 0 else ["auto"]):
            plan = bf.Plan(f=f, layout=a.layout, variant=variant)
            plan.set_precoders(torch.from_numpy(syn.to_planar(W) if planar else W).to(dev))
            R = torch.empty(plan.r_shape(n), dtype=plan.r_dtype, device=dev)
            for _ in range(3):
                plan.apply(S, out=R)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            plan.set_profiling(True)
            plan.kernel_time()
            e0.record()
            for _ in range(a.reps):
                plan.apply(S, out=R)
            e1.record()
            torch.cuda.synchronize()
            step_ms = e0.elapsed_time(e1) / a.reps
            kms, kn = plan.kernel_time()
            kern_ms = kms / kn if kn else step_ms
            r_blk = 15360 if a.layout in ("interleaved_f16out", "interleaved_i16out") else 30720
            gbs = (480 * f + r_blk) * n / (kern_ms * 1e-3) / 1e9
            tf = wl.block_flops * n / (kern_ms * 1e-3) / 1e12
            print(json.dumps({"f": f, "variant": variant, "layout": a.layout, "blocks": n,
                              "kernel_ms": kern_ms, "step_ms": step_ms, "GBps": gbs,
                              "hbm_frac": gbs / peaks["hbm_gbs"], "TFLOPs": tf,
                              "fp32_frac": tf / p32,
                              "Mblocks_per_s": n / (kern_ms * 1e-3) / 1e6}), flush=True)
            plan.close()
            del R
        del S
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
