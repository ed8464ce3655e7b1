#!/usr/bin/env python3
"""Runtime-f batch kernel (bf_apply_batch, one job) against the per-f kernel (bf_apply) on
the same untagged blocks, per f (not part of the product): isolates what the runtime-f
form costs (f = 36 shared-memory sizing: 2-stage S ring, one W buffer)."""
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
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--f", type=int, nargs="*", default=[5, 7, 15, 19, 24, 32, 35])
    ap.add_argument("--modes", nargs="*", default=["per_f", "batch"])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--repeat", type=int, default=1, help="timings per mode (noise check)")
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
        res = {"f": f}
        for mode in [m for _ in range(a.repeat) for m in a.modes]:
            run = (lambda: p.apply(S, out=R)) if mode == "per_f" else \
                (lambda: bf.apply_batch([(p, S, None, None, R)]))
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            frac = n * 480 * (f + 64) / (ms * 1e-3) / 1e9 / hbm
            if a.repeat > 1:
                res.setdefault(mode + "_frac", []).append(round(frac, 4))
            else:
                res[mode + "_frac"] = frac
        print(json.dumps(res), flush=True)
        p.close()


if __name__ == "__main__":
    main()
