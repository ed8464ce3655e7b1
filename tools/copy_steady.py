#!/usr/bin/env python3
"""Sustained copy bandwidth under the board's power cap (not part of the product): the
denominator context for the steady-state and power-capped bench lines.  Back-to-back
D2D copies (torch copy_, read + write bytes) for --seconds with nvidia-smi sampling; the
write share can be raised with extra memsets (c5 writes ~78 % of its bytes).

    python tools/copy_steady.py [--seconds 10] [--gib 4] [--write-extra 0]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=10.0)
    ap.add_argument("--gib", type=float, default=4.0)
    ap.add_argument("--write-extra", type=float, default=0.0, help="a second copy, this fraction of the first")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = int(a.gib * (1 << 30)) // 4
    # random bits: the power drawn depends on the data (constant data toggles almost no bits)
    src = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device=dev).view(torch.float32)
    dst = torch.empty_like(src)
    ne = max(1, int(n * a.write_extra))
    extra = torch.empty(ne, dtype=torch.float32, device=dev)
    esrc = torch.randint(-2**31, 2**31 - 1, (ne,), dtype=torch.int32, device=dev).view(torch.float32)
    per = 8 * n + 8 * ne * (a.write_extra > 0)
    for _ in range(3):
        dst.copy_(src)
    torch.cuda.synchronize()
    mon = benchkit.ClockSampler(0, period_ms=50).start()
    rates = []
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < a.seconds:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            dst.copy_(src)
            if a.write_extra > 0:
                extra.copy_(esrc)
        e1.record()
        torch.cuda.synchronize()
        rates.append(4 * per / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    c = mon.stop()
    hbm = benchkit.measured_peaks()["hbm_gbs"]
    first, settled = rates[0], sorted(rates[len(rates) // 2:])[len(rates) // 4]
    print(json.dumps({"write_extra": a.write_extra, "first_gbs": round(first, 1), "settled_gbs": round(settled, 1),
                      "settled_frac_of_burst_peak": round(settled / hbm, 4), "sm_mhz": c.get("sm_mhz"),
                      "power_w_median": c.get("power_w_median"), "reasons": c.get("reasons")}), flush=True)


if __name__ == "__main__":
    main()
