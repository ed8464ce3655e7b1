"""Steady-state power of plain device copies (the HBM energy reference): idle floor,
cudaMemcpy D2D (50 % read / 50 % write) and a 36:64 read:write mix (two copies of
different sizes interleaved), 4 s each."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: E402

import benchkit  # noqa: E402


def sample(fn, secs=4.0):
    clk = benchkit.ClockSampler(0, period_ms=50).start()
    t0 = time.time()
    gbs = []
    while time.time() - t0 < secs:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        nbytes = fn()
        b.record()
        b.synchronize()
        gbs.append(nbytes / a.elapsed_time(b) / 1e6)
    c = clk.stop()
    pw = [float(r[2]) for r in clk.rows[len(clk.rows) // 2:]]
    return {"GBps": round(statistics.median(gbs[len(gbs) // 2:])) if gbs else None,
            "power_w": round(statistics.median(pw)), "sm_mhz": c["sm_mhz"], "reasons": c["reasons"]}


n = 4 << 30   # floats: 16 GB per buffer
src = torch.empty(n, device="cuda")
dst = torch.empty(n, device="cuda")
src.uniform_()
torch.cuda.synchronize()
print(json.dumps({"mode": "idle", **sample(lambda: (time.sleep(0.05), 0)[1] + 1, 3.0)}), flush=True)


def copy():
    for _ in range(4):
        dst.copy_(src)
    return 4 * 2 * n * 4


print(json.dumps({"mode": "d2d_copy", **sample(copy)}), flush=True)


def fill():
    for _ in range(4):
        dst.fill_(1.0)
    return 4 * n * 4


print(json.dumps({"mode": "fill", **sample(fill)}), flush=True)
