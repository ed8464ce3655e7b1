"""Energy per MAC: cta_group::1 (M = 128) vs cta_group::2 (M = 256) MMAs, 4 s each."""
import ctypes, json, os, statistics, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: F401
import benchkit
H = os.path.dirname(os.path.abspath(__file__))
L1 = ctypes.CDLL(os.path.join(H, "libmmp.so"))
L2 = ctypes.CDLL(os.path.join(H, "libmmp2.so"))
for L, fn in ((L1, "mmp_run"), (L2, "mmp2_run")):
    getattr(L, fn).argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
iters = 20000
torch.zeros(1, device="cuda")
clk = benchkit.ClockSampler(0, period_ms=50).start(); time.sleep(2); idle = clk.stop()
idle_w = statistics.median([float(r[2]) for r in clk.rows])
print(json.dumps({"idle_w": idle_w}), flush=True)
for name, L, fn, kind, M, K in (("1sm tf32", L1, "mmp_run", 0, 128, 8), ("2sm tf32", L2, "mmp2_run", 0, 256, 8),
                                ("1sm bf16", L1, "mmp_run", 1, 128, 16), ("2sm bf16", L2, "mmp2_run", 1, 256, 16)):
    clk = benchkit.ClockSampler(0, period_ms=50).start()
    t0 = time.time(); mss = []
    while time.time() - t0 < 4.0:
        ms = ctypes.c_float()
        rc = getattr(L, fn)(kind, iters, 3, ctypes.byref(ms))
        assert rc == 0, rc
        mss.append(ms.value)
    c = clk.stop()
    pw = statistics.median([float(r[2]) for r in clk.rows[len(clk.rows) // 2:]])
    ms = statistics.median(mss[len(mss) // 2:])
    n_instr = (148 if M == 128 else 74) * iters * 9
    macs = n_instr * M * 128 * K
    print(json.dumps({"mode": name, "ms": ms, "TMAC_per_s": macs / (ms * 1e-3) / 1e12, "power_w": pw,
                      "pJ_per_kMAC_above_idle": (pw - idle_w) / (macs / (ms * 1e-3)) * 1e12 * 1e3,
                      "sm_mhz": c["sm_mhz"], "reasons": c["reasons"]}), flush=True)
