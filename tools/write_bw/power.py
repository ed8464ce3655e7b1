"""Steady-state power of the write-path micro-benchmarks (3 s each)."""
import ctypes, os, sys, json, time, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
import benchkit
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwbw.so"))
L.wbw_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
n = 1 << 20
R = torch.empty(n * 7680, device="cuda")
for mode, name, cps in [(0, "stg64-4w", 1), (5, "stg128shfl-4w", 1), (4, "stg64-8w", 1), (1, "stg128-seq", 1), (2, "bulk", 1), (3, "memset", 1)]:
    clk = benchkit.ClockSampler(0, period_ms=50).start()
    t0 = time.time(); mss = []
    while time.time() - t0 < 3.0:
        ms = ctypes.c_float()
        L.wbw_run(mode, R.data_ptr(), n, cps, 3, ctypes.byref(ms)); mss.append(ms.value)
    c = clk.stop()
    pw = [float(r[2]) for r in clk.rows[len(clk.rows) // 2:]]
    ms = statistics.median(mss[len(mss) // 2:])
    gbs = n * 30720 / ms / 1e6
    P = statistics.median(pw)
    print(json.dumps({"mode": name, "GBps": round(gbs), "power_w": round(P), "sm_mhz": c["sm_mhz"],
                      "pJ_per_byte_above_200W": round((P - 200) / (gbs * 1e9) * 1e12, 1)}), flush=True)
