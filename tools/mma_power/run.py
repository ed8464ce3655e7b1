"""Steady-state power per MMA kind (tools/mma_power/mma_power.cu), 4 s per mode."""
import ctypes, json, os, statistics, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: F401  (CUDA context)
import benchkit
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmmp.so"))
L.mmp_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
iters = 20000
names = {0: "tf32 K=8", 1: "bf16 K=16", 2: "fp16 K=16", 3: "tf32 K=8 zero A"}
for mode in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3").split(",")]:
    clk = benchkit.ClockSampler(0, period_ms=50).start()
    t0 = time.time(); mss = []
    while time.time() - t0 < 4.0:
        ms = ctypes.c_float()
        assert L.mmp_run(mode, iters, 3, ctypes.byref(ms)) == 0
        mss.append(ms.value)
    c = clk.stop()
    pw = statistics.median([float(r[2]) for r in clk.rows[len(clk.rows) // 2:]])
    ms = statistics.median(mss[len(mss) // 2:])
    rate = 148 * iters * 9 / (ms * 1e-3)   # MMAs/s
    print(json.dumps({"mode": names[mode], "ms": ms, "G_mma_per_s": rate / 1e9,
                      "TFLOPs": rate * 2 * 128 * 128 * (8 if mode in (0, 3) else 16) / 1e12,
                      "power_w": pw, "sm_mhz": c["sm_mhz"], "reasons": c["reasons"]}), flush=True)
