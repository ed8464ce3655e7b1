import ctypes, os, sys, json, time, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
import benchkit
HERE = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(HERE, os.environ.get("TCX_LIB", "libtcexp.so")))
L.tcx_run.restype = ctypes.c_float
L.tcx_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
S = torch.randn(n * 36 * 60 * 2, device="cuda")
R = torch.empty(n * 7680, device="cuda")
W = torch.zeros(2 * 72 * 128, device="cuda")
if os.environ.get("TCX_W", "zero") == "random":
    W = torch.randn(2 * 72 * 128, device="cuda") * 0.1
    W[72 * 128:] *= 2.0 ** -12          # second term ~ the W2 residual of a real split
names = {0: "full", 1: "no-mma", 2: "no-store", 3: "no-mma,no-store", 4: "no-split", 5: "no-mma,no-split",
         6: "no-store,no-split", 7: "only-loads", 8: "no-loads", 10: "no-loads,no-store", 12: "no-loads,no-split",
         14: "only-mma", 15: "nothing"}
# (round-2 energy experiments on the tf32 kernel — DBG 16 / 48 / 64 / 240: products as fp16
# MMAs on reinterpreted or fp16-packed terms — led to the fp16-term kernel, DESIGN.md §7;
# their code paths went with the tf32 kernel)
modes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1, 2, 4, 8, 3, 6, 10, 12, 14, 5, 7, 15]
for dbg in modes:
    rec = {}
    if secs > 0:
        clk = benchkit.ClockSampler(0, period_ms=50).start()
        t0 = time.time(); mss = []
        while time.time() - t0 < secs:
            mss.append(L.tcx_run(dbg, S.data_ptr(), R.data_ptr(), W.data_ptr(), n, 5))
        c = clk.stop()
        ms = statistics.median(mss[len(mss) // 2:])
        rec = {"sm_mhz": c["sm_mhz"], "power_w_max": c["power_w_max"], "reasons": c["reasons"],
               "power_median": statistics.median([float(r[2]) for r in clk.rows[len(clk.rows) // 2:]])}
    else:
        ms = L.tcx_run(dbg, S.data_ptr(), R.data_ptr(), W.data_ptr(), n, 10)
    print(json.dumps({"dbg": dbg, "what": names[dbg], "ms": ms, "Mblk_s": n / ms / 1e3,
                      "GBps": n * 48000 / ms / 1e6, **rec}), flush=True)
