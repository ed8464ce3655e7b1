"""Latency of one short tensor-kernel launch (c2: 770 blocks, one W) with a cold L2,
per DBG mode and grid size: where the ~19 us of a one-slot launch go.
    python tools/tc_exp/lat.py [n] [modes] [grids]"""
import ctypes, os, sys, json
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(HERE, "libtcexp.so"))
L.tcx_lat.restype = ctypes.c_float
L.tcx_lat.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                      ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 770
modes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 4, 8, 15]
grids = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [148]
S = torch.randn(n * 36 * 60 * 2, device="cuda")
R = torch.empty(n * 7680, device="cuda")
W = torch.randn(2 * 72 * 128, device="cuda") * 0.1
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
names = {0: "full", 1: "no-mma", 2: "no-store", 4: "no-split", 8: "no-loads", 15: "nothing"}
for g in grids:
    for dbg in modes:
        cold = L.tcx_lat(dbg, S.data_ptr(), R.data_ptr(), W.data_ptr(), n, g, fl.data_ptr(), fl.numel(), 21)
        warm = L.tcx_lat(dbg, S.data_ptr(), R.data_ptr(), W.data_ptr(), n, g, None, 0, 21)
        print(json.dumps({"n": n, "grid": g, "dbg": dbg, "what": names[dbg], "cold_us": cold * 1e3,
                          "warm_us": warm * 1e3}), flush=True)
# an empty launch of the same kernel (n = 0 returns before TMEM allocation)
e = L.tcx_lat(0, S.data_ptr(), R.data_ptr(), W.data_ptr(), 0, 148, None, 0, 21)
print(json.dumps({"n": 0, "grid": 148, "what": "empty launch", "warm_us": e * 1e3}))
