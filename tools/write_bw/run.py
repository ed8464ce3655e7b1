import ctypes, os, json
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwbw.so"))
L.wbw_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
n = 1 << 20
R = torch.empty(n * 7680, device="cuda")
for mode, name in [(0, "stg64"), (4, "stg64x8warps"), (5, "stg128shfl"), (2, "bulk"), (3, "memset")]:
    for cps in ([1, 2] if mode != 3 else [1]):
        ms = ctypes.c_float()
        rc = L.wbw_run(mode, R.data_ptr(), n, cps, 5, ctypes.byref(ms))
        print(json.dumps({"mode": name, "ctas_per_sm": cps, "rc": rc, "ms": ms.value,
                          "GBps": n * 30720 / ms.value / 1e6}), flush=True)
