"""Write bandwidth of STG.128 vs STG.256 from 4-32 warps per SM (tools/write_bw)."""
import ctypes, json, os
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwbw.so"))
L.wbw_vec.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int,
                      ctypes.POINTER(ctypes.c_float)]
n = 1 << 18
R = torch.empty(n * 7680, device="cuda")
for order in (0, 1, 2):
    for vec, warps in ((4, 8), (8, 8), (4, 32)):
        ms = ctypes.c_float()
        rc = L.wbw_vec(vec, warps, order, R.data_ptr(), n, 10, ctypes.byref(ms))
        print(json.dumps({"order": ["range", "grid-stride", "random"][order], "vec": vec, "warps": warps,
                          "rc": rc, "GBps": round(n * 30720 / ms.value / 1e6)}), flush=True)
