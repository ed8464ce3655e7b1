import ctypes, os
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(HERE, "libtcprobe_bf16.so"))
L.tcp_bf16.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int]

def to_bf16(x):   # round-to-nearest-even fp32 -> bf16 bits
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return b.astype(np.uint16)

def from_bf16(u):
    return (u.astype(np.uint32) << 16).view(np.float32)

rng = np.random.default_rng(0)
K = 144
A = to_bf16(rng.standard_normal((128, K)).astype(np.float32))
B = to_bf16(rng.standard_normal((128, K)).astype(np.float32))
D = np.zeros((128, 128), np.float32)
assert L.tcp_bf16(A.ctypes.data, B.ctypes.data, D.ctypes.data, K) == 0
ref = from_bf16(A).astype(np.float64) @ from_bf16(B).astype(np.float64).T
print("bf16 TS MMA: max err rel", np.abs(D - ref).max() / np.abs(ref).max(), D[0, :3], ref[0, :3])
