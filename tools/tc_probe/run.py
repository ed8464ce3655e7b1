"""Checks the tcgen05 probe against numpy (run on a B200)."""
import ctypes, os, sys
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(HERE, "libtcprobe.so"))
L.tcp_run.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int]

def tf32(x):
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x1000) & 0xFFFFE000   # round half away (magnitude), like cvt.rna
    return b.astype(np.uint32).view(np.float32)

def run(A, B):
    K = A.shape[1]
    D = np.zeros((128, 128), np.float32)
    rc = L.tcp_run(A.ctypes.data, B.ctypes.data, D.ctypes.data, K)
    assert rc == 0, rc
    return D

rng = np.random.default_rng(0)
K = 72
A = tf32(rng.standard_normal((128, K)).astype(np.float32))
B = tf32(rng.standard_normal((128, K)).astype(np.float32))
D = run(A, B)
ref = A.astype(np.float64) @ B.astype(np.float64).T
err = np.abs(D - ref).max() / np.abs(A).max() / np.abs(B).max() / K
print("random: max err (rel to K*max|a||b|):", err, "D[0,:4]", D[0, :4], "ref", ref[0, :4])
# exactness: B = selection (identity-like) picks A columns; splits summed
S = rng.standard_normal(128).astype(np.float32)
s1 = tf32(S); s2 = tf32(S - s1); s3 = (S - s1 - s2).astype(np.float32)
assert np.array_equal(tf32(s3), s3)
A2 = np.zeros((128, 8), np.float32); A2[:, 0] = s1; A2[:, 1] = s2; A2[:, 2] = s3
B2 = np.zeros((128, 8), np.float32); B2[0, :3] = 1.0          # D[:,0] = s1 + s2 + s3
D2 = run(A2, B2)
print("3-split identity exact:", np.array_equal(D2[:, 0], S), "zeros +0:",
      not D2[:, 1:].view(np.uint32).any())
# signed zeros: negative A times zero B
A3 = -np.abs(tf32(rng.standard_normal((128, 8)).astype(np.float32)))
B3 = np.zeros((128, 8), np.float32)
D3 = run(A3, B3)
print("neg*0 sign bits set:", int((D3.view(np.uint32) >> 31).sum()), "of", D3.size)
# accumulation rounding vs fp32 RN of exact sum: many terms
A4 = tf32(rng.uniform(0.5, 1, (128, K)).astype(np.float32))
B4 = tf32(rng.uniform(0.5, 1, (128, K)).astype(np.float32))
D4 = run(A4, B4)
ex = A4.astype(np.float64) @ B4.astype(np.float64).T
ulp = np.spacing(np.abs(ex).astype(np.float32)).astype(np.float64)
print("positive sums: max |D-exact| in ulps:", (np.abs(D4 - ex) / ulp).max(),
      "mean signed err/ulp:", ((D4 - ex) / ulp).mean())
