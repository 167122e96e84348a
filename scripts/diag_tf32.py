"""Diagnostic: accuracy of the real32 path's 3xTF32 GEMM by operand kind."""
import numpy as np
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_28760_b200.engine import test_gemm_tf32x3


def tf32(x):
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)


rng = np.random.default_rng(0)
M, N, K = 256, 256, 768
A = rng.standard_normal((M, K)).astype(np.float32)
W = (0.02 * rng.standard_normal((K, N))).astype(np.float32).astype(np.float64)
scale = np.sqrt(K) * 0.02
for name, a, w in [("both tf32-exact", tf32(A), tf32(W).astype(np.float64)), ("A exact", tf32(A), W),
                   ("W exact", A, tf32(W).astype(np.float64)), ("general", A, W)]:
    got = test_gemm_tf32x3(a, w).astype(np.float64)
    ref = a.astype(np.float64) @ w
    e = np.abs(got - ref) / scale
    print(f"{name:18s} max {e.max():.3e} rms {np.sqrt((e**2).mean()):.3e}")
# K sweep: error growth with K
for K in (32, 64, 256, 1024, 4096):
    a = rng.standard_normal((128, K)).astype(np.float32)
    w = tf32(0.02 * rng.standard_normal((K, 128))).astype(np.float64)
    a = tf32(a)
    got = test_gemm_tf32x3(a, w).astype(np.float64)
    ref = a.astype(np.float64) @ w
    print("K", K, "exact operands max rel", (np.abs(got - ref) / (np.sqrt(K) * 0.02)).max())
# single column probe: a = e_k, result must equal w row exactly
a = np.zeros((128, 64), np.float32); a[np.arange(64), np.arange(64)] = 1.0
w = (0.02 * rng.standard_normal((64, 128)))
got = test_gemm_tf32x3(a, w)
print("identity max abs err vs fp32(w)", np.abs(got[:64] - w.astype(np.float32)).max())
