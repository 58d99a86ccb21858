"""Diagnostic (not collected by pytest): accumulation precision of tcgen05
kind::tf32 on B200. Inputs pre-rounded to tf32 make every product exact, so
any error is accumulator rounding/truncation."""
import sys

import numpy as np

sys.path.insert(0, "tests")
from test_gpu_gemm import gemm  # noqa: E402
from cabi import Ranks  # noqa: E402


def tf32(x):
    u = x.astype(np.float32).view(np.uint32)
    u = (u + np.uint32(0x1000)) & np.uint32(0xFFFFE000)
    return u.view(np.float32)


rng = np.random.default_rng(0)
with Ranks(1) as R:
    for K in (32, 128, 512, 2048, 8192):
        a = tf32(rng.uniform(0, 1, (128, K)))
        b = tf32(rng.uniform(0, 1, (128, K)))
        exact = a.astype(np.float64) @ b.astype(np.float64).T
        seq32 = np.zeros((128, 128), np.float32)
        for k in range(K):
            seq32 = (seq32 + np.outer(a[:, k], b[:, k]).astype(np.float32)).astype(np.float32)
        got1, _ = gemm(R, "tf32", a, b)
        got3, _ = gemm(R, "tf32x3", a, b)
        e = lambda g: float(np.mean((g.astype(np.float64) - exact) / exact))
        m = lambda g: float(np.max(np.abs(g.astype(np.float64) - exact) / exact))
        print("K=%5d tf32(exact products): mean rel %+.3e max %.3e | 3x: mean %+.3e max %.3e | seq fp32: mean %+.3e max %.3e"
              % (K, e(got1), m(got1), e(got3), m(got3), e(seq32), m(seq32)))
