"""Diagnostic (not collected): where a bf16 GEMM result differs from fp64."""
import sys

import numpy as np

sys.path.insert(0, "tests")
from test_gpu_gemm import bf16_round, gemm  # noqa: E402
from cabi import Ranks  # noqa: E402

for (M, N, K) in ((8192, 384, 2048), (4096, 2048, 512), (1024, 512, 2048), (8192, 512, 512), (256, 384, 2048)):
    rng = np.random.default_rng(M + N + K)
    a = bf16_round(rng.uniform(-1, 1, (M, K)))
    b = bf16_round(rng.uniform(-1, 1, (N, K)))
    want = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        got, _ = gemm(R, "bf16", a, b)
    bad = np.abs(got - want) > 1e-3 * np.maximum(1, np.abs(want))
    rows = np.where(bad.any(1))[0]
    cols = np.where(bad.any(0))[0]
    print((M, N, K), "bad", int(bad.sum()), "rows", rows[:3], rows[-3:] if rows.size else [], "n", rows.size,
          "cols", cols[:3], cols[-3:] if cols.size else [], "n", cols.size)
