"""Diagnostic (not collected; run under ncu): C4 all-reduce mean of a 256 MiB
f32 replicated variable, W=2 ranks on GPU 0 (peer-memory chunk kernels)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

n = (256 << 20) // 4
with sk.Pool(workers=2, devices=[0, 0]) as pool:
    var = sk.replicate(pool, np.zeros(1, np.float32))
    var.set(0, np.ones(n, np.float32))
    var.set(1, np.full(n, 2.0, np.float32))
    for _ in range(3):
        var.all_reduce("mean")
    assert var.coherent
print("ok")
