"""Diagnostic (not collected): latency of ONE 4096-row batch per Function.call
(bench.py's single_batch_call: row_count kernel over the HBM mirror of a
SharedInput, pinned int64 index list). Prints us/call; run with
SYNK_CALL_TRACE=1 on a trace build for the executor's per-stage stamps."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
B = 4096
rng = np.random.default_rng(0)
with sk.Pool(workers=1) as pool:
    arr = sk.SharedInput.alloc([rows, 256], "f32")
    arr.mirror(pool)
    f = sk.make_function(pool, sk.row_count_kernel(), ["scatter"], ["sum"])
    sk.distribute(pool)
    idx = []
    for _ in range(64):
        b = sk.pinned_array(B, "int64")
        b[:] = rng.integers(0, rows, B)
        idx.append(b)
    for rep in range(3):
        for s in range(200):
            f.call([arr], indexes=idx[s % 64])
        t0 = time.perf_counter()
        for s in range(2000):
            (cnt,) = f.call([arr], indexes=idx[s % 64])
        dt = (time.perf_counter() - t0) / 2000
        assert float(cnt) == B
        print("single-batch call: %.2f us" % (1e6 * dt), flush=True)
