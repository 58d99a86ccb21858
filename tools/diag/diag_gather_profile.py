"""Diagnostic (not collected; run under ncu): the two gather launches the bench
measures, on the 10M x 256 f32 HBM mirror with 262,144-row steps --
launches 0-2: index list in HBM (bench `value`, C-ABI synk_gather_rows);
launches 3-5: Function.call(indexes=<pinned int64 array>) (bench `e2e`: the
kernel reads the index list in place over PCIe)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

rows, n = 10_000_000, 4096 * 64
lib = ctypes.CDLL(os.path.join("paper_1710_04162_b200", "_lib", "libsynk_cuda.so"))
vp, u64 = ctypes.c_void_p, ctypes.c_uint64
rng = np.random.default_rng(0)
with sk.Pool(workers=1) as pool:
    arr = sk.SharedInput.alloc([rows, 256], "f32")
    arr.mirror(pool)
    h = vp(pool.device_handle(0))
    idx = rng.integers(0, rows, n).astype(np.uint64)
    d_idx, d_out = vp(), vp()
    assert lib.synk_alloc(h, u64(idx.nbytes), ctypes.byref(d_idx)) == 0
    assert lib.synk_alloc(h, u64(n * 1024), ctypes.byref(d_out)) == 0
    assert lib.synk_copy(h, d_idx, idx.ctypes.data_as(vp), u64(idx.nbytes)) == 0
    for _ in range(3):
        assert lib.synk_gather_rows(h, vp(arr.mirror_ptr(0)), u64(rows), u64(1024), d_idx, u64(n), d_out) == 0
    assert lib.synk_sync(h) == 0
    f = sk.make_function(pool, sk.row_count_kernel(), ["scatter"], ["sum"])
    sk.distribute(pool)
    pinned = sk.pinned_array(n, "int64")
    pinned[:] = idx
    for _ in range(3):
        (c,) = f.call([arr], indexes=pinned)
        assert float(c) == n
print("ok")
