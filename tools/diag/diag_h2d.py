"""Diagnostic (not collected): host->device copy paths for a 2 MiB index list."""
import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
from cabi import Ranks, check, lib  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p
n = 262144
idx = np.random.default_rng(0).integers(0, 10**7, n).astype(np.uint64)
with Ranks(1) as R:
    d = R.alloc(n * 8)
    pinned = _vp()
    check(lib().synk_host_alloc(_u64(n * 8), ctypes.byref(pinned)), "pin")
    pin_np = np.ctypeslib.as_array(ctypes.cast(pinned, ctypes.POINTER(ctypes.c_uint64)), shape=(n,))
    for name, fn in (
        ("pageable cudaMemcpyAsync+sync", lambda: (lib().synk_copy(R[0], _vp(d), idx.ctypes.data_as(_vp), _u64(n * 8)), R.sync())),
        ("numpy copy into pinned", lambda: np.copyto(pin_np, idx)),
        ("pinned DMA+sync", lambda: (lib().synk_copy(R[0], _vp(d), pinned, _u64(n * 8)), R.sync())),
        ("list(int) conversion", lambda: idx.tolist()),
        ("int64 astype copy", lambda: idx.astype(np.int64)),
    ):
        for _ in range(3):
            fn()
        t0 = time.perf_counter()
        for _ in range(20):
            fn()
        print("%-34s %8.1f us" % (name, (time.perf_counter() - t0) / 20 * 1e6))
