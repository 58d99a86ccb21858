"""Diagnostic (not collected): host cost per launch of C-ABI entry points
(no synchronisation inside the loop): small-param kernels vs the collective
kernels whose parameter block carries 64 peer pointers."""
import ctypes
import sys
import time

sys.path.insert(0, "tests")
from cabi import Ranks, check, lib, ptr_array  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p
with Ranks(2) as R:
    h = R[0]
    a, b, c = R.alloc(4096), R.alloc(4096, 1), R.alloc(4096)
    ptrs = ptr_array([a, b])
    cases = {
        "copy_small (3 args)": lambda: lib().synk_copy_small(h, _vp(c), _vp(a), _u64(1024)),
        "fill (4 args)": lambda: lib().synk_fill(h, 1, _vp(c), ctypes.c_double(1.0), _u64(256)),
        "broadcast_whole (64-ptr block)": lambda: lib().synk_broadcast_whole(h, 2, 0, ptrs, _u64(1024)),
        "all_reduce_whole (64-ptr block)": lambda: lib().synk_all_reduce_whole(h, 2, 1, 1, ptrs, _u64(256)),
    }
    for name, fn in cases.items():
        for _ in range(200):
            fn()
        check(R.sync(), "sync")
        t = time.perf_counter()
        for _ in range(2000):
            fn()
        dt = (time.perf_counter() - t) / 2000
        check(R.sync(), "sync")
        t2 = time.perf_counter()
        for _ in range(500):
            fn()
            R.sync()
        rt = (time.perf_counter() - t2) / 500
        print("%-34s launch %5.2f us   launch+sync %5.2f us" % (name, dt * 1e6, rt * 1e6))
