"""Diagnostic (not collected by pytest): small-message latency of the phase +
collective path (C4's 1 KiB end), and of the raw launch + stream sync."""
import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from cabi import F32, Ranks, check, lib  # noqa: E402

import paper_1710_04162_b200 as sk  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p


def per_call(fn, reps=2000):
    for _ in range(50):
        fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return 1e6 * (time.perf_counter() - t) / reps


with Ranks(1) as R:
    d = R.alloc(1024)
    print("C-ABI launch(fill 256) + synk_sync: %.2f us" % per_call(
        lambda: (lib().synk_fill(R[0], F32, _vp(d), ctypes.c_double(1.0), _u64(256)), lib().synk_sync(R[0]))))
    print("C-ABI synk_sync (idle stream):      %.2f us" % per_call(lambda: lib().synk_sync(R[0])))

for world in (1, 2, 4):
    with sk.Pool(workers=world) as pool:
        v = sk.replicate(pool, np.zeros(256, np.float32))
        print("W=%d all_reduce 1 KiB: %.2f us   broadcast 1 KiB: %.2f us" % (
            world, per_call(lambda: v.all_reduce("mean")), per_call(lambda: v.broadcast(0))))
        f = sk.make_function(pool, sk.row_count_kernel(), ["scatter"], ["sum"])
        sk.distribute(pool)
        x = np.zeros((64, 4), np.float32)
        print("W=%d call(row_count, 64x4 host input): %.2f us" % (world, per_call(lambda: f.call([x]), 500)))
