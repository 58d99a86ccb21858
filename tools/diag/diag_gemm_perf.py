"""Diagnostic (not collected by pytest): tcgen05 GEMM throughput via the C-ABI."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, "tests")
from cabi import Ranks, check, lib  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p


def bench(M, N, K, reps=20):
    with Ranks(1) as R:
        a = R.alloc(M * K * 2)
        b = R.alloc(N * K * 2)
        c = R.alloc(M * N * 4)
        lib().synk_memset(R[0], _vp(a), 0, _u64(M * K * 2))
        lib().synk_memset(R[0], _vp(b), 0, _u64(N * K * 2))
        marks = []
        for i in range(reps + 3):
            m = ctypes.c_int()
            if i == 3:
                check(lib().synk_mark(R[0], ctypes.byref(m)), "mark")
                marks.append(m.value)
            check(lib().synk_gemm_tc(R[0], 0, _u64(M), _u64(N), _u64(K), _vp(a), None, _u64(K), _vp(b), None, _u64(K),
                                     0, 1, _vp(c), _u64(N), None, _u64(0), None, None, _u64(0)), "gemm")
        m = ctypes.c_int()
        check(lib().synk_mark(R[0], ctypes.byref(m)), "mark")
        check(R.sync(), "sync")
        s = ctypes.c_double()
        check(lib().synk_mark_elapsed(R[0], marks[0], m.value, ctypes.byref(s)), "el")
        t = s.value / reps
        print("M=%5d N=%5d K=%5d  %.3f ms  %.1f TFLOP/s" % (M, N, K, t * 1e3, 2.0 * M * N * K / t / 1e12))


for shape in ((8192, 4096, 4096), (4096, 4096, 4096), (8192, 8192, 8192), (2048, 4096, 8192), (8192, 100, 4096)):
    bench(*shape)
