"""Diagnostic (not collected): the C5 narrow (N=100) bf16 products -- forward
8192x100x4096 (A K-major, B = W^T K-major) and weight gradient 4097x100x8192
(A = a^T, B = delta^T) -- timed via the C-ABI with zero operands (the products are load-bound), split-K
fold included. SYNK_SPLITK_CTAS / SYNK_SPLITK_MINKB select the split."""
import ctypes
import os
import sys

sys.path.insert(0, "tests")
from cabi import Ranks, check, lib  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p


def bench(M, N, K, reps=50):
    with Ranks(1) as R:
        a = R.alloc(M * K * 2)
        b = R.alloc(128 * K * 2)
        c = R.alloc(M * N * 4)
        lib().synk_memset(R[0], _vp(a), 0, _u64(M * K * 2))
        lib().synk_memset(R[0], _vp(b), 0, _u64(128 * K * 2))
        marks = []
        for i in range(reps + 5):
            m = ctypes.c_int()
            if i == 5:
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
        print("%s/%s M=%5d N=%3d K=%5d  %.1f us  A %.0f GB/s" % (os.environ.get("SYNK_SPLITK_CTAS", "296"),
              os.environ.get("SYNK_SPLITK_MINKB", "8"), M, N, K, t * 1e6, M * K * 2 / t / 1e9))


bench(8192, 100, 4096)
bench(4097, 100, 8192)
