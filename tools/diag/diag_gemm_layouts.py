"""Diagnostic (not collected): bf16 tcgen05 GEMM time per operand layout
(synk_gemm_tc2 layout bits) on the C5 shapes; device time by rank-stream
events, 20 launches after 3 warm-ups."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, "tests")
from cabi import Ranks, check, lib  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p
shapes = [(8192, 4096, 4096), (8192, 4096, 2048), (4097, 4096, 8192), (2049, 4096, 8192), (8192, 100, 4096),
          (4097, 100, 8192)]
with Ranks(1) as R:
    h = R[0]
    for M, N, K in shapes:
        a = R.alloc(max(M, K) * (max(M, K) + 8) * 2)
        b = R.alloc(max(N, K) * (max(N, K) + 8) * 2)
        c = R.alloc(M * N * 4)
        lib().synk_memset(h, _vp(a), 0, _u64(max(M, K) * (max(M, K) + 8) * 2))
        lib().synk_memset(h, _vp(b), 0, _u64(max(N, K) * (max(N, K) + 8) * 2))
        row = []
        for layout in (0, 1, 2, 3):
            lda = (M + 8) // 8 * 8 if layout & 1 else (K + 7) // 8 * 8
            ldb = (N + 7) // 8 * 8 if layout & 2 else (K + 7) // 8 * 8

            def run():
                check(lib().synk_gemm_tc2(h, 0, _u64(M), _u64(N), _u64(K), _vp(a), None, _u64(lda), _vp(b), None,
                                          _u64(ldb), layout, 0, 1, _vp(c), _u64(N), None, _u64(0), None, None,
                                          _u64(0)), "gemm")
            for _ in range(3):
                run()
            m0, m1 = ctypes.c_int(), ctypes.c_int()
            lib().synk_mark_reset(h)
            lib().synk_mark(h, ctypes.byref(m0))
            for _ in range(20):
                run()
            lib().synk_mark(h, ctypes.byref(m1))
            check(R.sync(), "sync")
            sec = ctypes.c_double()
            lib().synk_mark_elapsed(h, m0.value, m1.value, ctypes.byref(sec))
            t = sec.value / 20
            row.append("L%d %7.1f us %6.0f TF/s" % (layout, t * 1e6, 2 * M * N * K / t / 1e12))
        print("%5d x %5d x %5d: %s" % (M, N, K, " | ".join(row)), flush=True)
