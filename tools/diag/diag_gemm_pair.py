"""Diagnostic (not collected): persistent bf16 GEMM throughput with random
operands (8192 x 4096 x 4096 and C5's other wide shapes), K-major and
MN-major B, bf16 output; run with SYNK_GEMM_PAIR=0|1 to compare the 1-CTA
128x256 and the CTA-pair 256x256 kernels."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, "tests")
from cabi import Ranks, check, lib  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p
rng = np.random.default_rng(0)


def rand_bf16(n):
    x = rng.standard_normal(n, dtype=np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)


def bench(M, N, K, layout, reps=30):
    with Ranks(1) as R:
        a = R.upload(rand_bf16(M * K))
        b = R.upload(rand_bf16(N * K))
        c = R.alloc(M * N * 2)
        marks = []
        for i in range(reps + 5):
            m = ctypes.c_int()
            if i == 5:
                check(lib().synk_mark(R[0], ctypes.byref(m)), "mark")
                marks.append(m.value)
            check(lib().synk_gemm_tc2(R[0], 0, _u64(M), _u64(N), _u64(K), _vp(a), None, _u64(K), _vp(b), None,
                                      _u64(N if layout else K), layout, 0, 3, _vp(c), _u64(N), None, _u64(0), None,
                                      None, _u64(0)), "gemm")
        m = ctypes.c_int()
        check(lib().synk_mark(R[0], ctypes.byref(m)), "mark")
        check(R.sync(), "sync")
        s = ctypes.c_double()
        check(lib().synk_mark_elapsed(R[0], marks[0], m.value, ctypes.byref(s)), "el")
        t = s.value / reps
        print("pair=%s %5dx%5dx%5d B-%s  %.1f us  %.0f TFLOP/s" % (os.environ.get("SYNK_GEMM_PAIR", "0"), M, N, K,
              "MN" if layout else "K ", t * 1e6, 2 * M * N * K / t / 1e12))


for shape in [(8192, 4096, 4096), (8192, 4096, 2048), (4097, 4096, 8192), (2049, 4096, 8192)]:
    for layout in (0, 2):
        bench(*shape, layout)
