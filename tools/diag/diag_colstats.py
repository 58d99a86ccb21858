"""Diagnostic (not collected by pytest): column-statistics kernel throughput
(C3's per-slice aggregation pass) via the C-ABI, input generated in HBM."""
import ctypes
import sys

sys.path.insert(0, "tests")
from cabi import F32, Ranks, check, lib  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p


def bench(rows, cols, reps=10):
    nbytes = rows * cols * 4
    with Ranks(1) as R:
        x = R.alloc(nbytes)
        s, m = R.alloc(cols * 4), R.alloc(cols * 4)
        check(lib().synk_fill_uniform(R[0], F32, _vp(x), _u64(rows * cols), _u64(3), _u64(0)), "fill")
        marks = []
        for i in range(reps + 2):
            mk = ctypes.c_int()
            if i == 2:
                check(lib().synk_mark(R[0], ctypes.byref(mk)), "mark")
                marks.append(mk.value)
            check(lib().synk_column_stats(R[0], F32, _vp(x), _u64(rows), _u64(cols), _vp(s), _vp(m), None), "cs")
        mk = ctypes.c_int()
        check(lib().synk_mark(R[0], ctypes.byref(mk)), "mark")
        check(R.sync(), "sync")
        el = ctypes.c_double()
        check(lib().synk_mark_elapsed(R[0], marks[0], mk.value, ctypes.byref(el)), "el")
        t = el.value / reps
        print("rows=%8d cols=%5d  %.3f ms  %.1f GB/s" % (rows, cols, t * 1e3, nbytes / t / 1e9))


for shape in ((2097152, 1024), (8388608, 1024), (1048576, 256), (4194304, 4096 // 4)):
    bench(*shape)
