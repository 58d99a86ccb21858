"""Diagnostic (not collected): the C5 short-K backward product dX_2 =
(delta . W_2^T) * (1 - a_2^2): M=8192, N=4096, K=100, bf16 operands, the
tanh-derivative epilogue reading the bf16 activation and writing bf16 --
epilogue/HBM bound (64 MB act read + 64 MB write). Timed via the C-ABI."""
import ctypes
import sys

sys.path.insert(0, "tests")
from cabi import Ranks, check, lib  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p
M, N, K = 8192, 4096, 100
KP = 104  # 16-byte aligned rows
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
with Ranks(1) as R:
    a = R.alloc(M * KP * 2)
    b = R.alloc(N * KP * 2)
    act = R.alloc(M * N * 2)
    c = R.alloc(M * N * 2)
    for p, n in ((a, M * KP * 2), (b, N * KP * 2), (act, M * N * 2)):
        lib().synk_memset(R[0], _vp(p), 0, _u64(n))
    marks = []
    for i in range(reps + 5):
        if i == 5:
            m = ctypes.c_int()
            check(lib().synk_mark(R[0], ctypes.byref(m)), "mark")
            marks.append(m.value)
        check(lib().synk_gemm_tc2(R[0], 0, _u64(M), _u64(N), _u64(K), _vp(a), None, _u64(KP), _vp(b), None, _u64(KP),
                                  0, 3, 3, _vp(c), _u64(N), None, _u64(0), None, _vp(act), _u64(N)), "gemm")
    m = ctypes.c_int()
    check(lib().synk_mark(R[0], ctypes.byref(m)), "mark")
    check(R.sync(), "sync")
    s = ctypes.c_double()
    check(lib().synk_mark_elapsed(R[0], marks[0], m.value, ctypes.byref(s)), "el")
    t = s.value / reps
    print("dX short-K M=%d N=%d K=%d: %.1f us  act+C %.0f GB/s" % (M, N, K, t * 1e6, 2 * M * N * 2 / t / 1e9))
