"""Diagnostic (not collected): the C5 GEMM shapes with their real epilogues, timed per launch."""
import ctypes
import sys

sys.path.insert(0, "tests")
from cabi import Ranks, check, lib  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p
BF, F32 = 3, 1


def pad8(v):
    return (v + 7) // 8 * 8


def run(R, name, M, N, K, epi, out_bf16, with_ct, with_act, reps=10):
    a = R.alloc(M * pad8(K) * 2)
    b = R.alloc(N * pad8(K) * 2)
    es = 2 if out_bf16 else 4
    c = R.alloc(M * pad8(N) * es)
    ct = R.alloc(N * pad8(M) * es) if with_ct else 0
    act = R.alloc(M * pad8(N) * es) if with_act else 0
    bias = R.alloc(N * 4)
    for p, n in ((a, M * pad8(K) * 2), (b, N * pad8(K) * 2), (bias, N * 4)):
        lib().synk_memset(R[0], _vp(p), 0, _u64(n))
    if act:
        lib().synk_memset(R[0], _vp(act), 0, _u64(M * pad8(N) * es))
    marks = []
    for i in range(reps + 2):
        m = ctypes.c_int()
        if i >= 2:
            check(lib().synk_mark(R[0], ctypes.byref(m)), "mark")
            marks.append(m.value)
        check(lib().synk_gemm_tc(R[0], 0, _u64(M), _u64(N), _u64(K), _vp(a), None, _u64(pad8(K)), _vp(b), None,
                                 _u64(pad8(K)), epi, BF if out_bf16 else F32, _vp(c), _u64(pad8(N)), _vp(ct or None),
                                 _u64(pad8(M)), _vp(bias), _vp(act or None), _u64(pad8(N))), name)
        if i >= 2:
            check(lib().synk_mark(R[0], ctypes.byref(m)), "mark")
            marks.append(m.value)
    check(R.sync(), "sync")
    ts = []
    for x, y in zip(marks[0::2], marks[1::2]):
        s = ctypes.c_double()
        lib().synk_mark_elapsed(R[0], x, y, ctypes.byref(s))
        ts.append(s.value)
    t = sorted(ts)[len(ts) // 2]
    print("%-22s M=%5d N=%5d K=%5d  median %.1f us  max %.1f us  %.0f TFLOP/s" % (name, M, N, K, t * 1e6, max(ts) * 1e6,
                                                                              2.0 * M * N * K / t / 1e12))


only = sys.argv[1] if len(sys.argv) > 1 else None
_run = run


def run(R, name, *a, **k):  # noqa: F811
    if only is None or name.startswith(only):
        _run(R, name, *a, **k)


with Ranks(1) as R:
    n = 8192
    run(R, "fwd1 store bf16", n, 4096, 4096, 0, True, False, False)
    run(R, "fwd1 bias_tanh", n, 4096, 4096, 2, True, False, False)
    run(R, "fwd1 store bf16+ct", n, 4096, 4096, 0, True, True, False)
    run(R, "fwd0 bias_tanh+ct", n, 4096, 2048, 2, True, True, False)
    run(R, "fwd1 bias_tanh+ct", n, 4096, 4096, 2, True, True, False)
    run(R, "fwd2 bias f32", n, 100, 4096, 1, False, False, False)
    run(R, "gW2 store", 4096, 100, n, 0, False, False, False)
    run(R, "dX2 tanhgrad+ct", n, 4096, 100, 3, True, True, True)
    run(R, "gW1 store", 4096, 4096, n, 0, False, False, False)
    run(R, "dX1 tanhgrad+ct", n, 4096, 4096, 3, True, True, True)
    run(R, "gW0 store", 2048, 4096, n, 0, False, False, False)
