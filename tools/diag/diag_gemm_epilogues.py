"""Diagnostic (not collected): persistent bf16 GEMM 8192x4096x4096 time per
epilogue variant (the C5 products), device time by rank-stream events."""
import ctypes
import sys

sys.path.insert(0, "tests")
from cabi import Ranks, check, lib  # noqa: E402

_u64, _vp = ctypes.c_uint64, ctypes.c_void_p
M, N, K = 8192, 4096, 4096
F32, BF16 = 1, 3
with Ranks(1) as R:
    h = R[0]
    a = R.alloc(M * K * 2)
    b = R.alloc(N * K * 2)
    c = R.alloc(M * N * 4)
    ct = R.alloc(M * N * 2)
    act = R.alloc(M * N * 2)
    bias = R.alloc(N * 4)
    zeros = len(sys.argv) > 1 and sys.argv[1] == "zeros"
    for p, nb in ((a, M * K * 2), (b, N * K * 2), (act, M * N * 2), (bias, N * 4)):
        lib().synk_memset(h, _vp(p), 0, _u64(nb))
    if not zeros:  # random bf16 operands: U[-1,1) f32 -> bf16 (power/clock behaviour of real data)
        tmp = R.alloc(max(M, N) * K * 4)
        for p, rows in ((a, M), (b, N)):
            lib().synk_fill_uniform(h, 1, _vp(tmp), _u64(rows * K), _u64(rows), _u64(0))
            check(lib().synk_gemm_prep2_bf16(h, _vp(tmp), _u64(rows), _u64(K), _u64(K), _vp(p), _u64(K), None,
                                             _u64(0)), "prep")
    variants = [
        ("store f32", 0, F32, False, False, 0),
        ("store bf16", 0, BF16, False, False, 0),
        ("bias bf16", 1, BF16, False, False, 0),
        ("bias_tanh bf16", 2, BF16, False, False, 0),
        ("bias_tanh bf16 + C^T", 2, BF16, True, False, 0),
        ("tanh_grad bf16 (act)", 3, BF16, False, True, 0),
        ("tanh_grad bf16 + C^T", 3, BF16, True, True, 0),
        ("bias_tanh bf16, B MN", 2, BF16, False, False, 2),
        ("bias_tanh bf16 + C^T, B MN", 2, BF16, True, False, 2),
    ]
    for name, epi, odt, with_t, with_act, layout in variants:
        ldb = N if layout & 2 else K

        def run():
            check(lib().synk_gemm_tc2(h, 0, _u64(M), _u64(N), _u64(K), _vp(a), None, _u64(K), _vp(b), None, _u64(ldb),
                                      layout, epi, odt, _vp(c), _u64(N), _vp(ct) if with_t else None, _u64(M),
                                      _vp(bias), _vp(act) if with_act else None, _u64(N)), "gemm")
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
        print("%-28s %7.1f us %6.0f TF/s  %s" % (name, t * 1e6, 2 * M * N * K / t / 1e12, "zeros" if zeros else "random"),
              flush=True)
