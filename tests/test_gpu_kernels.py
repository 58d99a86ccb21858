"""Kernel-level parity through the C-ABI (libsynk_cuda.so) against the oracle.

Bar: bit-exact for gather / combine max-min / collectives (tree order) /
optimizer updates; elem_err tolerances stated inline for floating-point sums
whose association order differs from the reference (column sums, MLP GEMMs).
"""

import ctypes

import numpy as np
import pytest

import cabi
from cabi import F32, F64, OPS, RULES, Ranks, check, lib, ptr_array
from conftest import golden

pytestmark = pytest.mark.gpu
_u64 = ctypes.c_uint64
_vp = ctypes.c_void_p


def test_gather_bit_exact_vs_oracle(oracle):
    rng = np.random.default_rng(0)
    with Ranks(1) as R:
        for dtype, shape in ((np.float32, (10000, 256)), (np.float32, (513, 37)), (np.float64, (300, 8)),
                             (np.float32, (64, 10)), (np.float64, (5, 1))):
            src = rng.uniform(-1, 1, shape).astype(dtype)
            for n_idx in (0, 1, 3, 4096, 4099):
                idx = rng.integers(0, shape[0], n_idx).astype(np.uint64)
                d_src, d_idx = R.upload(src), R.upload(idx)
                d_out = R.alloc(n_idx * src[0].nbytes)
                check(lib().synk_gather_rows(R[0], _vp(d_src), _u64(shape[0]), _u64(src[0].nbytes), _vp(d_idx),
                                             _u64(n_idx), _vp(d_out)), "gather")
                check(R.sync(), "sync")
                got = R.download(d_out, (n_idx,) + shape[1:], dtype)
                assert got.tobytes() == oracle.gather_rows(src, idx).tobytes()


def test_fill_uniform_matches_oracle_stream(oracle):
    with Ranks(1) as R:
        for dtype, code in ((np.float32, F32), (np.float64, F64)):
            for n, first, off in ((1, 0, 0), (4099, 0, 0), (1000, 123457, 0), (1001, 5, 1), (1 << 20, 1 << 33, 0)):
                d = R.alloc((n + off) * np.dtype(dtype).itemsize)
                check(lib().synk_fill_uniform(R[0], code, _vp(d + off * np.dtype(dtype).itemsize), _u64(n), _u64(9),
                                              _u64(first)), "fill_uniform")
                check(R.sync(), "sync")
                got = R.download(d, (n + off,), dtype)[off:]
                assert got.tobytes() == oracle.fill_uniform(n, 9, first, dtype).tobytes()
                assert got.min() >= -1 and got.max() < 1


def test_gather_golden_vectors():
    g = golden("gather.npz")
    with Ranks(1) as R:
        for tag, dtype in (("f32", np.float32), ("f64", np.float64)):
            src, idx = g[tag + "_src"], g[tag + "_idx"].astype(np.uint64)
            d_src, d_idx = R.upload(src), R.upload(idx)
            d_out = R.alloc(len(idx) * src[0].nbytes)
            check(lib().synk_gather_rows(R[0], _vp(d_src), _u64(src.shape[0]), _u64(src[0].nbytes), _vp(d_idx),
                                         _u64(len(idx)), _vp(d_out)), "gather")
            got = R.download(d_out, (len(idx),) + src.shape[1:], dtype)
            assert got.tobytes() == g[tag + "_w3_list"].tobytes()


def test_gather_from_pinned_host_memory(oracle):
    """The shared dataset may stay in pinned, mapped host memory: the same
    kernel then reads rows over PCIe."""
    rng = np.random.default_rng(1)
    src = rng.uniform(-1, 1, (2000, 256)).astype(np.float32)
    host = _vp()
    check(lib().synk_host_alloc(_u64(src.nbytes), ctypes.byref(host)), "host alloc")
    try:
        ctypes.memmove(host, src.ctypes.data, src.nbytes)
        kind, dev = ctypes.c_int(), ctypes.c_int()
        lib().synk_ptr_kind(host, ctypes.byref(kind), ctypes.byref(dev))
        assert kind.value == 1
        idx = rng.integers(0, 2000, 1000).astype(np.uint64)
        with Ranks(1) as R:
            d_idx = R.upload(idx)
            d_out = R.alloc(1000 * 1024)
            check(lib().synk_gather_rows(R[0], host, _u64(2000), _u64(1024), _vp(d_idx), _u64(1000), _vp(d_out)), "g")
            got = R.download(d_out, (1000, 256), np.float32)
        assert got.tobytes() == oracle.gather_rows(src, idx).tobytes()
    finally:
        lib().synk_host_free(host)


def _pinned_copy(arr):
    host = _vp()
    check(lib().synk_host_alloc(_u64(max(arr.nbytes, 1)), ctypes.byref(host)), "host alloc")
    ctypes.memmove(host, arr.ctypes.data, arr.nbytes)
    return host


@pytest.mark.parametrize("idx_in", ["hbm", "pinned"])
def test_gather_wide_rows(oracle, idx_in):
    """Rows of 4-8 KiB (odd sizes too); index lists in HBM or in pinned host
    memory (read in place over PCIe). Run again with SYNK_GATHER_BULK=1 by
    test_gather_bulk_kernel_subprocess for the cp.async.bulk kernel."""
    rng = np.random.default_rng(3)
    with Ranks(1) as R:
        for dtype, shape in ((np.float32, (3000, 1024)), (np.float64, (500, 1024)), (np.float32, (257, 2048)),
                             (np.float32, (300, 1028))):
            src = rng.uniform(-1, 1, shape).astype(dtype)
            d_src = R.upload(src)
            for n_idx in (1, 5, 31, 33, 1000, 4099):
                idx = rng.integers(0, shape[0], n_idx).astype(np.uint64)
                hidx = _pinned_copy(idx) if idx_in == "pinned" else None
                d_idx = hidx.value if hidx is not None else R.upload(idx)
                d_out = R.alloc(n_idx * src[0].nbytes)
                check(lib().synk_gather_rows(R[0], _vp(d_src), _u64(shape[0]), _u64(src[0].nbytes), _vp(d_idx),
                                             _u64(n_idx), _vp(d_out)), "gather")
                check(R.sync(), "sync")
                if hidx is not None:
                    lib().synk_host_free(hidx)
                got = R.download(d_out, (n_idx,) + shape[1:], dtype)
                assert got.tobytes() == oracle.gather_rows(src, idx).tobytes()
            bad = np.array([0, 3, shape[0], 1] * 20, np.uint64)
            d_out = R.alloc(bad.size * src[0].nbytes)
            check(lib().synk_gather_rows(R[0], _vp(d_src), _u64(shape[0]), _u64(src[0].nbytes), _vp(R.upload(bad)),
                                         _u64(bad.size), _vp(d_out)), "gather")
            assert R.sync() == -1  # SYNK_EBOUNDS
            assert R.sync() == 0


@pytest.mark.parametrize("variant", ["SYNK_GATHER_BULK", "SYNK_GATHER_TMA4"])
def test_gather_bulk_kernel_subprocess(variant):
    """The opt-in TMA gathers -- per-row cp.async.bulk (SYNK_GATHER_BULK=1) and
    four-rows-per-request tensor-map gather4 (SYNK_GATHER_TMA4=1); both read
    once per process -- through the gather parity tests in a child."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, **{variant: "1"})
    here = os.path.dirname(os.path.abspath(__file__))
    out = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", os.path.join(here, "test_gpu_kernels.py"),
                          "-k", "gather and not subprocess"], env=env, capture_output=True, text=True, timeout=600,
                         cwd=os.path.dirname(here))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]


def test_gather_index_list_in_pinned_host_memory(oracle):
    """The 16-byte vector kernel reading its index list over PCIe (e2e path of
    Function.call with a pinned index array)."""
    rng = np.random.default_rng(4)
    src = rng.uniform(-1, 1, (5000, 256)).astype(np.float32)
    with Ranks(1) as R:
        d_src = R.upload(src)
        for n_idx in (1, 4, 5, 4096, 100003):
            idx = rng.integers(0, 5000, n_idx).astype(np.uint64)
            hidx = _pinned_copy(idx)
            d_out = R.alloc(n_idx * 1024)
            check(lib().synk_gather_rows(R[0], _vp(d_src), _u64(5000), _u64(1024), hidx, _u64(n_idx), _vp(d_out)), "g")
            check(R.sync(), "sync")
            lib().synk_host_free(hidx)
            assert R.download(d_out, (n_idx, 256), np.float32).tobytes() == oracle.gather_rows(src, idx).tobytes()


@pytest.mark.parametrize("pinned", [False, True])
def test_gather_shared_index_lines_ragged_and_bad_index(oracle, pinned):
    """Each CTA's 8 warps share one 32-index line (gather.cu): lists that end
    inside a line, inside a warp's 4-row chunk, or after many grid strides are
    bit-exact, and one bad index anywhere in a line (first / last warp of a
    line, the final partial line) raises SYNK_EBOUNDS at the next sync while
    every other row is still gathered correctly."""
    rng = np.random.default_rng(11)
    src = rng.uniform(-1, 1, (3001, 64)).astype(np.float32)  # 256-byte rows: 32-byte lanes
    with Ranks(1) as R:
        d_src = R.upload(src)

        def gather(idx):
            d_idx = _pinned_copy(idx) if pinned else _vp(R.upload(idx))
            d_out = R.alloc(max(len(idx), 1) * 256)
            check(lib().synk_gather_rows(R[0], _vp(d_src), _u64(3001), _u64(256), d_idx, _u64(len(idx)),
                                         _vp(d_out)), "gather")
            rc = R.sync()
            if pinned:
                lib().synk_host_free(d_idx)
            return rc, R.download(d_out, (len(idx), 64), np.float32)

        for n_idx in (4097, 4099, 4128, 4133, 9 * 4096 + 7, 300007):
            idx = rng.integers(0, 3001, n_idx).astype(np.uint64)
            rc, got = gather(idx)
            assert rc == 0 and got.tobytes() == oracle.gather_rows(src, idx).tobytes(), n_idx
        n_idx = 4133  # 129 full lines + a partial line of 5
        for pos in (0, 3, 28, 31, 32, 4127, 4128, 4132):
            idx = rng.integers(0, 3001, n_idx).astype(np.uint64)
            idx[pos] = 3001
            rc, got = gather(idx)
            assert rc == -1, pos  # SYNK_EBOUNDS
            keep = np.arange(n_idx) != pos  # the bad row's content is kernel-defined (row 0 or zeros)
            want = oracle.gather_rows(src, np.where(idx == 3001, 0, idx).astype(np.uint64))
            assert got[keep].tobytes() == want[keep].tobytes(), pos
        assert R.sync() == 0  # flag cleared


def test_gather_inline_list_bit_exact(oracle):
    """synk_gather_rows_inline: a host list (pageable numpy memory) of at most
    SYNK_GATHER_INLINE_MAX indices rides in the launch as u32 kernel
    parameters. Every vector width (1/4/8/16/32-byte lanes by row size and
    alignment), ragged counts, and the golden vectors."""
    rng = np.random.default_rng(6)
    with Ranks(1) as R:
        for dtype, shape in ((np.float32, (10000, 256)), (np.float32, (513, 37)), (np.float64, (300, 8)),
                             (np.float32, (64, 10)), (np.float64, (5, 1)), (np.uint8, (777, 3)),
                             (np.float32, (300, 1028)), (np.float64, (257, 1024))):
            src = (rng.uniform(-1, 1, shape) * 100).astype(dtype)
            d_src = R.upload(src)
            for n_idx in (1, 3, 4, 5, 31, 33, 1000, 4095, 4096):
                idx = rng.integers(0, shape[0], n_idx).astype(np.uint64)
                d_out = R.alloc(n_idx * src[0].nbytes)
                check(lib().synk_gather_rows_inline(R[0], _vp(d_src), _u64(shape[0]), _u64(src[0].nbytes),
                                                    idx.ctypes.data_as(_vp), _u64(n_idx), _vp(d_out)), "gather inline")
                check(R.sync(), "sync")
                got = R.download(d_out, (n_idx,) + shape[1:], dtype)
                assert got.tobytes() == oracle.gather_rows(src, idx).tobytes(), (shape, n_idx)
        g = golden("gather.npz")
        for tag in ("f32", "f64"):
            src, idx = g[tag + "_src"], np.ascontiguousarray(g[tag + "_idx"].astype(np.uint64))
            d_src, d_out = R.upload(src), R.alloc(len(idx) * src[0].nbytes)
            check(lib().synk_gather_rows_inline(R[0], _vp(d_src), _u64(src.shape[0]), _u64(src[0].nbytes),
                                                idx.ctypes.data_as(_vp), _u64(len(idx)), _vp(d_out)), "gather inline")
            assert R.download(d_out, (len(idx),) + src.shape[1:], src.dtype).tobytes() == g[tag + "_w3_list"].tobytes()


def test_gather_inline_list_bounds_and_limits():
    """Out-of-range index: row 0 is read, SYNK_EBOUNDS at the next sync, then
    cleared (the device check's contract). Lists past the inline maximum or
    sources past 2^32 rows are refused (SYNK_EARG), nothing launched."""
    with Ranks(1) as R:
        src = np.arange(8, dtype=np.float64).reshape(4, 2)
        d_src, d_out = R.upload(src), R.alloc(32)
        bad = np.array([1, 4], np.uint64)
        check(lib().synk_gather_rows_inline(R[0], _vp(d_src), _u64(4), _u64(16), bad.ctypes.data_as(_vp), _u64(2),
                                            _vp(d_out)), "g")
        assert R.sync() == -1  # SYNK_EBOUNDS
        assert R.sync() == 0
        assert R.download(d_out, (2, 2), np.float64).tolist() == [[2.0, 3.0], [0.0, 1.0]]
        long = np.zeros(4097, np.uint64)
        assert lib().synk_gather_rows_inline(R[0], _vp(d_src), _u64(4), _u64(16), long.ctypes.data_as(_vp),
                                             _u64(4097), _vp(d_out)) != 0
        assert lib().synk_gather_rows_inline(R[0], _vp(d_src), _u64(1 << 33), _u64(16), bad.ctypes.data_as(_vp),
                                             _u64(2), _vp(d_out)) != 0
        assert lib().synk_gather_rows_inline(R[0], _vp(d_src), _u64(4), _u64(16), bad.ctypes.data_as(_vp), _u64(0),
                                             _vp(d_out)) == 0
        check(R.sync(), "sync")


def test_follow_up_fill_and_copy_after_inline_gather():
    """The inline gather releases its dependents at entry; a small fill or
    copy_small right behind it launches programmatically (PDL) and must still
    see the gather's rows: copy_small reads the gathered block, fill writes
    over part of it (its store lands after every gather store)."""
    rng = np.random.default_rng(7)
    src = rng.uniform(-1, 1, (20000, 256)).astype(np.float32)
    with Ranks(1) as R:
        d_src = R.upload(src)
        for it in range(20):
            idx = rng.integers(0, 20000, 4096).astype(np.uint64)
            d_out, d_cp = R.alloc(4096 * 1024), R.alloc(4096 * 1024)
            check(lib().synk_gather_rows_inline(R[0], _vp(d_src), _u64(20000), _u64(1024), idx.ctypes.data_as(_vp),
                                                _u64(4096), _vp(d_out)), "g")
            check(lib().synk_copy_small(R[0], _vp(d_cp), _vp(d_out + 4095 * 1024), _u64(1024)), "copy_small")
            check(lib().synk_gather_rows_inline(R[0], _vp(d_src), _u64(20000), _u64(1024), idx.ctypes.data_as(_vp),
                                                _u64(4096), _vp(d_out)), "g")
            check(lib().synk_fill(R[0], F32, _vp(d_out + 4095 * 1024), ctypes.c_double(it), _u64(256)), "fill")
            check(R.sync(), "sync")
            want = src[idx]
            assert R.download(d_cp, (1, 256), np.float32).tobytes() == want[4095:].tobytes()
            got = R.download(d_out, (4096, 256), np.float32)
            assert got[:4095].tobytes() == want[:4095].tobytes()
            assert (got[4095] == it).all()


def test_gather_out_of_range_raises_bounds():
    with Ranks(1) as R:
        src = np.zeros((4, 2))
        d_src, d_idx = R.upload(src), R.upload(np.array([1, 4], np.uint64))
        d_out = R.alloc(32)
        check(lib().synk_gather_rows(R[0], _vp(d_src), _u64(4), _u64(16), _vp(d_idx), _u64(2), _vp(d_out)), "g")
        assert R.sync() == -1  # SYNK_EBOUNDS, deferred to the phase-exit barrier
        assert R.sync() == 0   # flag cleared


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("op", ["sum", "max", "min", "prod"])
def test_combine_bit_exact(oracle, dtype, op):
    rng = np.random.default_rng(2)
    with Ranks(1) as R:
        for n in (1, 7, 4096, 100003):
            a = rng.uniform(-1, 1, n).astype(dtype)
            b = rng.uniform(-1, 1, n).astype(dtype)
            if n >= 7:  # reference NaN / signed-zero semantics: accumulator wins
                a[:4] = [np.nan, 1.0, -0.0, 0.0]
                b[:4] = [1.0, np.nan, 0.0, -0.0]
            da, db = R.upload(a), R.upload(b)
            check(lib().synk_combine(R[0], cabi.dt(dtype), OPS[op], _vp(da), _vp(db), _u64(n)), "combine")
            got = R.download(da, (n,), dtype)
            want = oracle.combine(a, b, op)
            if op in ("max", "min"):  # selects: every bit, NaN and signed zeros included
                assert got.tobytes() == want.tobytes()
            else:
                # arithmetic: bit-exact on every non-NaN result; a NaN result
                # stays NaN (x86 keeps the operand's payload, sm_100 returns
                # the canonical NaN -- payload bits carry no value)
                nan = np.isnan(want)
                assert np.array_equal(np.isnan(got), nan)
                assert got[~nan].tobytes() == want[~nan].tobytes()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_weighted_mean_scale_fill_bit_exact(oracle, dtype):
    rng = np.random.default_rng(3)
    with Ranks(1) as R:
        a = rng.uniform(-1, 1, 10001).astype(dtype)
        b = rng.uniform(-1, 1, 10001).astype(dtype)
        da, db = R.upload(a), R.upload(b)
        check(lib().synk_weighted_mean(R[0], cabi.dt(dtype), _vp(da), ctypes.c_double(3), _vp(db),
                                       ctypes.c_double(7), _u64(a.size)), "wmean")
        assert R.download(da, a.shape, dtype).tobytes() == oracle.weighted_mean(a, 3, b, 7).tobytes()
        dc = R.upload(a)
        check(lib().synk_scale(R[0], cabi.dt(dtype), _vp(dc), ctypes.c_double(1.0 / 3.0), _u64(a.size)), "scale")
        assert R.download(dc, a.shape, dtype).tobytes() == oracle.scale(a, 1.0 / 3.0).tobytes()
        assert lib().synk_weighted_mean(R[0], cabi.dt(dtype), _vp(da), ctypes.c_double(0), _vp(db),
                                        ctypes.c_double(0), _u64(a.size)) == -4  # ArgumentError


@pytest.mark.parametrize("op", ["sum", "mean", "max", "min", "prod"])
@pytest.mark.parametrize("count", [1, 3, 70])
def test_left_fold_bit_exact(oracle, op, count):
    rng = np.random.default_rng(4)
    with Ranks(1) as R:
        parts = [rng.uniform(-1, 1, 999).astype(np.float32) for _ in range(count)]
        weights = rng.integers(1, 9, count).astype(np.uint64)
        ptrs = [R.upload(p) for p in parts]
        out = R.alloc(999 * 4)
        w = np.ascontiguousarray(weights)
        check(lib().synk_left_fold(R[0], F32, OPS[op], _vp(out), ptr_array(ptrs), w.ctypes.data_as(_vp),
                                   ctypes.c_uint32(count), _u64(999)), "fold")
        got = R.download(out, (999,), np.float32)
        assert got.tobytes() == oracle.left_fold(parts, op, weights).tobytes()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_column_stats(oracle, dtype):
    rng = np.random.default_rng(5)
    with Ranks(1) as R:
        for rows, cols in ((1, 3), (37, 5), (5000, 1024), (20000, 300)):
            x = rng.uniform(-1, 1, (rows, cols)).astype(dtype)
            dx = R.upload(x)
            ds, dm, dn = R.alloc(cols * x.itemsize), R.alloc(cols * x.itemsize), R.alloc(cols * x.itemsize)
            check(lib().synk_column_stats(R[0], cabi.dt(dtype), _vp(dx), _u64(rows), _u64(cols), _vp(ds), _vp(dm),
                                          _vp(dn)), "colstats")
            s = R.download(ds, (cols,), dtype)
            assert R.download(dm, (cols,), dtype).tobytes() == oracle.column_fold(x, "max").tobytes()
            assert R.download(dn, (cols,), dtype).tobytes() == oracle.column_fold(x, "min").tobytes()
            # Sum: f64 accumulation in a fixed tree order; the reference folds
            # sequentially in T. Tolerance: elem_err <= rows * eps(T) (the
            # reference's own recursive-summation bound, Higham 4.2).
            tol = rows * float(np.finfo(dtype).eps)
            exact = np.array([float(np.sum(x[:, c].astype(np.longdouble))) for c in range(cols)])
            if dtype == np.float32:  # f64 accumulation of f32 data: one final rounding
                assert oracle.elem_err(s, exact) <= 2 * float(np.finfo(np.float32).eps)
            else:
                assert oracle.elem_err(s, exact) <= tol
            assert oracle.elem_err(s, oracle.column_fold(x, "sum")) <= tol


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_all_reduce_bitwise_vs_reference_golden(world):
    g = golden("collectives.npz")
    with Ranks(world) as R:
        for tag, dtype in (("f32", np.float32), ("f64", np.float64)):
            vals = g["in_%s_w%d" % (tag, world)]
            for op in ("sum", "mean", "max", "min", "prod"):
                ptrs = [R.upload(vals[r], r) for r in range(world)]
                arr = ptr_array(ptrs)
                for r in range(world):  # every rank issues its chunk (one phase)
                    check(lib().synk_all_reduce(R[r], world, cabi.dt(dtype), OPS[op], arr, _u64(vals.shape[1])), "ar")
                for r in range(world):
                    check(R.sync(r), "sync")
                ref = g["allreduce_%s_%s_w%d" % (op, tag, world)]
                for r in range(world):
                    assert R.download(ptrs[r], ref.shape, dtype, r).tobytes() == ref.tobytes(), (op, tag, r)


def test_all_reduce_large_and_ragged(oracle):
    rng = np.random.default_rng(6)
    for world, n in ((2, 1), (3, 17), (4, 1 << 20), (8, 1000003), (5, 33)):
        vals = [rng.uniform(-1, 1, n).astype(np.float32) for _ in range(world)]
        with Ranks(world) as R:
            ptrs = [R.upload(v, r) for r, v in enumerate(vals)]
            arr = ptr_array(ptrs)
            for r in range(world):
                check(lib().synk_all_reduce(R[r], world, F32, OPS["mean"], arr, _u64(n)), "ar")
            for r in range(world):
                check(R.sync(r), "sync")
            ref = oracle.tree_fold(vals, "mean")
            for r in range(world):
                assert R.download(ptrs[r], (n,), np.float32, r).tobytes() == ref.tobytes()


def test_broadcast_and_tree_reduce(oracle):
    rng = np.random.default_rng(7)
    world, n = 4, 5000
    vals = [rng.uniform(-1, 1, n) for _ in range(world)]
    with Ranks(world) as R:
        ptrs = [R.upload(v, r) for r, v in enumerate(vals)]
        out = R.alloc(n * 8, 1)
        check(lib().synk_tree_reduce(R[1], world, F64, OPS["sum"], ptr_array(ptrs), _u64(n), _vp(out)), "reduce")
        assert R.download(out, (n,), np.float64, 1).tobytes() == oracle.tree_fold(vals, "sum").tobytes()
        arr = ptr_array(ptrs)
        for r in range(world):
            check(lib().synk_broadcast(R[r], world, 2, arr, _u64(n * 8)), "bcast")
        for r in range(world):
            check(R.sync(r), "sync")
        for r in range(world):
            assert R.download(ptrs[r], (n,), np.float64, r).tobytes() == vals[2].tobytes()


def _rule_args(rule):
    return {"sgd": [0.0], "momentum": [0.9], "rmsprop": [0.9, 1e-6], "adam": [0.9, 0.999, 1e-8]}[rule]


def _oracle_step(oracle, rule, p, g, aux, lr, t):
    h = _rule_args(rule)
    if rule == "sgd":
        return oracle.sgd(p, g, lr), []
    if rule == "momentum":
        p2, v = oracle.momentum(p, aux[0], g, h[0], lr)
        return p2, [v]
    if rule == "rmsprop":
        p2, a = oracle.rmsprop(p, aux[0], g, h[0], h[1], lr)
        return p2, [a]
    p2, m, v = oracle.adam(p, aux[0], aux[1], g, h[0], h[1], h[2], lr, t)
    return p2, [m, v]


@pytest.mark.parametrize("rule", ["sgd", "momentum", "rmsprop", "adam"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_optimizer_step_bit_exact(oracle, rule, dtype):
    rng = np.random.default_rng(8)
    n = 12345
    naux = {"sgd": 0, "momentum": 1, "rmsprop": 1, "adam": 2}[rule]
    p = rng.uniform(-1, 1, n).astype(dtype)
    aux = [np.abs(rng.uniform(0, 0.1, n)).astype(dtype) for _ in range(naux)]
    hyper = np.array(_rule_args(rule), np.float64)
    with Ranks(1) as R:
        dp = R.upload(p)
        daux = [R.upload(a) for a in aux]
        for t in (1, 2, 3):
            g = rng.uniform(-1, 1, n).astype(dtype)
            dg = R.upload(g)
            check(lib().synk_optimizer_step(R[0], cabi.dt(dtype), RULES[rule], hyper.ctypes.data_as(_vp),
                                            ctypes.c_double(0.01), _u64(t), _vp(dp), _vp(dg),
                                            _vp(daux[0] if naux > 0 else None), _vp(daux[1] if naux > 1 else None),
                                            _u64(n)), "step")
            p, aux = _oracle_step(oracle, rule, p, g, aux, 0.01, t)
            assert R.download(dp, (n,), dtype).tobytes() == p.tobytes()
            for da, a in zip(daux, aux):
                assert R.download(da, (n,), dtype).tobytes() == a.tobytes()


@pytest.mark.parametrize("rule", ["sgd", "adam"])
@pytest.mark.parametrize("coherent,grads_local", [(True, False), (False, False), (True, True)])
def test_fused_all_reduce_step_bit_exact(oracle, rule, coherent, grads_local):
    """Gradient tree all-reduce (mean) + update in one kernel per rank =
    reference all_reduce(Mean) followed by the per-rank step. With
    SYNK_STEP_GRADS_LOCAL (deferred all-gather) rank r writes the reduced
    gradient into its own replica's chunk only; every other byte of the
    gradient replicas is left as it was."""
    rng = np.random.default_rng(9)
    world, n = 4, 40961
    naux = 2 if rule == "adam" else 0
    base = rng.uniform(-1, 1, n).astype(np.float32)
    params = [base.copy() if coherent else rng.uniform(-1, 1, n).astype(np.float32) for _ in range(world)]
    aux = [[np.zeros(n, np.float32) for _ in range(naux)] for _ in range(world)]
    grads = [rng.uniform(-1, 1, n).astype(np.float32) for _ in range(world)]
    hyper = np.array(_rule_args(rule), np.float64)
    with Ranks(world) as R:
        dp = [R.upload(params[r], r) for r in range(world)]
        dg = [R.upload(grads[r], r) for r in range(world)]
        da = [[R.upload(aux[r][k], r) for r in range(world)] for k in range(naux)]
        a0 = ptr_array(da[0]) if naux > 0 else None
        a1 = ptr_array(da[1]) if naux > 1 else None
        P, G = ptr_array(dp), ptr_array(dg)
        for r in range(world):
            check(lib().synk_all_reduce_step(R[r], world, F32, OPS["mean"], RULES[rule], hyper.ctypes.data_as(_vp),
                                             ctypes.c_double(0.01), _u64(1), P, G, a0, a1, _u64(n),
                                             (1 if coherent else 0) | (2 if grads_local else 0)), "fused")
        for r in range(world):
            check(R.sync(r), "sync")
        g_ref = oracle.tree_fold(grads, "mean")
        for r in range(world):
            p_ref, aux_ref = _oracle_step(oracle, rule, params[r], g_ref, aux[r], 0.01, 1)
            got = R.download(dg[r], (n,), np.float32, r)
            if grads_local:
                lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
                check(lib().synk_chunk_range(_u64(n), world, r, ctypes.byref(lo), ctypes.byref(hi)), "chunk")
                want = grads[r].copy()
                want[lo.value:hi.value] = g_ref[lo.value:hi.value]
                assert got.tobytes() == want.tobytes()
            else:
                assert got.tobytes() == g_ref.tobytes()
            assert R.download(dp[r], (n,), np.float32, r).tobytes() == p_ref.tobytes()
            for k in range(naux):
                assert R.download(da[k][r], (n,), np.float32, r).tobytes() == aux_ref[k].tobytes()


def _mlp(R, params, dims, x, y, dtype):
    dims_a = np.array(dims, np.uint64)
    ws = _u64(0)
    check(lib().synk_mlp_workspace_bytes(cabi.dt(dtype), dims_a.ctypes.data_as(_vp), ctypes.c_uint32(len(dims) - 1),
                                         _u64(x.shape[0]), ctypes.byref(ws)), "ws")
    d_ws, d_p, d_x, d_y = R.alloc(ws.value), R.upload(params), R.upload(x), R.upload(y)
    d_loss, d_g = R.alloc(8), R.alloc(params.nbytes)
    check(lib().synk_mlp_loss_grad(R[0], cabi.dt(dtype), dims_a.ctypes.data_as(_vp), ctypes.c_uint32(len(dims) - 1),
                                   _vp(d_p), _vp(d_x), _vp(d_y), _u64(x.shape[0]), _vp(d_loss), _vp(d_g), _vp(d_ws),
                                   ws), "mlp")
    return float(R.download(d_loss, (), np.float64)), R.download(d_g, params.shape, dtype)


def test_mlp_loss_grad_vs_reference_golden(oracle):
    g = golden("mlp.npz")
    with Ranks(1) as R:
        loss, grad = _mlp(R, g["params"], [784, 512, 10], g["x"], g["y"], np.float32)
        # fp32 kernel vs the reference's f64-internal loops (north_star: 1e-5 fp32)
        assert oracle.elem_err(loss, float(g["loss"])) <= 1e-5
        assert oracle.elem_err(grad, g["grad"]) <= 1e-5
        loss, grad = _mlp(R, g["params64"], [8, 16, 16, 16, 4], g["x64"], g["y64"], np.float64)
        assert oracle.elem_err(loss, float(g["loss64"])) <= 1e-12
        assert oracle.elem_err(grad, g["grad64"]) <= 1e-12


def test_gather_from_host_registered_memory(sk, oracle):
    """An index list in cudaHostRegister'd (page-locked, not cudaHostAlloc'd)
    memory is borrowed in place and read by the gather kernel through its
    device address (synk_host_device_ptr), bit-exact."""
    import torch

    rng = np.random.default_rng(8)
    src = rng.uniform(-1, 1, (3000, 64)).astype(np.float32)
    idx = rng.integers(0, 3000, 777).astype(np.int64)
    cudart = torch.cuda.cudart()
    for a in (src, idx):
        assert int(cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)) == 0
    try:
        with sk.Pool(workers=2) as pool:
            f = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
            sk.distribute(pool)
            (got,) = f.call([src], indexes=idx)
            assert got.tobytes() == oracle.gather_rows(src, idx.astype(np.uint64)).tobytes()
    finally:
        for a in (src, idx):
            cudart.cudaHostUnregister(a.ctypes.data)
