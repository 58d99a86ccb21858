"""fp32-accurate tensor-core GEMM (synk_gemm_f32x3, 3xTF32 with per-K-block
TMEM flush into fp32 registers) and its operand staging (synk_tf32_split),
checked against fp64 numpy.

Tolerance: the f32 example function's bar is 1e-5 relative (BASELINE
north_star). Because the tcgen05 accumulator only ever holds one 32-element K
block, the error must NOT grow with K the way a single long TMEM chain does
(~6.7e-9 relative per product, profiles/r01_tcgen05_tf32_accumulation.txt):
the mean signed error is held to 5e-7 at every K (a plain chain reaches
5.5e-5 at K=8192) and the max error to the 1e-5 bar.
"""

import ctypes

import numpy as np
import pytest

from cabi import Ranks, check, lib

pytestmark = pytest.mark.gpu
_u64 = ctypes.c_uint64
_vp = ctypes.c_void_p
EPI = {"store": 0, "bias": 1, "bias_tanh": 2, "tanh_grad": 3}


def rna_tf32(x):
    """cvt.rna.tf32.f32: round to 10 mantissa bits, ties away from zero."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x1000) & ~np.uint64(0x1FFF)
    return u.astype(np.uint32).view(np.float32)


def split_host(x):
    hi = rna_tf32(x)
    lo = rna_tf32((x - hi).astype(np.float32))
    return hi, lo


def pad4(n):
    return (n + 3) // 4 * 4


def dev_split(R, x, rowmap=None, want_rows=True, want_t=False):
    """Upload x (fp32 [rows, cols]) and split it on the device."""
    rows = len(rowmap) if rowmap is not None else x.shape[0]
    cols = x.shape[1]
    dx = R.upload(np.ascontiguousarray(x, np.float32))
    dmap = R.upload(np.asarray(rowmap, np.uint64)) if rowmap is not None else 0
    ld, ldt = pad4(cols), pad4(rows)
    hi = R.alloc(rows * ld * 4) if want_rows else 0
    lo = R.alloc(rows * ld * 4) if want_rows else 0
    hit = R.alloc(cols * ldt * 4) if want_t else 0
    lot = R.alloc(cols * ldt * 4) if want_t else 0
    check(lib().synk_tf32_split(R[0], _vp(dx), _vp(dmap or None), _u64(rows), _u64(cols), _u64(cols), _vp(hi or None),
                                _vp(lo or None), _u64(ld), _vp(hit or None), _vp(lot or None), _u64(ldt)), "split")
    return (hi, lo, ld), (hit, lot, ldt)


def gemm(R, a, b, epi="store", bias=None, act=None, outs=("c",)):
    """epi(a @ b.T) through synk_gemm_f32x3; returns the requested outputs."""
    M, K = a.shape
    N = b.shape[0]
    (ahi, alo, lda), _ = dev_split(R, a)
    (bhi, blo, ldb), _ = dev_split(R, b)
    c = R.alloc(M * N * 4) if "c" in outs else 0
    ldh, ldt = pad4(N), pad4(M)
    h = R.alloc(M * ldh * 4) if "split" in outs else 0
    l = R.alloc(M * ldh * 4) if "split" in outs else 0
    ht = R.alloc(N * ldt * 4) if "split_t" in outs else 0
    lt = R.alloc(N * ldt * 4) if "split_t" in outs else 0
    dbias = R.upload(bias.astype(np.float32)) if bias is not None else 0
    dact = R.upload(act.astype(np.float32)) if act is not None else 0
    check(lib().synk_gemm_f32x3(R[0], _u64(M), _u64(N), _u64(K), _vp(ahi), _vp(alo), _u64(lda), _vp(bhi), _vp(blo),
                                _u64(ldb), EPI[epi], _vp(c or None), _u64(N), _vp(dbias or None), _vp(dact or None),
                                _u64(N), _vp(h or None), _vp(l or None), _u64(ldh), _vp(ht or None), _vp(lt or None),
                                _u64(ldt)), "gemm_f32x3")
    check(R.sync(), "sync")
    res = {}
    if c:
        res["c"] = R.download(c, (M, N), np.float32)
    if h:
        res["hi"] = R.download(h, (M, ldh), np.float32)[:, :N]
        res["lo"] = R.download(l, (M, ldh), np.float32)[:, :N]
    if ht:
        res["hi_t"] = R.download(ht, (N, ldt), np.float32)[:, :M]
        res["lo_t"] = R.download(lt, (N, ldt), np.float32)[:, :M]
    return res


def rel_err(got, want):
    scale = np.maximum(1.0, np.abs(want))
    return float(np.max(np.abs(got.astype(np.float64) - want) / scale))


# C1's five products (784-512-10, batch 256) plus ragged, single-tile,
# split and unsplit shapes and a long K (where a plain TMEM chain drifts).
SHAPES = [(256, 512, 784), (256, 10, 512), (513, 10, 256), (256, 512, 10), (785, 512, 256), (1, 1, 1),
          (128, 128, 32), (300, 130, 1000), (64, 700, 4096), (256, 256, 8192),
          (2048, 2048, 256), (1700, 2100, 40)]  # the last two: >= 148 tiles of 128x128 -> 128-wide tiles, no split


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_f32x3_matches_fp64_flat_in_k(M, N, K):
    rng = np.random.default_rng(M * 31 + N * 7 + K)
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        got = gemm(R, a, b)["c"]
    scale = np.sqrt(K) / 3 + 1.0  # typical |C| of uniform(-1,1) products
    err = (got.astype(np.float64) - want) / scale
    assert float(np.max(np.abs(err))) <= 1e-5, float(np.max(np.abs(err)))
    assert abs(float(np.mean(err))) <= 5e-7  # no K-proportional accumulator bias


def test_f32x3_all_positive_long_k_has_no_drift():
    """All-positive operands: every accumulator rounding has the same sign,
    the worst case for a biased accumulator (K=8192: a plain TMEM chain is
    off by ~5.5e-5 relative, r01_tcgen05_tf32_accumulation.txt)."""
    rng = np.random.default_rng(5)
    M, N, K = 256, 256, 8192
    a = rng.uniform(0, 1, (M, K)).astype(np.float32)
    b = rng.uniform(0, 1, (N, K)).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        got = gemm(R, a, b)["c"]
    rel = (got.astype(np.float64) - want) / want
    assert float(np.max(np.abs(rel))) <= 3e-6, float(np.max(np.abs(rel)))
    assert abs(float(np.mean(rel))) <= 5e-7, float(np.mean(rel))


@pytest.mark.parametrize("M,N,K", [(256, 512, 784), (256, 10, 512), (100, 40, 64), (1664, 1800, 96)])
@pytest.mark.parametrize("epi", ["bias", "bias_tanh", "tanh_grad"])
def test_f32x3_epilogues_and_split_outputs(M, N, K, epi):
    rng = np.random.default_rng(M + N + K + len(epi))
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32) / np.sqrt(K)
    b = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, N).astype(np.float32)
    act = np.tanh(rng.uniform(-2, 2, (M, N))).astype(np.float32)
    z = a.astype(np.float64) @ b.astype(np.float64).T
    want = {"bias": z + bias, "bias_tanh": np.tanh(z + bias), "tanh_grad": z * (1.0 - act.astype(np.float64) ** 2)}[epi]
    with Ranks(1) as R:
        res = gemm(R, a, b, epi, bias=bias if epi != "tanh_grad" else None,
                   act=act if epi == "tanh_grad" else None, outs=("c", "split", "split_t"))
    assert rel_err(res["c"], want) <= 2e-6
    hi, lo = split_host(res["c"])
    np.testing.assert_array_equal(res["hi"], hi)
    np.testing.assert_array_equal(res["lo"], lo)
    np.testing.assert_array_equal(res["hi_t"], hi.T)
    np.testing.assert_array_equal(res["lo_t"], lo.T)


def test_f32x3_deterministic():
    rng = np.random.default_rng(9)
    a = rng.uniform(-1, 1, (256, 784)).astype(np.float32)
    b = rng.uniform(-1, 1, (512, 784)).astype(np.float32)
    with Ranks(1) as R:
        r1 = gemm(R, a, b)["c"]
        r2 = gemm(R, a, b)["c"]
    np.testing.assert_array_equal(r1, r2)


@pytest.mark.parametrize("rows,cols", [(256, 784), (33, 10), (1, 1), (513, 70)])
def test_tf32_split_matches_host(rows, cols):
    rng = np.random.default_rng(rows + cols)
    x = (rng.standard_normal((rows, cols)) * 10.0 ** rng.integers(-6, 6, (rows, cols))).astype(np.float32)
    with Ranks(1) as R:
        (h, l, ld), (ht, lt, ldt) = dev_split(R, x, want_t=True)
        hi = R.download(h, (rows, ld), np.float32)[:, :cols]
        lo = R.download(l, (rows, ld), np.float32)[:, :cols]
        hit = R.download(ht, (cols, ldt), np.float32)[:, :rows]
        lot = R.download(lt, (cols, ldt), np.float32)[:, :rows]
    eh, el = split_host(x)
    np.testing.assert_array_equal(hi, eh)
    np.testing.assert_array_equal(lo, el)
    np.testing.assert_array_equal(hit, eh.T)
    np.testing.assert_array_equal(lot, el.T)
    # hi + lo carries x to ~2^-22 relative
    assert np.all(np.abs(eh.astype(np.float64) + el - x) <= np.abs(x.astype(np.float64)) * 2.0 ** -21 + 1e-45)


def test_tf32_split_rowmap_gathers():
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (1000, 70)).astype(np.float32)
    idx = rng.integers(0, 1000, 129)
    with Ranks(1) as R:
        (h, l, ld), (ht, lt, ldt) = dev_split(R, x, rowmap=idx, want_t=True)
        hi = R.download(h, (129, ld), np.float32)[:, :70]
        hit = R.download(ht, (70, ldt), np.float32)[:, :129]
    eh, _ = split_host(x[idx])
    np.testing.assert_array_equal(hi, eh)
    np.testing.assert_array_equal(hit, eh.T)


class Tf32Rows(ctypes.Structure):
    _fields_ = [("hi", _vp * 64), ("lo", _vp * 64), ("len", _u64 * 64), ("count", ctypes.c_uint32),
                ("value", ctypes.c_float)]


def test_tf32_fill_rows():
    with Ranks(1) as R:
        bufs = [(R.alloc(1000 * 4), R.alloc(1000 * 4), n) for n in (1000, 5, 257)]
        rows = Tf32Rows()
        for i, (h, l, n) in enumerate(bufs):
            rows.hi[i], rows.lo[i], rows.len[i] = h, l, n
        rows.count, rows.value = len(bufs), 1.0
        check(lib().synk_tf32_fill_rows(R[0], ctypes.byref(rows)), "fill")
        check(R.sync(), "sync")
        for h, l, n in bufs:
            assert np.all(R.download(h, (n,), np.float32) == 1.0)
            assert np.all(R.download(l, (n,), np.float32) == 0.0)


def _mlp_ex(R, compute, params, dims, x, y):
    dims_a = np.array(dims, np.uint64)
    ws = _u64(0)
    check(lib().synk_mlp_workspace_bytes_ex(1, compute, dims_a.ctypes.data_as(_vp), ctypes.c_uint32(len(dims) - 1),
                                            _u64(x.shape[0]), ctypes.byref(ws)), "ws")
    d_ws, d_p, d_x, d_y = R.alloc(ws.value), R.upload(params), R.upload(x), R.upload(y)
    d_loss, d_g = R.alloc(8), R.alloc(params.nbytes)
    check(lib().synk_mlp_loss_grad_ex(R[0], 1, compute, dims_a.ctypes.data_as(_vp), ctypes.c_uint32(len(dims) - 1),
                                      _vp(d_p), _vp(d_x), _vp(d_y), _u64(x.shape[0]), _vp(d_loss), _vp(d_g), _vp(d_ws),
                                      ws), "mlp")
    return float(R.download(d_loss, (), np.float64)), R.download(d_g, params.shape, np.float32)


@pytest.mark.parametrize("path", ["tensor_cores", "ffma"])
def test_c1_loss_grad_both_f32_paths_vs_reference_golden(path, oracle, monkeypatch):
    """C1's loss/gradient (784-512-10 f32, batch 256) on the default f32 path
    (3xTF32 tensor cores, SYNK_MLP_NATIVE) and on the FFMA A/B path, each
    against the unmodified reference's golden at the 1e-5 fp32 bar; the
    explicit SYNK_MLP_F32_TC mode is bitwise the default."""
    from conftest import golden

    g = golden("mlp.npz")
    if path == "ffma":
        monkeypatch.setenv("SYNK_MLP_F32", "ffma")
    else:
        monkeypatch.delenv("SYNK_MLP_F32", raising=False)
    with Ranks(1) as R:
        loss, grad = _mlp_ex(R, 0, g["params"], [784, 512, 10], g["x"], g["y"])
        assert oracle.elem_err(loss, float(g["loss"])) <= 1e-5
        assert oracle.elem_err(grad, g["grad"]) <= 1e-5
        if path == "tensor_cores":
            loss2, grad2 = _mlp_ex(R, 2, g["params"], [784, 512, 10], g["x"], g["y"])
            assert loss2 == loss and grad2.tobytes() == grad.tobytes()


def test_f32_tc_deep_mlp_vs_oracle(oracle):
    """A 4-layer f32 MLP (every product kind incl. dX feeding another dX:
    the epilogue's row-major split of delta) against the oracle."""
    rng = np.random.default_rng(12)
    dims = [100, 70, 130, 40, 9]
    n = 77
    params = np.concatenate([np.concatenate([rng.uniform(-0.3, 0.3, dims[i] * dims[i + 1]),
                                             rng.uniform(-0.1, 0.1, dims[i + 1])]) for i in range(4)]).astype(np.float32)
    x = rng.uniform(-1, 1, (n, dims[0])).astype(np.float32)
    y = rng.uniform(-1, 1, (n, dims[-1])).astype(np.float32)
    with Ranks(1) as R:
        loss, grad = _mlp_ex(R, 2, params, dims, x, y)
    ref_loss, ref_grad = oracle.mlp_loss_grad(params, dims, x, y)
    assert oracle.elem_err(loss, ref_loss) <= 1e-5
    assert oracle.elem_err(grad, ref_grad) <= 1e-5
