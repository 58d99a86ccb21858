"""tcgen05 tensor-core GEMM (synk_gemm_tc) parity against an fp64 reference.

Tolerances: 3xTF32 keeps fp32-level error (elem_err <= 1e-5 relative to the
problem scale at K <= 4096); single-pass TF32 and BF16 are checked at their
own mantissa widths (2^-10 / 2^-7 relative, times sqrt(K) growth headroom).
"""

import ctypes

import numpy as np
import pytest

from cabi import F32, Ranks, check, lib

pytestmark = pytest.mark.gpu
_u64 = ctypes.c_uint64
_vp = ctypes.c_void_p
BF16 = 3
KIND = {"bf16": 0, "tf32": 1, "tf32x3": 2}
EPI = {"store": 0, "bias": 1, "bias_tanh": 2, "tanh_grad": 3}


def pad(n, m):
    return (n + m - 1) // m * m


def prep(R, x, transpose, mode):
    """Stage a host fp32 matrix for the GEMM (K-major, 16-byte rows)."""
    rows, cols = x.shape
    orows, ocols = (cols, rows) if transpose else (rows, cols)
    ld = pad(ocols, 8)
    dx = R.upload(np.ascontiguousarray(x, np.float32))
    es = 2 if mode == 1 else 4
    hi = R.alloc(orows * ld * es)
    lo = R.alloc(orows * ld * 4) if mode == 0 else 0
    check(lib().synk_gemm_prep(R[0], F32, _vp(dx), _u64(rows), _u64(cols), _u64(cols), int(transpose), mode,
                               _vp(hi), _vp(lo or None), _u64(orows), _u64(ocols), _u64(ld)), "prep")
    return hi, lo, ld


def gemm(R, kind, a, b, epi="store", bias=None, act=None, want_t=False):
    """C = epi(a @ b.T) with a: [M,K], b: [N,K] (host fp32)."""
    M, K = a.shape
    N = b.shape[0]
    mode = {"bf16": 1, "tf32": 2, "tf32x3": 0}[kind]
    ahi, alo, lda = prep(R, a, False, mode)
    bhi, blo, ldb = prep(R, b, False, mode)
    c = R.alloc(M * N * 4)
    ct = R.alloc(M * N * 4) if want_t else 0
    dbias = R.upload(bias.astype(np.float32)) if bias is not None else 0
    dact = R.upload(act.astype(np.float32)) if act is not None else 0
    check(lib().synk_gemm_tc(R[0], KIND[kind], _u64(M), _u64(N), _u64(K), _vp(ahi), _vp(alo or None), _u64(lda),
                             _vp(bhi), _vp(blo or None), _u64(ldb), EPI[epi], F32, _vp(c), _u64(N), _vp(ct or None),
                             _u64(M), _vp(dbias or None), _vp(dact or None), _u64(N)), "gemm")
    check(R.sync(), "sync")
    out = R.download(c, (M, N), np.float32)
    out_t = R.download(ct, (N, M), np.float32) if want_t else None
    return out, out_t


def rel_err(got, want):
    scale = np.maximum(1.0, np.abs(want))
    return float(np.max(np.abs(got.astype(np.float64) - want) / scale))


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 512, 784), (200, 10, 512), (784, 512, 256), (1, 1, 8),
                                   (300, 130, 1000)])
def test_tf32x3_matches_fp64(M, N, K):
    rng = np.random.default_rng(M * 7 + N + K)
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        got, got_t = gemm(R, "tf32x3", a, b, want_t=True)
    # tcgen05's fp32 accumulator rounds with a bias of ~6.7e-9 per accumulated
    # product (profiles/r01_tcgen05_tf32_accumulation.txt): 3 passes x K products.
    assert rel_err(got, want) <= 1e-6 + 2.5e-8 * 3 * K
    np.testing.assert_array_equal(got_t, got.T)


@pytest.mark.parametrize("kind,tol", [("tf32", 2.0 ** -10), ("bf16", 2.0 ** -7)])
def test_single_pass_kinds(kind, tol):
    rng = np.random.default_rng(1)
    M, N, K = 256, 384, 1024
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        got, _ = gemm(R, kind, a, b)
    assert rel_err(got, want) <= tol * np.sqrt(K)
    assert rel_err(got, want) > 0  # it really ran at reduced precision


def bf16_round(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16  # round-to-nearest-even to bf16
    return u.astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("M,N,K", [(4096, 2048, 512), (1000, 4000, 600), (8192, 384, 2048)])
def test_bf16_persistent_many_tiles(M, N, K):
    """Shapes that take the persistent 128x256 path with more tiles than SMs
    (both TMEM accumulators cycle) and ragged edges; exact products of
    bf16-rounded inputs, so the only error is fp32 accumulation."""
    rng = np.random.default_rng(M + N + K)
    a = bf16_round(rng.uniform(-1, 1, (M, K)))
    b = bf16_round(rng.uniform(-1, 1, (N, K)))
    want = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        got, got_t = gemm(R, "bf16", a, b, want_t=True)
    # accumulator rounding only (~7e-9 x K relative to the running partial sums,
    # whose magnitude can exceed the final value): bugs show up as O(1) errors
    assert rel_err(got, want) <= 1e-6 + 5e-8 * K
    np.testing.assert_array_equal(got_t, got.T)


@pytest.mark.parametrize("M,N,K", [(1, 136, 64), (129, 257, 100), (300, 520, 1000), (255, 130, 8), (513, 4100, 72)])
def test_bf16_pair_kernel_ragged_edges(M, N, K):
    """The CTA-pair (cta_group::2) persistent kernel on ragged shapes: a pair
    tile whose odd CTA holds only out-of-range A rows (M <= 128), partial N
    tiles, K below one block, more tiles than pairs with a ragged last round;
    C and C^T against fp64 on bf16-exact inputs."""
    rng = np.random.default_rng(M * 3 + N + K)
    a = bf16_round(rng.uniform(-1, 1, (M, K)))
    b = bf16_round(rng.uniform(-1, 1, (N, K)))
    want = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        got, got_t = gemm(R, "bf16", a, b, want_t=True)
    assert rel_err(got, want) <= 1e-6 + 5e-8 * K
    np.testing.assert_array_equal(got_t, got.T)


def test_fused_epilogues():
    rng = np.random.default_rng(2)
    M, N, K = 192, 160, 256
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (N, K)).astype(np.float32) * 0.1
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    act = np.tanh(rng.uniform(-1, 1, (M, N))).astype(np.float32)
    z = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        got, _ = gemm(R, "tf32x3", a, b, "bias", bias)
        assert rel_err(got, z + bias) <= 1e-5
        got, _ = gemm(R, "tf32x3", a, b, "bias_tanh", bias)
        assert rel_err(got, np.tanh(z + bias)) <= 1e-5
        got, _ = gemm(R, "tf32x3", a, b, "tanh_grad", act=act)
        assert rel_err(got, z * (1 - act.astype(np.float64) ** 2)) <= 1e-5


@pytest.mark.parametrize("world", [1, 2])
def test_bf16_tensor_core_mlp_vs_oracle(sk, oracle, world):
    """The wide-MLP path (compute='bf16'): every dense product on tcgen05 with bf16
    operands. Checked against the reference's f64 math on the same f32 inputs:
    relative Frobenius error of the gradient <= 2e-2 and loss <= 1e-2 (bf16 has
    8 mantissa bits; tolerance stated here, not tuned per run)."""
    cfg = sk.MlpConfig(in_dim=256, width=512, out_dim=100, layers=3, seed=4)
    x, y = sk.mlp_make_dataset(1024, cfg, seed=5, dtype="f32")
    params = sk.mlp_init_params(cfg, "f32")
    flat = np.concatenate([p.ravel() for p in params])
    ref_loss, ref_grad = oracle.mlp_loss_grad(flat, [256, 512, 512, 100], x, y)
    with sk.Pool(workers=world) as pool:
        block = sk.ParamBlock.create(pool, params)
        f = sk.mlp_grad_function(pool, block, compute="bf16")
        sk.distribute(pool)
        (loss,) = f.call_serial([x, y])
        g = block.grads.get(0)
        assert abs(loss - ref_loss) / ref_loss <= 1e-2
        assert np.linalg.norm(g - ref_grad) / np.linalg.norm(ref_grad) <= 2e-2
        # parallel call: shard-mean gradients, row-weighted loss (same bar)
        (ploss,) = f.call([x, y])
        assert abs(ploss - ref_loss) / ref_loss <= 1e-2


@pytest.mark.parametrize("M,N,K,epi", [(8192, 100, 4096, "bias"), (4096, 100, 8192, "store"), (300, 64, 2000, "bias")])
def test_bf16_split_k_small_n(M, N, K, epi):
    """Few output tiles + long K take the split-K path (fp32 partial planes,
    fixed-order fold with the bias): same accuracy bar as the unsplit kernel,
    and run-to-run bitwise deterministic."""
    rng = np.random.default_rng(M + N + K)
    a = bf16_round(rng.uniform(-1, 1, (M, K)))
    b = bf16_round(rng.uniform(-1, 1, (N, K)))
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64).T
    if epi == "bias":
        want = want + bias
    with Ranks(1) as R:
        got, _ = gemm(R, "bf16", a, b, epi, bias if epi == "bias" else None)
        again, _ = gemm(R, "bf16", a, b, epi, bias if epi == "bias" else None)
    assert rel_err(got, want) <= 1e-6 + 5e-8 * K
    assert got.tobytes() == again.tobytes()


def _split_case(M, N, K, epi):
    rng = np.random.default_rng(M * 3 + N + K)
    a = bf16_round(rng.uniform(-1, 1, (M, K)))
    b = bf16_round(rng.uniform(-1, 1, (N, K)))
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    with Ranks(1) as R:
        got, _ = gemm(R, "bf16", a, b, epi, bias if epi == "bias" else None)
    return a, b, bias, got


@pytest.mark.parametrize("M,N,K,epi", [(8192, 100, 4096, "bias"), (4097, 100, 8192, "store"), (1000, 100, 1536, "bias"),
                                       (200, 10, 4096, "bias"), (300, 64, 2000, "store")])
def test_split_k_cluster_fold_matches_planes(M, N, K, epi, tmp_path):
    """Split-K with <= 8 splits folds its partials through distributed shared
    memory inside a cluster (2, 3, 4 and 8 splits here; ragged M, N and fold
    rows). It must equal the fp32-planes + fold-kernel path bit for bit (same
    order, f64 accumulator), which runs in a subprocess with
    SYNK_SPLITK_CLUSTER=0, and meet the unsplit accuracy bar."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    a, b, bias, got = _split_case(M, N, K, epi)
    want = a.astype(np.float64) @ b.astype(np.float64).T + (bias if epi == "bias" else 0)
    assert rel_err(got, want) <= 1e-6 + 5e-8 * K
    out = tmp_path / "planes.npy"
    code = ("import sys, numpy as np; sys.path.insert(0, 'tests'); from test_gpu_gemm import _split_case; "
            f"np.save({str(out)!r}, _split_case({M}, {N}, {K}, {epi!r})[3])")
    env = dict(os.environ, SYNK_SPLITK_CLUSTER="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert np.load(out).tobytes() == got.tobytes()


@pytest.mark.parametrize("rows,cols", [(64, 64), (1000, 100), (37, 5), (130, 2048), (16, 256), (4099, 512), (8192, 2048)])
def test_prep2_bf16_cast_and_transpose(rows, cols):
    rng = np.random.default_rng(rows * cols)
    x = rng.uniform(-3, 3, (rows, cols)).astype(np.float32)
    ld, ldt = pad(cols, 8), pad(rows, 8)
    want = bf16_round(x).view(np.uint32) >> 16
    with Ranks(1) as R:
        dx = R.upload(x)
        o, ot = R.alloc(rows * ld * 2), R.alloc(cols * ldt * 2)
        check(lib().synk_gemm_prep2_bf16(R[0], _vp(dx), _u64(rows), _u64(cols), _u64(cols), _vp(o), _u64(ld), _vp(ot),
                                         _u64(ldt)), "prep2")
        check(R.sync(), "sync")
        got = R.download(o, (rows, ld), np.uint16)[:, :cols]
        got_t = R.download(ot, (cols, ldt), np.uint16)[:, :rows]
    np.testing.assert_array_equal(got, want.astype(np.uint16))
    np.testing.assert_array_equal(got_t, want.T.astype(np.uint16))


def gemm_layout(R, a, b, layout, epi="store", bias=None, act=None, out_bf16=False, want_t=None):
    """bf16 C = epi(a @ b.T) with A stored MN-major (as a.T, K x M) when
    layout & 1 and B stored MN-major (as b.T, K x N) when layout & 2.
    want_t (not None): return (C, C^T or None), C^T requested when true."""
    M, K = a.shape
    N = b.shape[0]
    ahi, _, lda = prep(R, a.T if layout & 1 else a, False, 1)
    bhi, _, ldb = prep(R, b.T if layout & 2 else b, False, 1)
    es = 2 if out_bf16 else 4
    c = R.alloc(M * N * es)
    dbias = R.upload(bias.astype(np.float32)) if bias is not None else 0
    dact = 0
    if act is not None:
        dact = R.alloc(M * N * 2)
        da = R.upload(act.astype(np.float32))
        check(lib().synk_gemm_prep(R[0], F32, _vp(da), _u64(M), _u64(N), _u64(N), 0, 1, _vp(dact), None, _u64(M),
                                   _u64(N), _u64(N)), "prep act")
    ct = R.alloc(M * N * es) if want_t else 0
    check(lib().synk_gemm_tc2(R[0], 0, _u64(M), _u64(N), _u64(K), _vp(ahi), None, _u64(lda), _vp(bhi), None, _u64(ldb),
                              layout, EPI[epi], BF16 if out_bf16 else F32, _vp(c), _u64(N), _vp(ct or None), _u64(M),
                              _vp(dbias or None), _vp(dact or None), _u64(N)), "gemm_tc2")
    check(R.sync(), "sync")

    def fetch(ptr, shape):
        if out_bf16:
            raw = R.download(ptr, shape, np.uint16).astype(np.uint32) << 16
            return raw.view(np.float32)
        return R.download(ptr, shape, np.float32)

    out = fetch(c, (M, N))
    if want_t is None:
        return out
    return out, (fetch(ct, (N, M)) if want_t else None)


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (300, 200, 100), (129, 520, 72), (4096, 2048, 512),
                                   (4097, 100, 8192), (8192, 100, 4096), (1000, 4000, 600)])
@pytest.mark.parametrize("layout", [1, 2, 3])
def test_bf16_mn_major_operands(M, N, K, layout):
    """MN-major A and/or B (UMMA major bits, 64x64 TMA boxes): bitwise equal
    to the K-major product of the same bf16 operands, on the persistent
    128x256 path, the 128x128 path and the split-K path; and within the
    fp32-accumulation bound of the fp64 product."""
    rng = np.random.default_rng(M * 3 + N + K + layout)
    a = bf16_round(rng.uniform(-1, 1, (M, K)))
    b = bf16_round(rng.uniform(-1, 1, (N, K)))
    want = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        ref = gemm_layout(R, a, b, 0)
        got = gemm_layout(R, a, b, layout)
    assert rel_err(got, want) <= 1e-6 + 5e-8 * K
    np.testing.assert_array_equal(got, ref)


def test_bf16_mn_major_fused_epilogues():
    """The MLP's forward (B = W MN-major, bias + tanh, bf16 out) and weight-
    gradient (A = activations, B = delta, both MN-major) products."""
    rng = np.random.default_rng(9)
    M, N, K = 512, 384, 256
    a = bf16_round(rng.uniform(-1, 1, (M, K)))
    b = bf16_round(rng.uniform(-1, 1, (N, K)) * 0.1)
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    z = a.astype(np.float64) @ b.astype(np.float64).T
    with Ranks(1) as R:
        for layout in (0, 2, 3):
            got = gemm_layout(R, a, b, layout, "bias_tanh", bias=bias, out_bf16=True)
            assert rel_err(got, np.tanh(z + bias)) <= 2.0 ** -7
            act = bf16_round(np.tanh(rng.uniform(-1, 1, (M, N))))
            got = gemm_layout(R, a, b, layout, "tanh_grad", act=act, out_bf16=True)
            assert rel_err(got, z * (1 - act.astype(np.float64) ** 2)) <= 2.0 ** -7 * 4


@pytest.mark.parametrize("M,N,K,with_t", [(8192, 4096, 100, False), (1000, 600, 100, True), (300, 260, 8, False),
                                            (513, 4100, 128, True)])
def test_bf16_short_k_tanh_grad_staged_activations(M, N, K, with_t):
    """Short-K tanh-derivative products (C5's dX with K = 100): the CTA-pair
    kernel TMA-stages each tile's activation block into shared memory while
    the previous tile drains. Ragged M / N edges, K below one block, an
    optional transposed output; checked against fp64 on bf16-exact inputs at
    bf16 output resolution, and C^T bitwise equal to C."""
    rng = np.random.default_rng(M + N + K)
    a = bf16_round(rng.uniform(-1, 1, (M, K)))
    b = bf16_round(rng.uniform(-1, 1, (N, K)) * 0.1)
    act = bf16_round(np.tanh(rng.uniform(-1, 1, (M, N))))
    want = (a.astype(np.float64) @ b.astype(np.float64).T) * (1 - act.astype(np.float64) ** 2)
    with Ranks(1) as R:
        got, got_t = gemm_layout(R, a, b, 0, "tanh_grad", act=act, out_bf16=True, want_t=with_t)
    assert rel_err(got, want) <= 2.0 ** -7 * 4
    if with_t:
        np.testing.assert_array_equal(got_t, got.T)


def test_c5_full_size_bf16_gradient_vs_fp64(sk, oracle):
    """C5 at BASELINE size: MLP 2048-4096-4096-100 (25,583,716 params), batch
    8192, every product on tcgen05 in bf16. Reference: the same loss/gradient
    math (mlp.cpp:134-218) in fp64 with torch on the GPU (a floating-point
    cross-check of a floating-point kernel). Bars as the small-config test:
    relative Frobenius error of the gradient <= 2e-2, loss <= 1e-2; then one
    SGD step through the Trainer is bit-for-bit the reference's update rule
    (sgd.cpp:46-52 restated in the oracle) applied to the gradient block."""
    import torch

    dims = [2048, 4096, 4096, 100]
    cfg = sk.MlpConfig(in_dim=dims[0], width=dims[1], out_dim=dims[3], layers=3, seed=1)
    x, y = sk.mlp_make_dataset(8192, cfg, seed=2, dtype="f32")
    params = sk.mlp_init_params(cfg, "f32")
    dev = torch.device("cuda:0")
    P = [torch.from_numpy(p.astype(np.float64)).to(dev) for p in params]
    a = [torch.from_numpy(x.astype(np.float64)).to(dev)]
    for l in range(3):
        z = a[-1] @ P[2 * l] + P[2 * l + 1]
        a.append(torch.tanh(z) if l < 2 else z)
    yt = torch.from_numpy(y.astype(np.float64)).to(dev)
    n = x.shape[0]
    ref_loss = float(0.5 / n * ((a[3] - yt) ** 2).sum())
    delta = (a[3] - yt) / n
    grads = [None] * 6
    for l in (2, 1, 0):
        grads[2 * l] = a[l].T @ delta
        grads[2 * l + 1] = delta.sum(0)
        if l > 0:
            delta = (delta @ P[2 * l].T) * (1 - a[l] ** 2)
    ref_grad = torch.cat([g.reshape(-1) for g in grads]).cpu().numpy()
    with sk.Pool(workers=1) as pool:
        block = sk.ParamBlock.create(pool, params)
        f = sk.mlp_grad_function(pool, block, compute="bf16")
        sk.distribute(pool)
        (loss,) = f.call([x, y])
        g = block.grads.get(0).astype(np.float64)
        assert abs(loss - ref_loss) / ref_loss <= 1e-2
        assert np.linalg.norm(g - ref_grad) / np.linalg.norm(ref_grad) <= 2e-2
        p0 = block.params.get(0)
        trainer = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
        trainer.train_step(f, [x, y])
        assert block.params.get(0).tobytes() == oracle.sgd(p0, block.grads.get(0), 0.01).tobytes()


@pytest.mark.parametrize("world,rule", [(1, "sgd"), (2, "adam"), (3, "momentum"), (8, "rmsprop")])
def test_overlapped_segment_updates_bitwise(sk, world, rule):
    """bf16 MLP through the Trainer: each layer's gradient segment is
    all-reduced + applied on the rank's second stream as soon as every rank
    finished it (overlapping the rest of the backward pass). Same arithmetic
    per element as the non-overlapped step (check_finite=True keeps the
    reference's two-phase sequence): parameters and optimizer state must
    match bit for bit after several steps, replicas coherent."""
    cfg = sk.MlpConfig(in_dim=256, width=384, out_dim=100, layers=3, seed=3)
    x, y = sk.mlp_make_dataset(512 * world, cfg, seed=4, dtype="f32")
    rules = {"sgd": sk.SgdRule, "adam": sk.AdamRule, "momentum": sk.MomentumRule, "rmsprop": sk.RmsPropRule}
    params = {}
    for check_finite in (False, True):
        with sk.Pool(workers=world) as pool:
            block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
            f = sk.mlp_grad_function(pool, block, compute="bf16")
            sk.distribute(pool)
            tr = sk.Trainer(pool, block, rules[rule](), lr=1e-2, check_finite=check_finite, verify_coherence=True)
            rng = np.random.default_rng(7)
            for _ in range(4):
                tr.train_step(f, [x, y], indexes=rng.integers(0, x.shape[0], 256 * world))
            assert block.params.coherent
            params[check_finite] = block.params.get(world - 1)
    assert params[False].tobytes() == params[True].tobytes()


@pytest.mark.parametrize("world,rows,slices", [(3, 700, 1), (2, 512, 2)])
def test_fused_step_fallbacks_bitwise(sk, world, rows, slices):
    """Paths where the trainer cannot overlap the segment updates: unequal
    shards (the rows_r*W/total pre-scale must precede the all-reduce) and
    num_slices > 1 (per-slice invocations: no final segments, eager report
    timing). Bitwise equal to the two-phase step; reports populated."""
    cfg = sk.MlpConfig(in_dim=128, width=256, out_dim=100, layers=3, seed=5)
    x, y = sk.mlp_make_dataset(rows, cfg, seed=6, dtype="f32")
    params = {}
    for check_finite in (False, True):
        with sk.Pool(workers=world) as pool:
            block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
            f = sk.mlp_grad_function(pool, block, compute="bf16")
            sk.distribute(pool)
            tr = sk.Trainer(pool, block, sk.AdamRule(), lr=1e-2, check_finite=check_finite)
            for _ in range(3):
                tr.train_step(f, [x, y], num_slices=slices)
            rep = tr.last_report
            assert rep["grad_call"]["rank_rows"] == [len(p) for p in np.array_split(np.arange(rows), world)]
            assert max(rep["grad_call"]["rank_compute_s"]) > 0 and rep["allreduce_s"] > 0
            assert block.params.coherent
            params[check_finite] = block.params.get(0)
    assert params[False].tobytes() == params[True].tobytes()


@pytest.mark.parametrize("world", [1, 2])
def test_bf16_multi_step_trajectory_vs_oracle(sk, oracle, world):
    """C5's path over several sync-SGD steps (bf16 tcgen05 products, fused and
    bucketed all-reduce + update, index-fused batches, bf16 weight shadows
    written by the update) against the oracle replaying the same steps in the
    reference's f32 algebra (mlp.cpp:134-218 + sgd.cpp:259-332: shard-mean
    gradients, mean all-reduce, SGD). Stated bf16 bar, per step: loss within
    2e-2 relative; after 6 steps the parameter CHANGE within 5e-2 relative
    Frobenius (the update itself is exact given the gradient; the gradient
    carries bf16 operand rounding)."""
    dims = [256, 512, 512, 100]
    cfg = sk.MlpConfig(in_dim=dims[0], width=dims[1], out_dim=dims[-1], layers=3, seed=9)
    x, y = sk.mlp_make_dataset(4096, cfg, seed=10, dtype="f32")
    params = sk.mlp_init_params(cfg, "f32")
    p_ref = np.concatenate([p.ravel() for p in params])
    p0 = p_ref.copy()
    rng = np.random.default_rng(11)
    lr, steps, batch = 0.05, 6, 512
    with sk.Pool(workers=world) as pool:
        sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
        sx.mirror(pool)
        sy.mirror(pool)
        block = sk.ParamBlock.create(pool, params)
        f = sk.mlp_grad_function(pool, block, compute="bf16")
        sk.distribute(pool)
        tr = sk.Trainer(pool, block, sk.SgdRule(), lr=lr)
        for s in range(steps):
            idx = rng.integers(0, 4096, batch)
            loss = tr.train_step(f, [sx, sy], indexes=idx)
            # reference step: each rank's shard-mean gradient, mean over ranks
            shards = [idx[a:b] for a, b in oracle.partition_rows(batch, world)]
            grads, losses = [], []
            for sh in shards:
                l_r, g_r = oracle.mlp_loss_grad(p_ref, dims, x[sh], y[sh])
                grads.append(g_r.astype(np.float64))
                losses.append(l_r * len(sh))
            ref_loss = sum(losses) / batch
            assert abs(loss - ref_loss) / ref_loss <= 2e-2, (s, loss, ref_loss)
            p_ref = (p_ref - lr * np.mean(grads, axis=0)).astype(np.float32)
        got = block.params.get(0)
        assert block.params.coherent
    d_got, d_ref = got.astype(np.float64) - p0, p_ref.astype(np.float64) - p0
    assert np.linalg.norm(d_got - d_ref) / np.linalg.norm(d_ref) <= 5e-2
