"""Coherence and lifetime cases of the executor (round-2 review findings):
writes through SharedInput.view() reach the HBM mirrors, host-kernel outputs
survive the pinned-buffer cache at W>1, and index lists over pageable
sources upload only the selected rows. Every result is checked against the
oracle or numpy, bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2])
def test_view_writes_reach_hbm_mirrors(sk, oracle, world):
    """shared_input.hpp view() aliases the store (reference
    shared_input.cpp:111-114): a write through it must be seen by the next
    call even though the call reads the HBM mirror."""
    rng = np.random.default_rng(5)
    src = rng.uniform(-1, 1, (4096, 64)).astype(np.float32)
    idx = rng.integers(0, 4096, 1024 * world)
    idx[:4] = [7, 7, 4095, 0]
    with sk.Pool(workers=world) as pool:
        arr = sk.SharedInput.from_array(src)
        arr.mirror(pool)
        f = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
        sk.distribute(pool)
        (before,) = f.call([arr], indexes=idx)
        assert before.tobytes() == oracle.gather_rows(src, idx.astype(np.uint64)).tobytes()
        v = arr.view()
        v[7] = 42.0
        v[4095, :3] = -1.5
        src[7] = 42.0
        src[4095, :3] = -1.5
        (after,) = f.call([arr], indexes=idx)           # view alive: mirrors refreshed
        assert after.tobytes() == oracle.gather_rows(src, idx.astype(np.uint64)).tobytes()
        v[0] = 3.0
        src[0] = 3.0
        del v                                           # written, then dropped before the call
        (dropped,) = f.call([arr], indexes=idx)
        assert dropped.tobytes() == oracle.gather_rows(src, idx.astype(np.uint64)).tobytes()
        arr.write(1, 2, np.full((1, 64), 9.0, np.float32))
        src[1] = 9.0
        (again,) = f.call([arr], indexes=np.arange(4, dtype=np.int64))
        assert again.tobytes() == src[:4].tobytes()


def test_host_kernel_large_outputs_many_ranks(sk):
    """A Python kernel's >= 1 MiB outputs/deltas are pinned cache blocks: the
    H2D copy must finish before the block goes back to the cache, where
    another rank takes it (function.cpp invoke, host path)."""
    n = 400_000  # 1.6 MB f32 output and update delta per rank per slice
    with sk.Pool(workers=4) as pool:
        acc = sk.replicate(pool, np.zeros(n, np.float32))

        def fn(inputs, ctx):
            x = inputs[0]
            out = np.full(n, float(x[0, 0]) + ctx.rank, np.float32)
            delta = np.full(n, float(ctx.rank + 1), np.float32)
            return [out, delta]

        f = sk.make_py_function(pool, "big", fn, ["scatter"], ["gather"], updates=[(acc, "add")])
        sk.distribute(pool)
        data = np.arange(8, dtype=np.float32).reshape(8, 1)
        for step in range(6):
            (out,) = f.call([data + step], num_slices=2)
            parts = []
            for r in range(4):
                for s in range(2):
                    first = 2 * r + s  # 2 rows per rank, 1 per slice
                    parts.append(np.full(n, float(first + step) + r, np.float32))
            assert out.tobytes() == np.concatenate(parts).tobytes(), step
        for r in range(4):
            # Add updates: 2 slices x 6 calls x (rank + 1)
            assert np.array_equal(acc.get(r), np.full(n, 12.0 * (r + 1), np.float32))


@pytest.mark.parametrize("world", [1, 3])
def test_pageable_source_index_list(sk, oracle, world):
    """A small ndarray argument stays in pageable memory: an index list over
    it gathers on the host and uploads only the selected rows."""
    rng = np.random.default_rng(17)
    src = rng.uniform(-1, 1, (300, 24)).astype(np.float64)  # 57.6 KB: below the pinned-cache threshold
    idx = rng.integers(0, 300, 257)
    with sk.Pool(workers=world) as pool:
        f = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
        sk.distribute(pool)
        (got,) = f.call([src], indexes=idx)
        assert got.tobytes() == oracle.gather_rows(src, idx.astype(np.uint64)).tobytes()
        bad = idx.copy()
        bad[100] = 300
        with pytest.raises(sk.BoundsError):
            f.call([src], indexes=bad)
        (again,) = f.call([src], indexes=idx[::-1].copy())
        assert again.tobytes() == oracle.gather_rows(src, idx[::-1].astype(np.uint64)).tobytes()


@pytest.mark.parametrize("world", [1, 2])
def test_bf16_weight_shadow_bitwise_and_invalidation(sk, world):
    """The bf16 MLP's weight shadow (bf16 operand copies written by the fused
    update, so the next step skips the weight casts) changes no bit: the
    trajectory equals the one with the casts every step (SYNK_MLP_SHADOW=0),
    also across parameter writes that must invalidate it (set_value,
    broadcast) and an unequal-shard step (pre-scale path)."""
    import os

    cfg = sk.MlpConfig(in_dim=192, width=320, out_dim=100, layers=3, seed=11)
    x, y = sk.mlp_make_dataset(1024, cfg, seed=12, dtype="f32")
    runs = {}
    for shadow in ("1", "0"):
        os.environ["SYNK_MLP_SHADOW"] = shadow
        try:
            with sk.Pool(workers=world) as pool:
                sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
                sx.mirror(pool)
                sy.mirror(pool)
                block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
                f = sk.mlp_grad_function(pool, block, compute="bf16")
                sk.distribute(pool)
                tr = sk.Trainer(pool, block, sk.MomentumRule(), lr=1e-2, verify_coherence=True)
                rng = np.random.default_rng(3)
                losses = []
                for step in range(7):
                    if step == 3:  # an outside write: every shadow must be rebuilt
                        p = block.params.get(0)
                        p[:50] += np.float32(0.25)
                        for r in range(world):
                            block.params.set(r, p)
                    if step == 5 and world > 1:
                        block.params.broadcast(world - 1)
                    n = 256 * world + (3 if step == 4 else 0)  # step 4: unequal shards
                    losses.append(tr.train_step(f, [sx, sy], indexes=rng.integers(0, 1024, n)))
                runs[shadow] = (losses, block.params.get(world - 1).tobytes(), block.grads.get(0).tobytes())
        finally:
            os.environ.pop("SYNK_MLP_SHADOW", None)
    assert runs["1"][0] == runs["0"][0]
    assert runs["1"][1] == runs["0"][1]
    assert runs["1"][2] == runs["0"][2]


@pytest.mark.parametrize("world,compute,batches", [
    (2, "native", [256, 256]),
    (3, "bf16", [768, 768]),
    (3, "bf16", [768, 2, 768, 2]),   # 2-row batches: rank 2 gets no rows (no update, pulls its chunks)
    (4, "native", [512, 3]),
])
def test_deferred_gradient_all_gather(sk, world, compute, batches):
    """The fused step leaves the reduced gradient sharded (rank r keeps chunk
    r of every segment, SYNK_STEP_GRADS_LOCAL): every reader -- get(r), a
    kernel taking the gradients as a broadcast input, all_reduce, coherent --
    and the next step's zero-row ranks must see exactly what the two-phase
    step (check_finite=True, which writes every replica) leaves, bit for bit."""
    cfg = sk.MlpConfig(in_dim=96, width=256, out_dim=100, layers=3, seed=11)
    x, y = sk.mlp_make_dataset(1024, cfg, seed=12, dtype="f32")
    seen = {}
    for two_phase in (False, True):
        with sk.Pool(workers=world) as pool:
            block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
            f = sk.mlp_grad_function(pool, block, compute=compute)
            ident = sk.make_function(pool, sk.identity_kernel(), ["broadcast"], ["gather"])
            sk.distribute(pool)
            tr = sk.Trainer(pool, block, sk.MomentumRule(), lr=1e-2, check_finite=two_phase)
            rng = np.random.default_rng(3)
            out = []
            for k, b in enumerate(batches):
                tr.train_step(f, [x, y], indexes=rng.integers(0, x.shape[0], b))
                if k == 0:  # a kernel reading the gradients right after a step
                    (cat,) = ident.call([block.grads])
                    out.append(cat)
            out += [block.grads.get(r) for r in range(world)]
            out.append(block.params.get(world - 1))
            assert block.grads.coherent and block.params.coherent
            block.grads.all_reduce("max")
            out.append(block.grads.get(0))
            seen[two_phase] = out
    for a, b in zip(seen[False], seen[True]):
        assert a.tobytes() == b.tobytes()
    cat = seen[False][0].reshape(world, -1)  # every rank's replica, as the kernel saw it
    assert all(cat[r].tobytes() == cat[0].tobytes() for r in range(world))
    assert cat.shape[1] == sum(p.size for p in sk.mlp_init_params(cfg, "f32"))
