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
