"""Driven by tests/test_gpu_api.py in a separate interpreter: the reference's
own Python binding (bindings/pymodule.cpp, compiled unchanged against this
repository's headers and library into oracle/_ref/ours_binding/) exercised
through its public API -- the reference's Python surface on the B200 executor.
(The reference's python/tests are re-expressed in test_gpu_api.py; this file
only drives the reference-built module.)"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "oracle", "_ref", "ours_binding"))
import _synkpar as sk  # noqa: E402

assert "ours_binding" in sk.__file__

# pool lifecycle
with sk.Pool(workers=2) as pool:
    assert pool.world_size == 2 and pool.alive
assert not pool.alive

with sk.Pool(workers=4) as pool:
    # scatter / gather round trip, partition extents
    data = np.arange(30, dtype=np.float64).reshape(10, 3)
    var = sk.replicate(pool, np.zeros((1, 3)))
    var.scatter(data)
    assert [var.get(r).shape[0] for r in range(4)] == [3, 3, 2, 2]
    np.testing.assert_array_equal(var.gather(), data)
    # all_reduce mean
    rng = np.random.default_rng(7)
    vals = [rng.standard_normal(16) for _ in range(4)]
    v = sk.replicate(pool, np.zeros(16))
    for r, x in enumerate(vals):
        v.set(r, x)
    v.all_reduce("mean")
    np.testing.assert_allclose(v.get(0), np.mean(vals, axis=0), rtol=1e-12)
    assert v.coherent
    # python kernel: column sums, with and without slicing and indexes
    k = sk.py_kernel("colsum", 1, lambda inputs, ctx: [inputs[0].sum(axis=0)])
    f = sk.make_function(pool, k, ["scatter"], ["sum"])
    sk.distribute(pool)
    x = rng.standard_normal((101, 5))
    (s1,) = f.call([x])
    (s3,) = f.call([x], num_slices=3)
    np.testing.assert_allclose(s1, x.sum(axis=0), rtol=1e-12)
    np.testing.assert_allclose(s3, s1, rtol=1e-12)
    idx = [5, 0, 3, 3, 100]
    (si,) = f.call([x], indexes=idx)
    np.testing.assert_allclose(si, x[idx].sum(axis=0), rtol=1e-12)
    try:
        f.call([x], indexes=[101])
        raise AssertionError("no BoundsError")
    except sk.BoundsError:
        pass
    assert pool.alive

# sync SGD with the reference's MLP kernel, through the reference's Trainer binding
cfg = sk.MlpConfig(in_dim=8, width=16, out_dim=4, layers=2, seed=1)
xs, ys = sk.mlp_make_dataset(128, cfg, seed=9)
with sk.Pool(workers=2) as pool:
    block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg))
    g = sk.make_function(pool, sk.mlp_grad_kernel(block), ["scatter", "scatter"], ["mean"],
                         [(block.grads, "weighted_mean")])
    sk.distribute(pool)
    tr = sk.Trainer(pool, block, sk.AdamRule(), lr=1e-2, verify_coherence=True)
    losses = [tr.train_step(g, [xs, ys]) for _ in range(30)]
    assert losses[-1] < 0.5 * losses[0], (losses[0], losses[-1])
    assert block.params.coherent and tr.step_count == 30
print("reference binding on the B200 executor: ok")
