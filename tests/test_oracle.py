"""Pin the CPU restatement (oracle/synk_oracle.c) before trusting it.

(1) Known answers of the reference's own unit tests, restated.
(2) Golden vectors produced by the unmodified reference (tests/golden/).
(3) When the reference module is built here, direct randomized comparison.
All CPU-only.
"""

import numpy as np
import pytest

from conftest import golden

# ---- (1) known answers restated from the reference unit tests ----------------------


def test_partition_known_answers(oracle):
    # test_tensor.cpp:191-229
    assert oracle.partition_rows(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert oracle.partition_rows(3, 8)[:4] == [(0, 1), (1, 2), (2, 3), (3, 3)]
    assert oracle.partition_rows(0, 4) == [(0, 0)] * 4


def test_gather_known_answers(oracle):
    # test_tensor.cpp:119-130: iota 4x2, idx {3,0,3} -> rows (6,7),(0,1),(6,7)
    src = np.arange(8, dtype=np.float64).reshape(4, 2)
    np.testing.assert_array_equal(oracle.gather_rows(src, [3, 0, 3]), [[6, 7], [0, 1], [6, 7]])
    with pytest.raises(IndexError):
        oracle.gather_rows(src, [4])


def test_combine_known_answers(oracle):
    # test_tensor.cpp:132-160
    a = np.array([1.0, -2.0])
    b = np.array([4.0, -5.0])
    np.testing.assert_array_equal(oracle.combine(a, b, "sum"), [5, -7])
    np.testing.assert_array_equal(oracle.combine(a, b, "max"), [4, -2])
    np.testing.assert_array_equal(oracle.combine(np.array([-5.0, 0.5]), np.array([3.0, 1.0]), "min"), [-5, 0.5])
    np.testing.assert_array_equal(oracle.combine(np.array([2.0, 1.5]), np.array([2.0, 1.0]), "prod"), [4, 1.5])
    with pytest.raises(ValueError):
        oracle.combine(a, b, "mean")
    # accumulator wins NaN and signed-zero ties (b > a ? b : a)
    assert np.isnan(oracle.combine(np.array([np.nan]), np.array([1.0]), "max")[0])
    assert oracle.combine(np.array([1.0]), np.array([np.nan]), "max")[0] == 1.0
    assert np.signbit(oracle.combine(np.array([-0.0]), np.array([0.0]), "max")[0])


def test_weighted_mean_known_answer(oracle):
    # test_tensor.cpp:162-175: (2*1 + 5*2) / 3 = 4
    assert oracle.weighted_mean(np.array([2.0]), 1, np.array([5.0]), 2)[0] == 4.0


def test_tree_fold_known_answers(oracle):
    # test_replicated.cpp:52-111: replicas {1,2,3,4}
    parts = [np.array([float(v)]) for v in (1, 2, 3, 4)]
    assert oracle.tree_fold(parts, "sum")[0] == 10
    assert oracle.tree_fold(parts, "mean")[0] == 2.5
    assert oracle.tree_fold(parts, "max")[0] == 4
    assert oracle.tree_fold(parts, "min")[0] == 1
    assert oracle.tree_fold(parts, "prod")[0] == 24


def test_function_mean_weighting(oracle):
    # test_function.cpp:81-92: shard means 2.0 (3 rows), 4.5 (2 rows) -> exactly 3.0
    out = oracle.left_fold([np.array([2.0]), np.array([4.5])], "mean", [3, 2])
    assert out[0] == 3.0


def test_optimizer_known_answers(oracle):
    # test_sgd.cpp:56-112
    p = oracle.sgd(np.array([1.0, 0.5]), np.array([0.5, 4.0]), 0.1)
    assert p[0] == 0.95 and p[1] == 0.09999999999999998
    p, v = oracle.momentum(np.array([0.0]), np.array([0.0]), np.array([1.0]), 0.9, 0.1)
    assert v[0] == -0.1 and p[0] == -0.19
    p, v = oracle.momentum(p, v, np.array([1.0]), 0.9, 0.1)
    assert v[0] == -0.19 and p[0] == -0.46099999999999997
    p, a = oracle.rmsprop(np.array([0.0]), np.array([0.0]), np.array([1.0]), 0.9, 1e-6, 0.1)
    assert a[0] == 0.09999999999999998
    assert abs(p[0] - -0.31622618488986637) <= 1e-15
    p, m, v = oracle.adam(np.array([0.0]), np.array([0.0]), np.array([0.0]), np.array([1.0]), 0.9, 0.999, 1e-8, 0.1, 1)
    assert abs(p[0] - -0.09999999900000002) <= 1e-15
    p, m, v = oracle.adam(p, m, v, np.array([1.0]), 0.9, 0.999, 1e-8, 0.1, 2)
    assert abs(p[0] - -0.19999999799999935) <= 1e-14


def test_mlp_finite_difference(oracle):
    # test_mlp.cpp:68-93: gradient matches central differences to 1e-6
    rng = np.random.default_rng(3)
    dims = [3, 5, 2]
    n_params = 3 * 5 + 5 + 5 * 2 + 2
    theta = rng.normal(0, 0.5, n_params)
    x = rng.normal(size=(7, 3))
    y = rng.normal(size=(7, 2))
    _, g = oracle.mlp_loss_grad(theta, dims, x, y)
    h = 1e-6
    for i in range(0, n_params, 3):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        fd = (oracle.mlp_loss_grad(tp, dims, x, y)[0] - oracle.mlp_loss_grad(tm, dims, x, y)[0]) / (2 * h)
        assert abs(fd - g[i]) <= 1e-6


# ---- (2) golden vectors from the unmodified reference ----------------------------


def test_gather_golden(oracle):
    g = golden("gather.npz")
    for tag in ("f32", "f64"):
        src, idx = g[tag + "_src"], g[tag + "_idx"]
        mine = oracle.gather_rows(src, idx)
        for world in (1, 3, 4):
            ref = g["%s_w%d_list" % (tag, world)]
            assert ref.dtype == mine.dtype
            assert mine.tobytes() == ref.tobytes()  # bit-exact
            np.testing.assert_array_equal(g["%s_w%d_range" % (tag, world)], src[11:290])


def test_collectives_golden(oracle):
    g = golden("collectives.npz")
    for world in (2, 3, 4, 8):
        for tag in ("f32", "f64"):
            vals = list(g["in_%s_w%d" % (tag, world)])
            for op in ("sum", "mean", "max", "min", "prod"):
                mine = oracle.tree_fold(vals, op)
                ref = g["allreduce_%s_%s_w%d" % (op, tag, world)]
                assert mine.tobytes() == ref.tobytes(), (op, tag, world)  # bitwise, incl. sum/mean
            assert oracle.tree_fold(vals, "sum").tobytes() == g["reduce_sum_%s_w%d" % (tag, world)].tobytes()


def test_mlp_golden(oracle):
    g = golden("mlp.npz")
    loss, grad = oracle.mlp_loss_grad(g["params"], [784, 512, 10], g["x"], g["y"])
    assert loss == float(g["loss"])  # same f64 loops, same order
    assert grad.tobytes() == g["grad"].tobytes()
    loss, grad = oracle.mlp_loss_grad(g["params64"], [8, 16, 16, 16, 4], g["x64"], g["y64"])
    assert loss == float(g["loss64"])
    assert grad.tobytes() == g["grad64"].tobytes()


# ---- (3) direct comparison with the reference build, when present -----------------


def test_oracle_matches_reference_module(oracle):
    ref = oracle.reference_module()
    if ref is None:
        pytest.skip("reference module not built in this environment (oracle/_ref)")
    rng = np.random.default_rng(123)
    for world in (1, 2, 5):
        vals = [rng.uniform(-1, 1, 64) for _ in range(world)]
        with ref.Pool(workers=world) as pool:
            v = ref.replicate(pool, np.zeros(64))
            for r in range(world):
                v.set(r, vals[r])
            v.all_reduce("mean")
            assert v.get(0).tobytes() == oracle.tree_fold(vals, "mean").tobytes()
