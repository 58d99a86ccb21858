"""API-level parity of the drop-in (paper_1710_04162_b200 == synkpar surface)
on the GPU: the reference's own Python smoke tests (python/tests/test_smoke.py),
the function-semantics known answers of test_function.cpp / test_replicated.cpp,
and trajectories against golden vectors produced by the unmodified reference.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


# ---- the reference's python/tests/test_smoke.py, unchanged in intent ----------------

def test_pool_lifecycle(sk):
    with sk.Pool(workers=2) as pool:
        assert pool.world_size == 2
        assert pool.alive
    assert not pool.alive


def test_scatter_gather_round_trip(sk):
    data = np.arange(30, dtype=np.float64).reshape(10, 3)
    with sk.Pool(workers=4) as pool:
        var = sk.replicate(pool, np.zeros((1, 3)))
        var.scatter(data)
        assert [var.get(r).shape[0] for r in range(4)] == [3, 3, 2, 2]
        np.testing.assert_array_equal(var.gather(), data)


def test_all_reduce_matches_numpy(sk):
    rng = np.random.default_rng(7)
    values = [rng.standard_normal(16) for _ in range(4)]
    with sk.Pool(workers=4) as pool:
        var = sk.replicate(pool, np.zeros(16))
        for r, v in enumerate(values):
            var.set(r, v)
        var.all_reduce("mean")
        assert var.coherent
        np.testing.assert_allclose(var.get(0), np.mean(values, axis=0), rtol=0, atol=1e-12)


def test_python_kernel_column_sum(sk):
    data = np.arange(24, dtype=np.float64).reshape(8, 3)
    with sk.Pool(workers=3) as pool:
        f = sk.make_py_function(pool, "column_sum", lambda inputs, ctx: [inputs[0].sum(axis=0)], ["scatter"], ["sum"])
        sk.distribute(pool)
        (out,) = f.call([data])
        np.testing.assert_allclose(out, data.sum(axis=0), rtol=0, atol=1e-12)
        (sliced,) = f.call([data], num_slices=3)
        np.testing.assert_allclose(sliced, out, rtol=0, atol=1e-12)
        (serial,) = f.call_serial([data])
        np.testing.assert_allclose(out, serial, rtol=0, atol=1e-12)


def test_python_kernel_update_delta(sk):
    data = np.array([[1.0], [2.0], [3.0], [4.0]])

    def shard_total(inputs, ctx):
        return [np.float64(inputs[0].sum()).reshape(()), inputs[0].sum(axis=0)]

    with sk.Pool(workers=2) as pool:
        acc = sk.replicate(pool, np.zeros(1))
        f = sk.make_py_function(pool, "shard_total", shard_total, ["scatter"], ["sum"], updates=[(acc, "add")])
        sk.distribute(pool)
        (total,) = f.call([data])
        assert total == pytest.approx(10.0)
        assert acc.get(0)[0] == pytest.approx(3.0)
        assert acc.get(1)[0] == pytest.approx(7.0)


def test_shared_input_and_indexes(sk):
    with sk.Pool(workers=2) as pool:
        arr = sk.SharedInput.from_array(np.arange(12, dtype=np.float64).reshape(6, 2))
        f = sk.make_py_function(pool, "first_col", lambda i, c: [i[0][:, :1].sum(axis=0)], ["scatter"], ["sum"])
        sk.distribute(pool)
        (full,) = f.call([arr])
        assert full[0] == pytest.approx(np.arange(0, 12, 2).sum())
        (ranged,) = f.call([arr], indexes=(0, 3))
        assert ranged[0] == pytest.approx(0.0 + 2.0 + 4.0)
        (picked,) = f.call([arr], indexes=[5, 0])
        assert picked[0] == pytest.approx(10.0 + 0.0)


def test_errors_map_to_python(sk):
    with sk.Pool(workers=2) as pool:
        var = sk.replicate(pool, np.zeros(2))
        with pytest.raises(sk.ArgumentError):
            var.get(9)
        with pytest.raises(sk.Error):
            var.all_reduce("gather")
    with pytest.raises(sk.LifecycleError):
        var.all_reduce("sum")


def test_trainer_loss_decreases(sk):
    cfg = sk.MlpConfig(in_dim=4, width=8, out_dim=2, layers=2, seed=1)
    x, y = sk.mlp_make_dataset(64, cfg, seed=9)
    with sk.Pool(workers=2) as pool:
        block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg))
        f = sk.mlp_grad_function(pool, block)
        sk.distribute(pool)
        trainer = sk.Trainer(pool, block, sk.AdamRule(), lr=1e-2, verify_coherence=True)
        losses = [trainer.train_step(f, [x, y]) for _ in range(30)]
        assert losses[-1] < 0.5 * losses[0]
        assert block.params.coherent
        assert trainer.step_count == 30


# ---- device built-in kernels: gather / slicing / aggregation -------------------------

@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_indexed_gather_bit_exact(sk, oracle, world):
    rng = np.random.default_rng(world)
    src = rng.uniform(-1, 1, (5000, 256)).astype(np.float32)
    idx = rng.integers(0, 5000, 4096 * world)
    with sk.Pool(workers=world) as pool:
        arr = sk.SharedInput.from_array(src)
        f = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
        sk.distribute(pool)
        (got,) = f.call([arr], indexes=idx)                  # pinned host source, gathered on GPU
        assert got.tobytes() == oracle.gather_rows(src, idx.astype(np.uint64)).tobytes()
        arr.mirror(pool)                                      # HBM mirror source
        (got2,) = f.call([arr], indexes=idx, num_slices=3)
        assert got2.tobytes() == got.tobytes()
        (serial,) = f.call_serial([arr], indexes=idx.tolist())
        assert serial.tobytes() == got.tobytes()


def test_borrowed_and_pinned_index_arrays(sk, oracle):
    """int64/uint64 ndarrays are read in place (no IndexList copy); pinned arrays
    are DMA'd; results identical to list indexes; validation unchanged."""
    rng = np.random.default_rng(21)
    src = rng.uniform(-1, 1, (3000, 64)).astype(np.float32)
    idx = rng.integers(0, 3000, 5000)
    pinned = sk.pinned_array(idx.size, "int64")
    pinned[:] = idx
    with sk.Pool(workers=3) as pool:
        arr = sk.SharedInput.from_array(src)
        f = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
        sk.distribute(pool)
        want = oracle.gather_rows(src, idx.astype(np.uint64)).tobytes()
        for sel in (idx, idx.astype(np.uint64), pinned, idx.tolist()):
            (got,) = f.call([arr], indexes=sel, num_slices=2)
            assert got.tobytes() == want
        bad = idx.copy()
        bad[17] = 3000
        with pytest.raises(sk.BoundsError):
            f.call([arr], indexes=bad)
        bad[17] = -1
        with pytest.raises(sk.BoundsError):
            f.call([arr], indexes=bad)
        assert pool.alive


@pytest.mark.parametrize("world", [1, 2])
def test_device_checked_indexes_raise_bounds_error(sk, world):
    """Device kernels without updates skip the host scan of the index list: the
    gather kernel checks every index and call() raises the same BoundsError
    (same message, pool alive) after the phase. Error order is the reference's:
    a bad index wins over errors validated after it (function.cpp:266)."""
    rng = np.random.default_rng(5)
    src = rng.uniform(-1, 1, (1000, 32)).astype(np.float32)
    with sk.Pool(workers=world) as pool:
        arr = sk.SharedInput.from_array(src)
        arr.mirror(pool)
        f = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
        cnt = sk.make_function(pool, sk.row_count_kernel(), ["scatter"], ["sum"])
        sk.distribute(pool)
        pinned = sk.pinned_array(900, "int64")
        pinned[:] = rng.integers(0, 1000, 900)
        pinned[850] = 1000  # only the last rank's share holds the bad index
        for sel in (pinned, np.asarray(pinned).copy(), np.asarray(pinned).astype(np.uint64)):
            for fn in (f, cnt):
                with pytest.raises(sk.BoundsError, match="1000 not within 1000 rows"):
                    fn.call([arr], indexes=sel)
                assert pool.alive
        pinned[850] = 999
        (got,) = f.call([arr], indexes=pinned)
        assert got.tobytes() == src[np.asarray(pinned)].tobytes()
        assert float(cnt.call([arr], indexes=pinned)[0]) == 900.0
        # error order: BoundsError before the replica_indexes ArgumentError
        pinned[3] = 5000
        with pytest.raises(sk.BoundsError):
            f.call([arr], indexes=pinned, replica_indexes=[(0, 1)])
        pinned[3] = 3
        with pytest.raises(sk.ArgumentError):
            f.call([arr], indexes=pinned, replica_indexes=[(0, 1)])


def test_bad_index_with_updates_leaves_variables_untouched(sk):
    """Kernels with updates keep the host-side check before the phase, so a
    BoundsError cannot leave a half-applied update behind."""
    data = np.arange(8.0).reshape(8, 1)

    def total(inputs, ctx):
        return [np.float64(inputs[0].sum()).reshape(()), inputs[0].sum(axis=0)]

    with sk.Pool(workers=2) as pool:
        acc = sk.replicate(pool, np.zeros(1))
        f = sk.make_py_function(pool, "total", total, ["scatter"], ["sum"], updates=[(acc, "add")])
        sk.distribute(pool)
        idx = sk.pinned_array(4, "int64")
        idx[:] = [1, 2, 3, 8]
        with pytest.raises(sk.BoundsError):
            f.call([data], indexes=idx)
        assert acc.get(0)[0] == 0.0 and acc.get(1)[0] == 0.0
        idx[3] = 7
        (t,) = f.call([data], indexes=idx)
        assert t == 13.0 and acc.get(0)[0] == 3.0 and acc.get(1)[0] == 10.0


def test_gather_golden_through_api(sk):
    g = golden("gather.npz")
    for tag in ("f32", "f64"):
        src, idx = g[tag + "_src"], g[tag + "_idx"]
        for world in (1, 3, 4):
            with sk.Pool(workers=world) as pool:
                f = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
                sk.distribute(pool)
                (got,) = f.call([src], indexes=idx, num_slices=2)
                assert got.tobytes() == g["%s_w%d_list" % (tag, world)].tobytes()
                (rng_,) = f.call([src], indexes=(11, 290))
                assert rng_.tobytes() == g["%s_w%d_range" % (tag, world)].tobytes()


@pytest.mark.parametrize("world,slices", [(1, 1), (2, 4), (3, 4), (4, 5), (8, 3)])
def test_slicing_aggregation_column_stats(sk, oracle, world, slices):
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, (4099, 1024)).astype(np.float32)
    with sk.Pool(workers=world) as pool:
        f = sk.make_function(pool, sk.column_stats_kernel(), ["scatter"], ["sum", "max", "gather"])
        sk.distribute(pool)
        s, m, g = f.call([x], num_slices=slices)
        assert g.tobytes() == x.tobytes()                                   # concat: bit-exact
        assert m.tobytes() == oracle.column_fold(x, "max").tobytes()        # max: bit-exact
        # sum: slice partials folded in T, ranks folded in rank order; vs the
        # reference's sequential T sum, elem_err <= rows*eps_f32.
        assert oracle.elem_err(s, oracle.column_fold(x, "sum")) <= x.shape[0] * 1.2e-7
        assert oracle.elem_err(s, x.astype(np.float64).sum(0)) <= 1e-5


@pytest.mark.parametrize("world,slices", [(1, 4), (2, 4), (3, 5)])
def test_hbm_resident_slicing_scatter_uniform(sk, oracle, world, slices):
    """C3 on an HBM-resident input: the dataset is generated per rank in HBM
    (scatter_uniform) and passed as an implicit scatter input (the replica);
    the same stream from the oracle checks data, Gather, Max and Sum."""
    rows, cols, seed = 3001, 256, 77
    want = oracle.fill_uniform(rows * cols, seed).reshape(rows, cols)
    with sk.Pool(workers=world) as pool:
        x = sk.replicate(pool, np.zeros(1, np.float32))
        x.scatter_uniform([rows, cols], "f32", seed)
        assert x.gather().tobytes() == want.tobytes()
        f = sk.make_function(pool, sk.column_stats_kernel(), ["scatter"], ["sum", "max", "gather"])
        sk.distribute(pool)
        s, m, g = f.call([x], num_slices=slices)
        assert g.tobytes() == want.tobytes()
        assert m.tobytes() == oracle.column_fold(want, "max").tobytes()
        assert oracle.elem_err(s, oracle.column_fold(want, "sum")) <= rows * 1.2e-7
        x64 = sk.replicate(pool, np.zeros(1))
        x64.scatter_uniform([7, 3], "f64", seed)
        assert x64.gather().tobytes() == oracle.fill_uniform(21, seed, dtype=np.float64).reshape(7, 3).tobytes()


def test_function_semantics_known_answers(sk):
    # test_function.cpp:65-96 colsum [3,3], bitwise invariant under slicing
    with sk.Pool(workers=3) as pool:
        data = np.array([[1, 0], [1, 0], [1, 0], [0, 1], [0, 1], [0, 1]], np.float64)
        f = sk.make_function(pool, sk.column_stats_kernel(), ["scatter"], ["sum", "max", "gather"])
        sk.distribute(pool)
        base = f.call([data])[0]
        np.testing.assert_array_equal(base, [3.0, 3.0])
        for s in (2, 3, 5):
            assert f.call([data], num_slices=s)[0].tobytes() == base.tobytes()
    # test_function.cpp:81-92: Mean by rows is 3.0 exactly, not 3.25
    with sk.Pool(workers=2) as pool:
        f = sk.make_py_function(pool, "mean", lambda i, c: [np.float64(i[0].mean()).reshape(())], ["scatter"], ["mean"])
        sk.distribute(pool)
        assert f.call([np.array([1.0, 2, 3, 4, 5])])[0] == 3.0
    # test_function.cpp:330-363: zero rows, rank_rows {1,0}
    with sk.Pool(workers=2) as pool:
        g = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
        s = sk.make_function(pool, sk.column_stats_kernel(), ["scatter"], ["sum", "max", "gather"])
        sk.distribute(pool)
        (e,) = g.call([np.zeros((0, 3))])
        assert e.ndim == 1 and e.size == 0
        with pytest.raises(sk.ArgumentError):
            s.call([np.zeros((0, 3))])
        assert pool.alive
        outs, rep = s.call_with_report([np.array([[5.0, 7.0, 9.0]])])
        assert outs[0][0] == 5.0 and rep["rank_rows"] == [1, 0]


def test_call_time_validation_leaves_pool_alive(sk):
    with sk.Pool(workers=2) as pool:
        data = np.arange(8.0).reshape(4, 2)
        f = sk.make_function(pool, sk.column_stats_kernel(), ["scatter"], ["sum", "max", "gather"])
        with pytest.raises(sk.LifecycleError):
            f.call([data])
        sk.distribute(pool)
        with pytest.raises(sk.ArgumentError):
            f.call([])
        with pytest.raises(sk.ArgumentError):
            f.call([data], num_slices=0)
        with pytest.raises(sk.ShapeError):
            f.call([np.float64(1.0)])
        with pytest.raises(sk.BoundsError):
            f.call([data], indexes=[4])
        with pytest.raises(sk.BoundsError):
            f.call([data], indexes=(2, 9))
        with pytest.raises(sk.ArgumentError):
            f.call([data], replica_indexes=[(0, 1)])
        assert pool.alive
        assert f.call([data])[0][0] == 0.0 + 2 + 4 + 6


def test_kernel_contract_violation_fail_stop(sk):
    with sk.Pool(workers=2) as pool:
        f = sk.make_py_function(pool, "two", lambda i, c: [np.zeros(()), np.ones(())], ["scatter"], ["sum"])
        sk.distribute(pool)
        with pytest.raises(sk.PhaseError):
            f.call([np.arange(4.0)])
        assert not pool.alive
    with sk.Pool(workers=2) as pool:  # a fresh pool can be forked after fail-stop
        assert pool.alive


@pytest.mark.parametrize("world", [2, 3])
def test_fused_step_rank_failure_fail_stop(sk, world):
    """The trainer chains the all-reduce + update into the gradient call's
    phase behind an in-phase rank rendezvous: a rank whose gradient kernel
    fails must abort it (PhaseError + fail-stop, as the reference), never
    leave its peers waiting."""
    params = np.zeros(3)

    def grad(inputs, ctx):
        if ctx.rank == world - 1:
            raise RuntimeError("injected gradient failure")
        return [np.float64(inputs[0].sum()).reshape(()), np.full(3, 1.0)]

    with sk.Pool(workers=world) as pool:
        block = sk.ParamBlock.create(pool, [params])
        f = sk.make_py_function(pool, "grad", grad, ["scatter"], ["mean"], updates=[(block.grads, "weighted_mean")])
        sk.distribute(pool)
        trainer = sk.Trainer(pool, block, sk.SgdRule(), lr=0.1)
        with pytest.raises(sk.PhaseError):
            trainer.train_step(f, [np.arange(12.0).reshape(12, 1)])
        assert not pool.alive


def test_fused_step_python_grad_kernel(sk):
    """A host (Python) gradient kernel through the fused step: mean of the
    per-rank gradients, one SGD update, replicas coherent."""
    def grad(inputs, ctx):
        return [np.float64(inputs[0].sum()).reshape(()), np.full(2, float(ctx.rank + 1))]

    with sk.Pool(workers=2) as pool:
        block = sk.ParamBlock.create(pool, [np.array([1.0, 2.0])])
        f = sk.make_py_function(pool, "grad", grad, ["scatter"], ["mean"], updates=[(block.grads, "weighted_mean")])
        sk.distribute(pool)
        trainer = sk.Trainer(pool, block, sk.SgdRule(), lr=0.1, verify_coherence=True)
        trainer.train_step(f, [np.arange(8.0).reshape(8, 1)])
        np.testing.assert_allclose(block.params.get(0), np.array([1.0, 2.0]) - 0.1 * 1.5, rtol=1e-15)
        np.testing.assert_array_equal(block.params.get(1), block.params.get(0))


def test_overwrite_and_slicing_conflict(sk):
    with sk.Pool(workers=2) as pool:
        v = sk.replicate(pool, np.zeros(1))
        f = sk.make_py_function(pool, "ow", lambda i, c: [np.zeros(()), i[0].copy()], ["scatter"], ["sum"],
                                updates=[(v, "overwrite")])
        sk.distribute(pool)
        data = np.arange(10.0).reshape(5, 2)
        f.call([data])
        assert v.get(0).shape == (3, 2) and v.get(1).shape == (2, 2)
        assert v.get(1)[0, 0] == data[3, 0]
        with pytest.raises(sk.SlicingConflictError):
            f.call([data], num_slices=2)
        assert pool.alive


def test_implicit_replica_scatter(sk):
    # test_function.cpp:246-287: 36 / 11 / 24 and the weighted mean 8
    with sk.Pool(workers=2) as pool:
        shards = sk.replicate(pool, np.zeros(1))
        shards.set(0, np.array([1.0, 2, 3]))
        shards.set(1, np.array([10.0, 20]))
        f = sk.make_py_function(pool, "sum", lambda i, c: [np.float64(i[0].sum()).reshape(())], ["scatter"], ["sum"])
        fm = sk.make_py_function(pool, "mean", lambda i, c: [np.float64(i[0].mean()).reshape(())], ["scatter"],
                                 ["mean"])
        sk.distribute(pool)
        assert f.call([shards])[0] == 36.0
        assert f.call([shards], replica_indexes=[(0, 1)])[0] == 11.0
        per_rank = [[2, 0], (1, 2)]
        assert f.call([shards], replica_indexes=per_rank)[0] == 24.0
        assert fm.call([shards], replica_indexes=per_rank)[0] == 8.0


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_collectives_bitwise_vs_reference_golden(sk, world):
    g = golden("collectives.npz")
    if world == 1:
        pytest.skip("golden set starts at W=2")
    for tag, dtype in (("f32", np.float32), ("f64", np.float64)):
        vals = g["in_%s_w%d" % (tag, world)]
        for op in ("sum", "mean", "max", "min", "prod"):
            with sk.Pool(workers=world) as pool:
                v = sk.replicate(pool, np.zeros(vals.shape[1], dtype))
                for r in range(world):
                    v.set(r, vals[r])
                v.all_reduce(op)
                assert v.coherent
                assert v.get(world - 1).tobytes() == g["allreduce_%s_%s_w%d" % (op, tag, world)].tobytes()
        with sk.Pool(workers=world) as pool:
            v = sk.replicate(pool, np.zeros(vals.shape[1], dtype))
            for r in range(world):
                v.set(r, vals[r])
            v.reduce("sum", world - 1)
            assert v.get(world - 1).tobytes() == g["reduce_sum_%s_w%d" % (tag, world)].tobytes()
            v.broadcast(world - 1)
            assert v.coherent
            once = v.get(0)
            v.broadcast(world - 1)
            assert v.get(0).tobytes() == once.tobytes()


def test_mlp_loss_grad_api_vs_golden(sk, oracle):
    g = golden("mlp.npz")
    with sk.Pool(workers=1) as pool:
        cfg = sk.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
        params = sk.mlp_init_params(cfg, "f32")
        flat = np.concatenate([p.ravel() for p in params])
        assert flat.tobytes() == g["params"].tobytes()           # identical seeded init
        x, y = sk.mlp_make_dataset(256, cfg, seed=2, dtype="f32")
        assert x.tobytes() == g["x"].tobytes() and y.tobytes() == g["y"].tobytes()
        block = sk.ParamBlock.create(pool, params)
        f = sk.mlp_grad_function(pool, block)
        sk.distribute(pool)
        (loss,) = f.call_serial([x, y])
        assert oracle.elem_err(loss, float(g["loss"])) <= 1e-5
        assert oracle.elem_err(block.grads.get(0), g["grad"]) <= 1e-5


def test_c1_sync_sgd_trajectory_vs_reference(sk, oracle):
    """Config C1 (784-512-10 f32, batch 256 indexed, grad all-reduce mean, W=2):
    params after 4 steps vs the unmodified reference, tolerance 1e-5 (fp32)."""
    g = golden("trajectories.npz")
    cfg = sk.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
    x, y = sk.mlp_make_dataset(4096, cfg, seed=2, dtype="f32")
    with sk.Pool(workers=2) as pool:
        block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
        f = sk.mlp_grad_function(pool, block)
        sk.distribute(pool)
        trainer = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01, verify_coherence=True)
        sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
        losses = [trainer.train_step(f, [sx, sy], indexes=g["c1_idx"][s]) for s in range(g["c1_idx"].shape[0])]
        assert block.params.coherent
        assert oracle.elem_err(np.array(losses), g["c1_losses"]) <= 1e-5
        assert oracle.elem_err(block.params.get(1), g["c1_params"]) <= 1e-5


@pytest.mark.parametrize("rule", ["adam", "momentum", "rmsprop", "sgd"])
def test_f64_trajectories_unequal_shards(sk, oracle, rule):
    """W=3, 47-row batches (16/16/15 unequal shards -> pre-scale path), 10 steps, f64:
    the reference's acceptance bar is 1e-10 (acceptance_main.cpp:39)."""
    g = golden("trajectories.npz")
    rules = {"adam": (sk.AdamRule(), 1e-3), "momentum": (sk.MomentumRule(), 5e-2),
             "rmsprop": (sk.RmsPropRule(), 1e-2), "sgd": (sk.SgdRule(), 5e-2)}
    r, lr = rules[rule]
    cfg = sk.MlpConfig(in_dim=8, width=16, out_dim=4, layers=4, seed=31)
    x, y = sk.mlp_make_dataset(480, cfg, seed=77, dtype="f64")
    with sk.Pool(workers=3) as pool:
        block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f64"))
        f = sk.mlp_grad_function(pool, block)
        sk.distribute(pool)
        trainer = sk.Trainer(pool, block, r, lr=lr, verify_coherence=True)
        losses = [trainer.train_step(f, [x, y], indexes=(s * 48, s * 48 + 47)) for s in range(10)]
        assert oracle.elem_err(np.array(losses), g["f64_%s_losses" % rule]) <= 1e-10
        assert oracle.elem_err(block.params.get(0), g["f64_%s_params" % rule]) <= 1e-10


def test_allreduce_ablation(sk):
    # acceptance criterion 5: without the all-reduce replicas diverge
    cfg = sk.MlpConfig(in_dim=4, width=8, out_dim=2, layers=2, seed=3)
    x, y = sk.mlp_make_dataset(32, cfg, seed=23)
    for all_reduce in (False, True):
        with sk.Pool(workers=2) as pool:
            block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg))
            f = sk.mlp_grad_function(pool, block)
            sk.distribute(pool)
            t = sk.Trainer(pool, block, sk.SgdRule(), lr=0.05, all_reduce=all_reduce)
            for _ in range(3):
                t.train_step(f, [x, y])
            assert block.params.coherent == all_reduce


def test_bench_report_shape(sk):
    # python/tests/test_smoke.py:135-143 of the reference
    report = sk.run_bench(workers=[1, 2], steps=2, batch=8, width=8, layers=2, in_dim=4, out_dim=2, seed=3)
    assert [run["workers"] for run in report["runs"]] == [1, 2]
    for run in report["runs"]:
        for key in ("total_s", "function_s", "shuffle_s", "straggler_s", "allreduce_s", "steps_per_s", "rows_per_s",
                    "speedup_vs_1", "speedup_vs_2"):
            assert key in run
    assert report["config"]["batch_mode"] == "scaled"


def test_bench_losses_match_reference(sk):
    """run_bench (src/bench.cpp:139-225): same seeds -> same batches -> the
    same f64 Adam loss at every step of every worker count as the unmodified
    reference's own run_bench (oracle/_ref/ref_driver --mode bench), within
    the trajectory bar 1e-10 (elem_err, acceptance_main.cpp:39)."""
    import json
    import os
    import subprocess

    from conftest import ROOT

    exe = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    assert os.path.exists(exe), "oracle/_ref/ref_driver not built (run __graft_entry__.build())"
    for mode in ("fixed", "scaled"):
        kw = dict(workers=[1, 2, 3], steps=5, batch=8, width=8, layers=2, in_dim=4, out_dim=2, seed=3, batch_mode=mode)
        ours = sk.run_bench_losses(**kw)
        out = subprocess.run([exe, "--mode", "bench", "--workers-list", "1,2,3", "--steps", "5", "--batch", "8",
                              "--width", "8", "--layers", "2", "--in", "4", "--out", "2", "--seed", "3",
                              "--batch-mode", mode], capture_output=True, text=True, timeout=120, check=True)
        theirs = json.loads(out.stdout.strip().splitlines()[-1])["runs"]
        assert [r["workers"] for r in ours] == [r["workers"] for r in theirs] == [1, 2, 3]
        for o, t in zip(ours, theirs):
            assert len(o["losses"]) == len(t["losses"]) == 5
            for a_, b_ in zip(o["losses"], t["losses"]):
                assert abs(a_ - b_) / max(1.0, abs(b_)) <= 1e-10, (mode, o["workers"], o["losses"], t["losses"])


@pytest.mark.parametrize("world", [1, 2])
def test_c3_full_scale_slicing_aggregation(sk, oracle, world):
    """C3 at BASELINE size: 8,388,608 x 1024 f32 (32 GiB) HBM-resident,
    num_slices=4. Size-independent checks: Gather is the generated stream
    (sampled rows vs the oracle, bit-exact), Max equals the max of the
    Gather result bit for bit, Sum within 16*eps_f32*sqrt(rows) absolute of
    the exact f64 column sums (the per-slice f32 partials, of magnitude
    ~sqrt(rows/3), are folded in f32 as the reference's combine_inplace
    does), far inside the reference's own rows*eps_f32 bar."""
    rows, cols, seed = 8_388_608, 1024, 3
    with sk.Pool(workers=world) as pool:
        x = sk.replicate(pool, np.zeros(1, np.float32))
        x.scatter_uniform([rows, cols], "f32", seed)
        f = sk.make_function(pool, sk.column_stats_kernel(), ["scatter"], ["sum", "max", "gather"])
        sk.distribute(pool)
        s, m, g = f.call([x], num_slices=4)
    assert g.shape == (rows, cols)
    rng = np.random.default_rng(5)
    for i in list(rng.integers(0, rows, 48)) + [0, rows // 2 - 1, rows // 2, rows - 1]:
        assert g[i].tobytes() == oracle.fill_uniform(cols, seed, int(i) * cols).tobytes()
    assert m.tobytes() == g.max(axis=0).tobytes()
    exact = g.sum(axis=0, dtype=np.float64)
    err = float(np.max(np.abs(s.astype(np.float64) - exact)))
    assert err <= 16 * 2.0 ** -23 * np.sqrt(rows), err
    assert oracle.elem_err(s, exact) <= rows * 2.0 ** -23


def _c2_pattern(rows, cols):
    """Exact-integer f32 rows (< 2^24): column 0 is the row index, so a gathered
    row identifies its source row; computable for any row subset."""
    r = np.asarray(rows, np.int32)[:, None]
    c = np.arange(cols, dtype=np.int32)[None, :] * np.int32(1009)
    return ((r + c) & np.int32(0xFFFFFF)).astype(np.float32)


@pytest.mark.parametrize("world", [1, 2])
def test_c2_full_scale_indexed_gather(sk, world):
    """C2 at BASELINE size: 10,000,000 x 256 f32 shared dataset (10.24 GB,
    pinned host store + HBM mirror), 64 x 4096-row shuffled batches per rank,
    index list pinned (read in place by the gather kernel): every gathered
    row bit-exact; a bad index at full size raises BoundsError, pool alive."""
    rows, cols = 10_000_000, 256
    arr = sk.SharedInput.alloc([rows, cols], "f32")
    block = 1 << 18
    for r0 in range(0, rows, block):
        r1 = min(rows, r0 + block)
        arr.write(r0, r1, _c2_pattern(np.arange(r0, r1), cols))
    rng = np.random.default_rng(11)
    n = 4096 * 64 * world
    idx = sk.pinned_array(n, "int64")
    idx[:] = rng.integers(0, rows, n)
    idx[:2] = [0, rows - 1]
    with sk.Pool(workers=world) as pool:
        arr.mirror(pool)
        f = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
        cnt = sk.make_function(pool, sk.row_count_kernel(), ["scatter"], ["sum"])
        sk.distribute(pool)
        (got,) = f.call([arr], indexes=idx)
        assert got.tobytes() == _c2_pattern(np.asarray(idx), cols).tobytes()
        assert float(cnt.call([arr], indexes=idx)[0]) == n
        idx[n // 2] = rows
        with pytest.raises(sk.BoundsError):
            cnt.call([arr], indexes=idx)
        assert pool.alive


def test_c4_full_scale_all_reduce_broadcast(sk):
    """C4 at its largest size: 1 GiB f32 replicas, W=2 (both ranks on one GPU
    here; the same peer-memory kernels cross NVLink on a multi-GPU box).
    all_reduce mean == (a + b) * 0.5 bit for bit (the reference's W=2 tree),
    max bit for bit, broadcast bit for bit, replicas coherent."""
    n = (1 << 30) // 4
    rng = np.random.default_rng(4)
    a = rng.random(n, dtype=np.float32) * 2 - 1
    b = rng.random(n, dtype=np.float32) * 2 - 1
    with sk.Pool(workers=2, devices=[0, 0]) as pool:
        var = sk.replicate(pool, np.zeros(1, np.float32))
        var.set(0, a)
        var.set(1, b)
        var.all_reduce("mean")
        assert var.coherent
        want = (a + b) * np.float32(0.5)
        assert var.get(1).tobytes() == want.tobytes()
        var.set(0, a)
        var.set(1, b)
        var.all_reduce("max")
        assert var.get(0).tobytes() == np.maximum(a, b).tobytes()
        var.set(0, b)
        var.broadcast(0)
        assert var.get(1).tobytes() == b.tobytes()
        assert var.coherent


@pytest.mark.parametrize("world", [1, 3])
def test_index_list_edge_cases(sk, world):
    """Empty index list, a list shorter than the world (ranks with no rows),
    all-duplicate indices, first/last rows, a RowRange, and 1-row / 3-byte-ish
    ragged row sizes (4-byte and 8-byte vector paths): every result equals
    numpy fancy indexing bit for bit; Sum over zero rows raises like the
    reference (function.cpp:330-363)."""
    rng = np.random.default_rng(13)
    with sk.Pool(workers=world) as pool:
        f = sk.make_function(pool, sk.identity_kernel(), ["scatter"], ["gather"])
        cnt = sk.make_function(pool, sk.row_count_kernel(), ["scatter"], ["sum"])
        sk.distribute(pool)
        for shape, dt in (((1000, 7), np.float32), ((333, 1), np.float64), ((50, 3), np.float32)):
            src = rng.uniform(-1, 1, shape).astype(dt)
            arr = sk.SharedInput.from_array(src)
            for mirror in (False, True):
                if mirror:
                    arr.mirror(pool)
                for idx in (np.zeros(0, np.int64), np.array([shape[0] - 1]), np.full(17, 5),
                            np.array([0, shape[0] - 1] * 3), rng.integers(0, shape[0], 1001)):
                    pinned = sk.pinned_array(max(idx.size, 1), "int64")[: idx.size]
                    pinned[:] = idx
                    for sel in (idx, pinned):
                        (got,) = f.call([arr], indexes=sel)
                        # no rows anywhere: concat_rows of no parts is zeros({0}) (tensor.cpp:288)
                        assert got.shape == ((idx.size,) + shape[1:] if idx.size else (0,))
                        assert got.tobytes() == src[idx].tobytes()
                    if idx.size == 0:
                        with pytest.raises(sk.ArgumentError):
                            cnt.call([arr], indexes=idx)
                    else:
                        assert float(cnt.call([arr], indexes=idx)[0]) == idx.size
                (rg,) = f.call([arr], indexes=(3, min(40, shape[0])))
                assert rg.tobytes() == src[3:min(40, shape[0])].tobytes()


def test_nccl_backend_optional(sk):
    """The optional NCCL collectives backend (library baseline): on one GPU it
    runs with one rank (identity all-reduce, the trainer's NCCL path), asks for
    distinct GPUs otherwise, and rejects unknown backends."""
    with pytest.raises(sk.ArgumentError):
        sk.Pool(workers=1, collectives="mpi")
    if not sk.nccl_available():
        pytest.skip("libnccl.so.2 not loadable here")
    if sk.device_count() < 2:
        with pytest.raises(sk.ArgumentError, match="distinct GPU"):
            sk.Pool(workers=2, devices=[0, 0], collectives="nccl")
    rng = np.random.default_rng(2)
    v = rng.standard_normal(1000)
    with sk.Pool(workers=1, collectives="nccl") as pool:
        var = sk.replicate(pool, v)
        var.all_reduce("mean")
        var.broadcast(0)
        assert var.get(0).tobytes() == v.tobytes()
        cfg = sk.MlpConfig(in_dim=16, width=32, out_dim=4, layers=2, seed=1)
        x, y = sk.mlp_make_dataset(64, cfg, seed=3)
        block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg))
        f = sk.mlp_grad_function(pool, block)
        sk.distribute(pool)
        p0 = block.params.get(0)
        sk.Trainer(pool, block, sk.SgdRule(), lr=0.1).train_step(f, [x, y])
        g = block.grads.get(0)
        np.testing.assert_allclose(block.params.get(0), p0 - 0.1 * g, rtol=0, atol=1e-15)


@pytest.mark.parametrize("world,compute,dtype", [(1, "bf16", "f32"), (2, "bf16", "f32"), (3, "bf16", "f32"),
                                                 (1, "native", "f32"), (2, "native", "f32"), (2, "native", "f64")])
def test_index_fused_mlp_inputs_bitwise(sk, world, compute, dtype):
    """Index-fused inputs: with x and y HBM-mirrored and selected by an index
    list, the MLP kernel reads the batch rows from the whole sources itself --
    the bf16 path stages x through the row list (gather + bf16 cast + transpose
    in one pass), the native path gathers x as the first node of its CUDA
    graph, and both losses read y through the list. Same arithmetic as the
    gathered path (un-mirrored inputs): parameters bit for bit after several
    trainer steps, and the same BoundsError for a bad index."""
    cfg = sk.MlpConfig(in_dim=256, width=384, out_dim=100, layers=3, seed=1)
    x, y = sk.mlp_make_dataset(4096, cfg, seed=2, dtype=dtype)
    out = {}
    for mirror in (True, False):
        rng = np.random.default_rng(5)
        with sk.Pool(workers=world) as pool:
            sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
            if mirror:
                sx.mirror(pool)
                sy.mirror(pool)
            block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, dtype))
            f = sk.mlp_grad_function(pool, block, compute=compute)
            sk.distribute(pool)
            tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.05)
            losses = [tr.train_step(f, [sx, sy], indexes=rng.integers(0, 4096, 256 * world)) for _ in range(4)]
            bad = rng.integers(0, 4096, 256 * world)
            bad[-1] = 4096
            with pytest.raises(sk.BoundsError):
                tr.train_step(f, [sx, sy], indexes=bad)
            assert pool.alive
            out[mirror] = (losses, block.params.get(world - 1))
    assert out[True][0] == out[False][0]
    assert out[True][1].tobytes() == out[False][1].tobytes()


def test_reference_acceptance_battery_on_our_executor():
    """The reference's own acceptance battery (tests/acceptance_main.cpp),
    compiled UNCHANGED against our headers and linked with our library
    (oracle/Makefile target acceptance_ours, built where the reference sources
    are): every criterion passes or is skipped (criterion 6 measures CPU
    thread scaling and skips when its W=4 ranks share one GPU)."""
    import os
    import subprocess

    from conftest import ROOT

    exe = os.path.join(ROOT, "oracle", "_ref", "acceptance_ours")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/acceptance_ours not built (needs the reference sources)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "[FAIL]" not in out.stdout, out.stdout


def test_reference_unit_tests_on_our_executor():
    """The reference's C++ unit tests (117 test cases: tensor, tensor_io,
    worker_pool, shared_input, replicated, function, sgd, mlp, bench), compiled
    UNCHANGED against our headers and library with our doctest-compatible shim
    (oracle/Makefile target unit_ours): all pass on the B200 executor."""
    import os
    import subprocess

    from conftest import ROOT

    exe = os.path.join(ROOT, "oracle", "_ref", "unit_ours")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/unit_ours not built (needs the reference sources)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "0 failed" in out.stdout


def test_reference_python_binding_on_our_executor():
    """The reference's own pybind11 module (bindings/pymodule.cpp), compiled
    unchanged against our headers and linked with our library
    (oracle/_ref/ours_binding): its Python API driven end to end on the B200
    executor (separate interpreter: two pybind11 modules binding the same C++
    types cannot share one)."""
    import glob
    import os
    import subprocess
    import sys

    from conftest import ROOT

    if not glob.glob(os.path.join(ROOT, "oracle", "_ref", "ours_binding", "_synkpar*.so")):
        pytest.skip("oracle/_ref/ours_binding not built (needs the reference sources)")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "ref_binding_checks.py")], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "ok" in out.stdout
