"""Generate golden vectors from the UNMODIFIED reference (oracle/_ref/_synkpar_ref).

Run in the build container (where /root/reference exists and `make -C oracle ref`
has built the reference pybind module):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz. The GPU box never runs this; it only reads the
committed fixtures. Every array here was produced by the reference's own code
path (its C++ kernels, collectives and trainer), not by our restatement.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402

ref = oracle.reference_module()
if ref is None:
    sys.exit("reference module not built: run `make -C oracle ref` first")


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in arrays.values()), "bytes")


def identity(inputs, ctx):
    return [inputs[0]]


def gen_gather():
    rng = np.random.default_rng(7)
    out = {}
    for tag, dtype, shape in (("f32", np.float32, (513, 37)), ("f64", np.float64, (300, 8))):
        src = rng.uniform(-1, 1, shape).astype(dtype)
        idx = rng.integers(0, shape[0], size=777).astype(np.int64)  # with replacement
        for world in (1, 3, 4):
            with ref.Pool(workers=world) as pool:
                f = ref.make_function(pool, ref.py_kernel("id", 1, identity), ["scatter"], ["gather"])
                ref.distribute(pool)
                (g,) = f.call([src], indexes=[int(i) for i in idx], num_slices=2)
                (r,) = f.call([src], indexes=(11, 290))
            out["%s_w%d_list" % (tag, world)] = g
            out["%s_w%d_range" % (tag, world)] = r
        out[tag + "_src"] = src
        out[tag + "_idx"] = idx
    save("gather.npz", **out)


def gen_collectives():
    rng = np.random.default_rng(11)
    out = {}
    for world in (2, 3, 4, 8):
        for tag, dtype in (("f32", np.float32), ("f64", np.float64)):
            vals = [rng.uniform(-1, 1, 129).astype(dtype) for _ in range(world)]
            out["in_%s_w%d" % (tag, world)] = np.stack(vals)
            for op in ("sum", "mean", "max", "min", "prod"):
                with ref.Pool(workers=world) as pool:
                    v = ref.replicate(pool, np.zeros(129, dtype))
                    for r in range(world):
                        v.set(r, vals[r])
                    v.all_reduce(op)
                    out["allreduce_%s_%s_w%d" % (op, tag, world)] = v.get(world - 1)
                    assert v.coherent
            with ref.Pool(workers=world) as pool:
                v = ref.replicate(pool, np.zeros(129, dtype))
                for r in range(world):
                    v.set(r, vals[r])
                v.reduce("sum", world - 1)
                out["reduce_sum_%s_w%d" % (tag, world)] = v.get(world - 1)
    save("collectives.npz", **out)


def gen_mlp():
    cfg = ref.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
    params = ref.mlp_init_params(cfg, "f32")
    x, y = ref.mlp_make_dataset(256, cfg, seed=2, dtype="f32")
    with ref.Pool(workers=1) as pool:
        block = ref.ParamBlock.create(pool, params)
        f = ref.make_function(pool, ref.mlp_grad_kernel(block), ["scatter", "scatter"], ["mean"],
                              [(block.grads, "weighted_mean")])
        ref.distribute(pool)
        (loss,) = f.call_serial([x, y])
        grad = block.grads.get(0)
        flat = block.params.get(0)
    # small f64 model too (for the 1e-12 class of checks)
    cfg2 = ref.MlpConfig(in_dim=8, width=16, out_dim=4, layers=4, seed=31)
    p2 = ref.mlp_init_params(cfg2, "f64")
    x2, y2 = ref.mlp_make_dataset(48, cfg2, seed=77, dtype="f64")
    with ref.Pool(workers=1) as pool:
        block = ref.ParamBlock.create(pool, p2)
        f = ref.make_function(pool, ref.mlp_grad_kernel(block), ["scatter", "scatter"], ["mean"],
                              [(block.grads, "weighted_mean")])
        ref.distribute(pool)
        (loss2,) = f.call_serial([x2, y2])
        grad2 = block.grads.get(0)
        flat2 = block.params.get(0)
    save("mlp.npz", params=flat, x=x, y=y, loss=np.asarray(loss), grad=grad,
         params64=flat2, x64=x2, y64=y2, loss64=np.asarray(loss2), grad64=grad2)


def gen_trajectories():
    """Config C1 at reduced length: sync SGD of the 784-512-10 f32 MLP, batch 256,
    indexed with replacement, W=2, plus an f64 Adam run."""
    out = {}
    cfg = ref.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
    x, y = ref.mlp_make_dataset(4096, cfg, seed=2, dtype="f32")
    rng = np.random.default_rng(5)
    steps = 4
    idx = rng.integers(0, 4096, size=(steps, 256)).astype(np.int64)
    with ref.Pool(workers=2) as pool:
        block = ref.ParamBlock.create(pool, ref.mlp_init_params(cfg, "f32"))
        f = ref.make_function(pool, ref.mlp_grad_kernel(block), ["scatter", "scatter"], ["mean"],
                              [(block.grads, "weighted_mean")])
        ref.distribute(pool)
        trainer = ref.Trainer(pool, block, ref.SgdRule(), lr=0.01, verify_coherence=True)
        sx, sy = ref.SharedInput.from_array(x), ref.SharedInput.from_array(y)
        losses = [trainer.train_step(f, [sx, sy], indexes=[int(i) for i in idx[s]]) for s in range(steps)]
        out["c1_params"] = block.params.get(1)
    out["c1_losses"] = np.asarray(losses)
    out["c1_idx"] = idx

    cfg = ref.MlpConfig(in_dim=8, width=16, out_dim=4, layers=4, seed=31)
    x, y = ref.mlp_make_dataset(16 * 3 * 10, cfg, seed=77, dtype="f64")
    for rule_name, rule, lr in (("adam", ref.AdamRule(), 1e-3), ("momentum", ref.MomentumRule(), 5e-2),
                                ("rmsprop", ref.RmsPropRule(), 1e-2), ("sgd", ref.SgdRule(), 5e-2)):
        with ref.Pool(workers=3) as pool:
            block = ref.ParamBlock.create(pool, ref.mlp_init_params(cfg, "f64"))
            f = ref.make_function(pool, ref.mlp_grad_kernel(block), ["scatter", "scatter"], ["mean"],
                                  [(block.grads, "weighted_mean")])
            ref.distribute(pool)
            trainer = ref.Trainer(pool, block, rule, lr=lr, verify_coherence=True)
            losses = []
            for s in range(10):
                # 47 rows: unequal shards 16/16/15 exercise the pre-scale path
                losses.append(trainer.train_step(f, [x, y], indexes=(s * 48, s * 48 + 47)))
            out["f64_%s_params" % rule_name] = block.params.get(0)
            out["f64_%s_losses" % rule_name] = np.asarray(losses)
    save("trajectories.npz", **out)


if __name__ == "__main__":
    gen_gather()
    gen_collectives()
    gen_mlp()
    gen_trajectories()
