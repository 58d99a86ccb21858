"""Diagnostic (not collected): C1 sync-SGD steps (784-512-10 f32, batch 256,
W=1 and W=2 on GPU 0) with the f32 products on the tensor cores (3xTF32,
default) vs FFMA (SYNK_MLP_F32=ffma), wall ms/step over 300 steps, plus the
loss difference between the two paths."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

cfg = sk.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
x, y = sk.mlp_make_dataset(65536, cfg, seed=2, dtype="f32")


def run(mode, world, steps=300):
    os.environ["SYNK_MLP_F32"] = mode
    rng = np.random.default_rng(0)
    with sk.Pool(workers=world, devices=[0] * world) as pool:
        sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
        sx.mirror(pool)
        sy.mirror(pool)
        block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
        g = sk.mlp_grad_function(pool, block)
        sk.distribute(pool)
        tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
        idx = [rng.integers(0, 65536, 256 * world) for _ in range(steps + 20)]
        losses = [tr.train_step(g, [sx, sy], indexes=idx[s]) for s in range(20)]
        t0 = time.perf_counter()
        for s in range(steps):
            losses.append(tr.train_step(g, [sx, sy], indexes=idx[20 + s]))
        dt = (time.perf_counter() - t0) / steps
        return dt * 1e3, np.array(losses), block.params.get(0)


for world in (1, 2):
    res = {m: run(m, world) for m in ("tc", "ffma", "tc")}
    tc_ms, tc_l, tc_p = run("tc", world)
    ff_ms, ff_l, ff_p = run("ffma", world)
    rel = np.max(np.abs(tc_l - ff_l) / np.abs(ff_l))
    prel = np.max(np.abs(tc_p - ff_p)) / np.max(np.abs(ff_p))
    print("W=%d  tc %.4f ms/step  ffma %.4f ms/step  | 320-step loss rel diff %.2e, param max diff/scale %.2e"
          % (world, tc_ms, ff_ms, rel, prel))
