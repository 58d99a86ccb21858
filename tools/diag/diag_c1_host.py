"""Diagnostic (not collected): C1 W=1 step wall time (300 steps, pinned index
lists) and the host-side cost of the pieces: python loop + train_step, and a
bare loss/grad call_serial for comparison."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

cfg = sk.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
x, y = sk.mlp_make_dataset(65536, cfg, seed=2, dtype="f32")
rng = np.random.default_rng(0)
with sk.Pool(workers=1) as pool:
    sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
    sx.mirror(pool)
    sy.mirror(pool)
    block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
    g = sk.mlp_grad_function(pool, block)
    sk.distribute(pool)
    tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)

    def pinned(n):
        b = sk.pinned_array(n, "int64")
        b[:] = rng.integers(0, 65536, n)
        return b

    sel = [pinned(256) for _ in range(400)]
    for s in range(50):
        tr.train_step(g, [sx, sy], indexes=sel[s])
    for rep in range(3):
        t0 = time.perf_counter()
        for s in range(50, 350):
            tr.train_step(g, [sx, sy], indexes=sel[s])
        print("train_step: %.1f us/step" % (1e6 * (time.perf_counter() - t0) / 300))
    t0 = time.perf_counter()
    for s in range(50, 350):
        g.call([sx, sy], indexes=sel[s])
    print("grad call only: %.1f us/call" % (1e6 * (time.perf_counter() - t0) / 300))
