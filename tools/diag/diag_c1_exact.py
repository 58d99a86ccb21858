"""Diagnostic (not collected): C1 exactly as configs[0] (784-512-10 f32, W=2
ranks, batch 256 global) on the GPUs given (default both ranks on GPU 0);
prints per-step host times. SYNK_DEBUG_GRAPHS=1 reports graph captures."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

devs = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 0]
cfg = sk.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
x, y = sk.mlp_make_dataset(65536, cfg, seed=2, dtype="f32")
rng = np.random.default_rng(0)
with sk.Pool(workers=len(devs), devices=devs) as pool:
    sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
    sx.mirror(pool)
    sy.mirror(pool)
    block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
    g = sk.mlp_grad_function(pool, block)
    sk.distribute(pool)
    tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
    sel = []
    for _ in range(80):
        b = sk.pinned_array(256, "int64")
        b[:] = rng.integers(0, 65536, 256)
        sel.append(b)
    ts = []
    for s in range(80):
        t = time.perf_counter()
        tr.train_step(g, [sx, sy], indexes=sel[s])
        ts.append(1e6 * (time.perf_counter() - t))
    print("per-step us:", " ".join("%.0f" % v for v in ts))
    print("median last 40: %.1f us" % np.median(ts[40:]))
