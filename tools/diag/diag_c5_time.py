"""Diagnostic (not collected): C5 step time (2048-4096-4096-100 bf16, 8192
rows, W=1 unless argv[1] lists devices), median over 40 timed steps after 10
warm-up steps; run under different SYNK_* knobs for A/B comparisons."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

devs = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0]
dims = [2048, 4096, 4096, 100]
cfg = sk.MlpConfig(in_dim=dims[0], width=dims[1], out_dim=dims[-1], layers=3, seed=1)
rng = np.random.default_rng(0)
x = rng.standard_normal((16384, 2048), dtype=np.float32)
y = rng.standard_normal((16384, 100), dtype=np.float32)
with sk.Pool(workers=len(devs), devices=devs) as pool:
    sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
    sx.mirror(pool)
    sy.mirror(pool)
    block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
    g = sk.mlp_grad_function(pool, block, compute="bf16")
    sk.distribute(pool)
    tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
    sel = []
    for _ in range(50):
        b = sk.pinned_array(8192 * len(devs), "int64")
        b[:] = rng.integers(0, 16384, 8192 * len(devs))
        sel.append(b)
    ts = []
    for s in range(50):
        t = time.perf_counter()
        tr.train_step(g, [sx, sy], indexes=sel[s])
        ts.append(1e3 * (time.perf_counter() - t))
    knobs = " ".join("%s=%s" % (k, v) for k, v in sorted(os.environ.items()) if k.startswith("SYNK_"))
    print("C5 W=%d median %.4f ms  min %.4f  [%s]" % (len(devs), np.median(ts[10:]), min(ts[10:]), knobs or "defaults"))
