"""Diagnostic (not collected; for ncu): a few C1 sync-SGD steps (784-512-10 f32,
batch 256, W=1)."""
import sys

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
    for s in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
        tr.train_step(g, [sx, sy], indexes=rng.integers(0, 65536, 256))
print("ok")
