"""Diagnostic (not collected by pytest): a few C5 (wide MLP, bf16 tcgen05) sync-SGD steps,
for an ncu launch list (kernel mix and shares of one step)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dims = [2048, 4096, 4096, 100]
cfg = sk.MlpConfig(in_dim=dims[0], width=dims[1], out_dim=dims[-1], layers=3, seed=1)
rng = np.random.default_rng(0)
x = rng.standard_normal((16384, 2048), dtype=np.float32)
y = rng.standard_normal((16384, 100), dtype=np.float32)
with sk.Pool(workers=1) as pool:
    sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
    sx.mirror(pool)
    sy.mirror(pool)
    block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
    g = sk.mlp_grad_function(pool, block, compute="bf16")
    sk.distribute(pool)
    tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
    for s in range(steps):
        t0 = time.perf_counter()
        loss = tr.train_step(g, [sx, sy], indexes=rng.integers(0, 16384, 8192))
        rep = tr.last_report
        print("step %d  %.3f ms  grad_call %.3f ms (compute %.3f, scatter %.3f)  allreduce %.3f ms  loss %.4f"
              % (s, 1e3 * (time.perf_counter() - t0), 1e3 * rep["grad_call"]["total_s"],
                 1e3 * max(rep["grad_call"]["rank_compute_s"]), 1e3 * rep["grad_call"]["scatter_s"],
                 1e3 * rep["allreduce_s"], loss))
