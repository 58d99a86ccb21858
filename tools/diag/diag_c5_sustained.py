"""Diagnostic (not collected): C5 sync-SGD steps back to back for ~3 s with
nvidia-smi sampling (SM clock, power) -- the sustained-power regime the
MEASURED_PEAKS 'sustained' bf16 figure describes."""
import subprocess
import sys
import threading
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

dims = [2048, 4096, 4096, 100]
cfg = sk.MlpConfig(in_dim=dims[0], width=dims[1], out_dim=dims[-1], layers=3, seed=1)
x, y = sk.mlp_make_dataset(16384, cfg, seed=2, dtype="f32")
rng = np.random.default_rng(0)
lines = []
with sk.Pool(workers=1) as pool:
    sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
    sx.mirror(pool)
    sy.mirror(pool)
    block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
    g = sk.mlp_grad_function(pool, block, compute="bf16")
    sk.distribute(pool)
    tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
    sel = []
    for _ in range(64):
        b = sk.pinned_array(8192, "int64")
        b[:] = rng.integers(0, 16384, 8192)
        sel.append(b)
    for s in range(10):
        tr.train_step(g, [sx, sy], indexes=sel[s % 64])
    proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                             "-lms", "100"], stdout=subprocess.PIPE, text=True)
    threading.Thread(target=lambda: [lines.append(l.strip()) for l in proc.stdout], daemon=True).start()
    t0 = time.perf_counter()
    n = 0
    marks = []
    while time.perf_counter() - t0 < 3.0:
        tr.train_step(g, [sx, sy], indexes=sel[n % 64])
        n += 1
        if n % 250 == 0:
            marks.append((n, time.perf_counter() - t0))
    dt = time.perf_counter() - t0
    proc.terminate()
flops = (6 * sum(a * b for a, b in zip(dims[:-1], dims[1:])) - 2 * dims[0] * dims[1]) * 8192
print("steps %d in %.2f s: %.3f ms/step, %.0f model TFLOP/s" % (n, dt, 1e3 * dt / n, flops * n / dt / 1e12))
prev = (0, 0.0)
for m in marks:
    print("  steps %4d-%4d: %.3f ms/step" % (prev[0], m[0], 1e3 * (m[1] - prev[1]) / (m[0] - prev[0])))
    prev = m
vals = [tuple(float(v) for v in l.split(",")) for l in lines if l.count(",") == 1]
if vals:
    sm = sorted(v[0] for v in vals)
    pw = sorted(v[1] for v in vals)
    print("SM clock MHz median %.0f (min %.0f), power W median %.0f (max %.0f), %d samples"
          % (sm[len(sm) // 2], sm[0], pw[len(pw) // 2], pw[-1], len(vals)))
