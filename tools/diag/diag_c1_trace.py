"""Diagnostic (not collected): CUPTI trace (torch.profiler, plumbing only) of C1
sync-SGD steps: per-step host time, CUDA runtime calls of one step in order
(thread, offset, duration), kernels of that step."""
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
per_rank = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = sk.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
x, y = sk.mlp_make_dataset(65536, cfg, seed=2, dtype="f32")
rng = np.random.default_rng(0)
torch.cuda.init()
with sk.Pool(workers=world) as pool:
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

    sel = [pinned(per_rank * world) for _ in range(400)]
    for s in range(50):
        tr.train_step(g, [sx, sy], indexes=sel[s])
    t0 = time.perf_counter()
    for s in range(50, 350):
        tr.train_step(g, [sx, sy], indexes=sel[s])
    print("W=%d untraced: %.1f us/step" % (world, 1e6 * (time.perf_counter() - t0) / 300))
    print("last report:", tr.last_report)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for s in range(350, 356):
            tr.train_step(g, [sx, sy], indexes=sel[s])
    evs = sorted(prof.events(), key=lambda e: e.time_range.start)
    cpu = [e for e in evs if e.device_type.name == "CPU" and e.name.startswith("cuda")]
    gpu = [e for e in evs if e.device_type.name == "CUDA"]
    # one step = the last sixth of the window
    t_end = max(e.time_range.end for e in evs)
    t_beg = min(e.time_range.start for e in evs)
    span = (t_end - t_beg) / 6
    lo = t_end - span
    print("---- runtime calls of the last step (offset us, dur us, thread) ----")
    for e in cpu:
        if e.time_range.start >= lo:
            print("%8.1f %7.1f  tid=%-8s %s" % (e.time_range.start - lo, e.cpu_time_total, e.thread, e.name[:60]))
    print("---- kernels / copies of the last step ----")
    for e in gpu:
        if e.time_range.start >= lo:
            print("%8.1f %7.1f  %s" % (e.time_range.start - lo, e.time_range.end - e.time_range.start, e.name[:80]))
    agg = {}
    for e in cpu:
        a = agg.setdefault(e.name, [0, 0.0])
        a[0] += 1
        a[1] += e.cpu_time_total
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
        print("cpu %-40s n/step=%5.1f  us/step %8.1f" % (k[:40], c / 6, t / 6))
