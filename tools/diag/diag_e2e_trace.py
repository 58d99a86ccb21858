"""Diagnostic (not collected): where the time of one e2e gather call goes
(bench.py's e2e leg: Function.call(indexes) with a row-count kernel over the
HBM mirror of a 10M x 256 f32 SharedInput). Prints per-call host time, the
CUDA runtime calls of one call (CUPTI via torch.profiler, plumbing only) and
the kernels/copies of that call."""
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
n_step = int(sys.argv[2]) if len(sys.argv) > 2 else 4096 * 64
rng = np.random.default_rng(0)
torch.cuda.init()
with sk.Pool(workers=1) as pool:
    arr = sk.SharedInput.alloc([rows, 256], "f32")
    arr.mirror(pool)
    f = sk.make_function(pool, sk.row_count_kernel(), ["scatter"], ["sum"])
    sk.distribute(pool)
    idx = []
    for _ in range(40):
        b = sk.pinned_array(n_step, "int64")
        b[:] = rng.integers(0, rows, n_step)
        idx.append(b)
    for s in range(5):
        f.call([arr], indexes=idx[s])
    t0 = time.perf_counter()
    for s in range(5, 35):
        f.call([arr], indexes=idx[s])
    dt = (time.perf_counter() - t0) / 30
    print("untraced: %.1f us/call = %.0f GB/s" % (1e6 * dt, n_step * 2056 / dt / 1e9))
    # floors on this box: one torch kernel + stream sync, and sync alone
    x = torch.zeros(1, device="cuda")
    for _ in range(100):
        x.add_(1)
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(1000):
        x.add_(1)
        torch.cuda.synchronize()
    print("torch 1 kernel + sync: %.1f us" % (1e3 * (time.perf_counter() - t0)))
    t0 = time.perf_counter()
    for _ in range(1000):
        x.add_(1)
        x.add_(1)
        torch.cuda.synchronize()
    print("torch 2 kernels + sync: %.1f us" % (1e3 * (time.perf_counter() - t0)))
    t0 = time.perf_counter()
    for _ in range(1000):
        torch.cuda.synchronize()
    print("sync alone: %.1f us" % (1e3 * (time.perf_counter() - t0)))
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for s in range(35, 40):
            f.call([arr], indexes=idx[s])
    evs = sorted(prof.events(), key=lambda e: e.time_range.start)
    cpu = [e for e in evs if e.device_type.name == "CPU" and e.name.startswith("cuda")]
    gpu = [e for e in evs if e.device_type.name == "CUDA"]
    t_end = max(e.time_range.end for e in evs)
    t_beg = min(e.time_range.start for e in evs)
    lo = t_end - (t_end - t_beg) / 5
    print("---- runtime calls of the last call (offset us, dur us, thread) ----")
    for e in cpu:
        if e.time_range.start >= lo:
            print("%8.1f %7.1f  tid=%-8s %s" % (e.time_range.start - lo, e.cpu_time_total, e.thread, e.name[:60]))
    print("---- kernels / copies of the last call ----")
    for e in gpu:
        if e.time_range.start >= lo:
            print("%8.1f %7.1f  %s" % (e.time_range.start - lo, e.time_range.end - e.time_range.start, e.name[:80]))
