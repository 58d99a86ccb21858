"""Diagnostic (not collected): where a 1 KiB broadcast / all-reduce spends its
~12 us (W=2 ranks on GPU 0): Python floor, then the CUDA runtime calls of one
collective (CUPTI via torch.profiler)."""
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402

torch.cuda.init()
with sk.Pool(workers=2, devices=[0, 0]) as pool:
    var = sk.replicate(pool, np.zeros(256, np.float32))
    for name, fn in (("var.world", lambda: var.world), ("broadcast", lambda: var.broadcast(0)),
                     ("all_reduce", lambda: var.all_reduce("mean"))):
        for _ in range(100):
            fn()
        t = time.perf_counter()
        for _ in range(2000):
            fn()
        print("%-12s %6.2f us" % (name, (time.perf_counter() - t) / 2000 * 1e6))
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(3):
            var.broadcast(0)
    evs = sorted(prof.events(), key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    for e in evs:
        print("%8.1f %6.1f %-5s %s" % (e.time_range.start - t0, e.time_range.end - e.time_range.start,
                                       e.device_type.name, e.name[:60]))
