"""Diagnostic (not collected): CUPTI trace (torch.profiler, plumbing only) of C5 steps
to find device stalls: prints every GPU activity longer than 1 ms and per-step spans."""
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_1710_04162_b200 as sk  # noqa: E402


def pin(a):
    b = sk.pinned_array(a.size, "int64")
    b[:] = a
    return b

dims = [2048, 4096, 4096, 100]
cfg = sk.MlpConfig(in_dim=dims[0], width=dims[1], out_dim=dims[-1], layers=3, seed=1)
rng = np.random.default_rng(0)
x = rng.standard_normal((16384, 2048), dtype=np.float32)
y = rng.standard_normal((16384, 100), dtype=np.float32)
torch.cuda.init()
with sk.Pool(workers=1) as pool:
    sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
    sx.mirror(pool)
    sy.mirror(pool)
    block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
    g = sk.mlp_grad_function(pool, block, compute="bf16")
    sk.distribute(pool)
    tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
    sel = [pin(rng.integers(0, 16384, 8192)) for _ in range(15)]
    for s in range(3):
        tr.train_step(g, [sx, sy], indexes=sel[12 + s])
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for s in range(12):
            t0 = time.perf_counter()
            tr.train_step(g, [sx, sy], indexes=sel[s])
            print("step %d %.3f ms" % (s, 1e3 * (time.perf_counter() - t0)))
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    print(len(evs), "cuda events")
    long = sorted(evs, key=lambda e: -e.device_time_total)[:15]
    for e in long:
        print("%10.1f us  %s" % (e.device_time_total, e.name[:90]))
    # gaps between consecutive kernels on the device timeline
    ks = sorted(evs, key=lambda e: e.time_range.start)
    gaps = []
    for a, b in zip(ks, ks[1:]):
        gaps.append((b.time_range.start - a.time_range.end, a.name[:50], b.name[:50]))
    for gp in sorted(gaps, reverse=True)[:8]:
        print("gap %10.1f us  after %s  before %s" % gp)
    t_end = max(e.time_range.end for e in evs)
    last = [e for e in sorted(evs, key=lambda e: e.time_range.start) if e.time_range.start >= t_end - 1500]
    print("---- launches of the last ~1.5 ms ----")
    for e in last:
        print("%8.1f %8.1f  %s" % (e.time_range.start - last[0].time_range.start, e.time_range.end - e.time_range.start,
                                    e.name[:70]))
    agg_k = {}
    for e in evs:
        a = agg_k.setdefault(e.name[:70], [0, 0.0])
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
    print("---- device time per step by kernel ----")
    for k, (c, t) in sorted(agg_k.items(), key=lambda kv: -kv[1][1])[:25]:
        print("%9.1f us/step  n/step=%5.1f  %s" % (t / 12, c / 12, k))
    cpu = [e for e in prof.events() if e.device_type.name == "CPU"]
    agg = {}
    for e in cpu:
        a = agg.setdefault(e.name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += e.cpu_time_total
        a[2] = max(a[2], e.cpu_time_total)
    for k, (c, t, m) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
        print("cpu %-40s n=%5d total %10.1f us  max %10.1f us" % (k[:40], c, t, m))
    # host runtime calls around the last step boundary (offsets vs the last device kernel of the step before)
    allev = sorted(prof.events(), key=lambda e: e.time_range.start)
    cu = [e for e in allev if e.device_type.name == "CPU" and e.name.startswith("cuda")]
    ks_end = [e for e in ks if "copy_small" in e.name]
    if len(ks_end) >= 2:
        t_b = ks_end[-2].time_range.end
        print("---- runtime calls within 120 us after the previous step's last kernel ----")
        for e in cu:
            if t_b - 60 <= e.time_range.start <= t_b + 120:
                print("%8.1f %6.1f %s" % (e.time_range.start - t_b, e.cpu_time_total, e.name[:50]))
        nxt = [e for e in ks if e.time_range.start > t_b]
        if nxt:
            print("next device activity at +%.1f us: %s" % (nxt[0].time_range.start - t_b, nxt[0].name[:60]))
