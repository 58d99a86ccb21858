#!/usr/bin/env python3
"""Benchmark of the Synkhronos hot path on B200 (one JSON line on stdout).

Headline workload (BASELINE.json configs[1]): input-indexing gather of
shuffled 4096-row batches from a 10M x 256 fp32 shared dataset.

  value    device-timed gather throughput (CUDA events on each rank's
           stream, max over GPUs) with the dataset resident in HBM (the
           SharedInput's HBM mirror), one launch per step covering
           `--batches` x 4096 rows per GPU. Algorithmic bytes per row:
           1024 read + 1024 written + 8 index = 2056 B.
  e2e      the same metric through the public API (Function.call with
           indexes, row-count kernel, Sum): every step copies its u64 index
           list host->device and reads the f64 result back.
  roofline gather kernel: algorithmic bytes / average launch duration vs
           the measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline  the unmodified reference (oracle/_ref/ref_driver, C++20)
           on this box's cores, bounded sample of the same workload.
  sync_sgd C1 (784-512-10 fp32 MLP, batch 256/GPU indexed, grad all-reduce
           mean fused with the SGD update), samples/s through Trainer.
  sync_sgd_wide_bf16  C5 (2048-4096-4096-100, bf16 tcgen05 GEMMs, 8192/GPU).
  slicing_c3  C3: column sums + maxima (+ Gather) over an 8M x 1024 fp32
           HBM-resident input, num_slices=4, vs the HBM roofline.
  collectives_c4  C4: all-reduce mean + broadcast sweep 1 KiB - 1 GiB.

`--impl reference` times only the reference CPU implementation on the same
config and prints its line. Under torchrun (N>1) the synkpar executor is one
process driving all N GPUs (the paper's master + workers model): rank 0 owns
the pool; other ranks wait at a gloo barrier.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sync-SGD samples/s at 1/2/4/8 B200; gather/reduce GB/s vs HBM & NVLink peak"
BYTES_PER_ROW_EXTRA = 8  # u64 index


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rows", type=int, default=10_000_000)
    p.add_argument("--cols", type=int, default=256)
    p.add_argument("--batch", type=int, default=4096)
    p.add_argument("--batches", type=int, default=64, help="4096-row batches gathered per launch (per step)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-sgd", action="store_true")
    p.add_argument("--no-c3", action="store_true", help="skip the C3 slicing/aggregation sub-measurement")
    p.add_argument("--c3-rows", type=int, default=8_388_608)
    p.add_argument("--c3-cols", type=int, default=1024)
    p.add_argument("--c3-slices", type=int, default=4)
    p.add_argument("--no-c4", action="store_true", help="skip the C4 shared-variable sync sweep")
    p.add_argument("--dry-run", action="store_true",
                   help="exercise only the launch/rank coordination (no GPU work); used by CPU tests")
    return p.parse_args()


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


TRAFFIC_CAPTURE = "profiles/r02_gather_ncu_full_raw.csv"


def ncu_traffic(bytes_per_launch, path=TRAFFIC_CAPTURE):
    """dram__bytes_read.sum + dram__bytes_write.sum of the committed
    `ncu --set full` capture of the same gather launch (same rows per launch),
    or None when the capture does not match this launch size."""
    try:
        vals = {}
        with open(os.path.join(ROOT, path)) as fh:
            for line in fh:
                f = line.strip().split(",")
                if len(f) == 3:
                    vals[f[0]] = (f[1], f[2])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        total = sum(float(vals[k][1]) * scale[vals[k][0]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        captured = float(vals.get("synk__algorithmic_bytes_per_launch", ("", "538968064"))[1])
        return total if abs(captured - bytes_per_launch) < 1 else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.lines = []

    def __enter__(self):
        if self.gpus <= 0:  # a non-zero torchrun rank: rank 0 samples every GPU of the box
            return self
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + q, "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or not f[0].isdigit() or int(f[0]) >= self.gpus:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method="env://", world_size=world, rank=rank)
        return rank, world, dist
    return rank, world, None


def run_reference_driver(mode, extra, timeout=1800):
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if not os.path.exists(exe):
        return None, "oracle/_ref/ref_driver not built"
    out = subprocess.run([exe, "--mode", mode, *map(str, extra)], capture_output=True, text=True, timeout=timeout)
    if out.returncode != 0:
        return None, out.stderr.strip()[-300:]
    return json.loads(out.stdout.strip().splitlines()[-1]), None


def reference_arm(args, n_gpus):
    cores = os.cpu_count() or 1
    rows_per_step = args.batch * args.batches * n_gpus
    steps = max(1, args.steps)
    res, err = run_reference_driver("gather", ["--rows", args.rows, "--cols", args.cols, "--batch", rows_per_step,
                                               "--steps", steps, "--warmup", max(1, min(args.warmup, 3)),
                                               "--workers", cores])
    line = {"impl": "reference", "metric": METRIC, "unit": "GB/s", "higher_is_better": True, "n_gpus": n_gpus,
            "steps": steps, "warmup": args.warmup, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, n_gpus)}
    if res is None:
        line["unavailable"] = err
        return line
    line.update({"value": res["gbs"], "ms_per_step": res["ms_per_step"],
                 "cpu_baseline": {"value": res["gbs"], "unit": "GB/s", "cores": res["workers"], "kind": "reference",
                                  "cpu_model": cpu_model(), "sample": "%d steps x %d rows gathered through call(indexes) with a no-op kernel "
                                            "from a %dx%d f32 SharedInputArray" % (steps, rows_per_step, args.rows,
                                                                                    args.cols)},
                 "e2e": {"value": res["gbs"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    return line


def workload_config(args, n_gpus):
    return {"workload": "indexed gather: shuffled %d-row batches from a %dx%d fp32 shared dataset" % (
        args.batch, args.rows, args.cols), "batches_per_step_per_gpu": args.batches,
        "rows_per_step": args.batch * args.batches * n_gpus, "row_bytes": args.cols * 4,
        "parallelism": "dp%d (one rank per GPU; under torchrun one process per GPU for this headline)" % n_gpus,
        "l2": "inputs larger than L2 (10.24 GB dataset, 2 rotating 256 MiB outputs per GPU)"}


def pinned_indexes(sk, rng, rows, n):
    """A step's index list in pinned host memory (what a data loader hands over)."""
    buf = sk.pinned_array(n, "int64")
    buf[:] = rng.integers(0, rows, n)
    return buf


def fill_dataset(sk, rows, cols):
    arr = sk.SharedInput.alloc([rows, cols], "f32")
    rng = np.random.default_rng(7)
    block = 1 << 18
    for r0 in range(0, rows, block):
        n = min(block, rows - r0)
        arr.write(r0, r0 + n, rng.random((n, cols), dtype=np.float32) * 2 - 1)
    return arr


def slicing_c3(sk, pool, args, n_gpus, peak, peak_kind):
    """C3: column sums (Sum) + column maxima (Max) + the shard (Gather) over an
    HBM-resident rows x cols f32 input scattered over the GPUs, num_slices
    slices per rank. Algorithmic bytes = one read of the input (4*rows*cols);
    the Gather output additionally crosses PCIe to the host result."""
    rows, cols, slices = args.c3_rows, args.c3_cols, args.c3_slices
    nbytes = rows * cols * 4
    t0 = time.time()
    x = sk.replicate(pool, np.zeros(1, np.float32))
    x.scatter_uniform([rows, cols], "f32", 3)
    gen_s = time.time() - t0
    f_red = sk.make_function(pool, sk.column_stats_kernel(with_shard=False), ["scatter"], ["sum", "max"])
    f_all = sk.make_function(pool, sk.column_stats_kernel(), ["scatter"], ["sum", "max", "gather"])
    sk.distribute(pool)

    def run(f, warm, steps):
        for _ in range(warm):
            f.call([x], num_slices=slices)
        dev, host = [], 0.0
        for _ in range(steps):
            t = time.perf_counter()
            outs, rep = f.call_with_report([x], num_slices=slices)
            host += time.perf_counter() - t
            dev.append(max(rep["rank_compute_s"]))
            del outs
        return host / steps, float(np.mean(dev)), rep

    red_host, red_dev, _ = run(f_red, 3, 10)
    all_host, all_dev, rep = run(f_all, 2, 3)
    per_gpu = nbytes / n_gpus
    out = {"config": "C3: %dx%d f32 (%.1f GiB) HBM-resident (scatter_uniform), num_slices=%d per rank, "
                     "column_stats kernel (Sum, Max[, Gather])" % (rows, cols, nbytes / 2**30, slices),
           "algorithmic_bytes_per_call": nbytes,
           "reduce_only": {"outputs": "sum, max", "ms_per_call": 1e3 * red_host,
                           "e2e_gbs": nbytes / red_host / 1e9, "device_gbs": nbytes / red_dev / 1e9,
                           "roofline": {"bound": "hbm", "achieved": per_gpu / red_dev / 1e9, "peak": peak,
                                        "unit": "GB/s", "frac": per_gpu / red_dev / 1e9 / peak, "peak_kind": peak_kind,
                                        "kernel": "colstats_partial_kernel + colstats_final_kernel (4 slices)"}},
           "with_gather": {"outputs": "sum, max, gather", "ms_per_call": 1e3 * all_host,
                           "e2e_gbs": nbytes / all_host / 1e9, "device_gbs": nbytes / all_dev / 1e9,
                           "d2h_bytes_per_call": nbytes, "reduce_s": rep["reduce_s"],
                           "note": "e2e bound by the %.1f GiB Gather result crossing PCIe into a pinned host "
                                   "buffer" % (nbytes / 2**30)},
           "generate_s": gen_s}
    if not args.no_cpu_baseline and n_gpus >= 1:
        sample = 262144
        res, err = run_reference_driver("slicing", ["--rows", sample, "--cols", cols, "--slices", slices,
                                                    "--steps", 2, "--warmup", 1, "--workers", os.cpu_count() or 1])
        out["cpu_baseline"] = err and {"unavailable": err} or {
            "value": res["gbs"], "unit": "GB/s", "cores": res["workers"], "kind": "reference", "cpu_model": cpu_model(),
            "sample": "2 calls over %dx%d f32 (explicit scatter input), num_slices=%d, Sum+Max+Gather" % (
                sample, cols, slices)}
    return out


def gather_headline(args, n_gpus, devices, dist, world):
    """C2 headline on this process's GPUs (`devices`): value / e2e / roofline.
    Under torchrun every rank runs this on its own GPU with its own one-GPU
    pool (the path partitions: no data-path collective); times are the max
    over ranks, bytes the sum."""
    import paper_1710_04162_b200 as sk

    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1710_04162_b200", "_lib", "libsynk_cuda.so"))
    lib.synk_last_error.restype = ctypes.c_char_p
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64

    def ok(rc, what):
        if rc != 0:
            raise RuntimeError("%s: %s" % (what, lib.synk_last_error().decode()))

    rows, cols, B = args.rows, args.cols, args.batch
    row_bytes = cols * 4
    n_step = B * args.batches  # rows per GPU per step
    peak, peak_kind = measured_peak_hbm()

    t_setup = time.time()
    arr = fill_dataset(sk, rows, cols)
    pool = sk.Pool(workers=len(devices), devices=list(devices))
    n_local = len(devices)
    arr.mirror(pool)
    setup_s = time.time() - t_setup

    handles = [vp(pool.device_handle(r)) for r in range(n_local)]
    rng = np.random.default_rng(11)
    total_steps = args.warmup + args.steps
    idx_dev, dst_dev, mirrors = [], [], []
    for r in range(n_local):
        h = handles[r]
        idx = rng.integers(0, rows, total_steps * n_step).astype(np.uint64)
        p = vp()
        ok(lib.synk_alloc(h, u64(idx.nbytes), ctypes.byref(p)), "alloc idx")
        ok(lib.synk_copy(h, p, idx.ctypes.data_as(vp), u64(idx.nbytes)), "H2D idx")
        idx_dev.append(p.value)
        outs = []
        for _ in range(2):
            q = vp()
            ok(lib.synk_alloc(h, u64(n_step * row_bytes), ctypes.byref(q)), "alloc out")
            outs.append(q.value)
        dst_dev.append(outs)
        mirrors.append(arr.mirror_ptr(pool.device_of(r)))
        ok(lib.synk_sync(h), "sync")

    def gather_launches(step_rows, steps, warm, per_launch_marks=True):
        """Launch `steps` gathers of step_rows rows per GPU; return (max over GPUs of
        the device time of the timed region, mean per-launch kernel time)."""
        marks = [[] for _ in range(n_local)]
        for r in range(n_local):
            ok(lib.synk_mark_reset(handles[r]), "marks")
        for s in range(warm + steps):
            for r in range(n_local):
                h = handles[r]
                m = ctypes.c_int()
                if s >= warm:
                    ok(lib.synk_mark(h, ctypes.byref(m)), "mark")
                    marks[r].append(m.value)
                ok(lib.synk_gather_rows(h, vp(mirrors[r]), u64(rows), u64(row_bytes),
                                        vp(idx_dev[r] + (s * step_rows % (total_steps * n_step - step_rows + 1)) * 8),
                                        u64(step_rows), vp(dst_dev[r][s % 2])), "gather")
                if s >= warm:
                    ok(lib.synk_mark(h, ctypes.byref(m)), "mark")
                    marks[r].append(m.value)
        region, launch = [], []
        for r in range(n_local):
            ok(lib.synk_sync(handles[r]), "sync")
            sec = ctypes.c_double()
            ok(lib.synk_mark_elapsed(handles[r], marks[r][0], marks[r][-1], ctypes.byref(sec)), "elapsed")
            region.append(sec.value)
            tot = 0.0
            for a, b in zip(marks[r][0::2], marks[r][1::2]):
                ok(lib.synk_mark_elapsed(handles[r], a, b, ctypes.byref(sec)), "elapsed")
                tot += sec.value
            launch.append(tot / steps)
        return max(region), float(np.mean(launch))

    def max_over_ranks(x):
        if dist is None:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if dist is not None:
            dist.barrier()

    sampler = ClockSampler(n_gpus) if not dist or dist.get_rank() == 0 else ClockSampler(0)
    with sampler as clocks:
        # Soak under the same load first so nvidia-smi (200 ms cadence) samples
        # clocks around the timed region even when K steps take milliseconds.
        t_soak = time.time()
        while time.time() - t_soak < 1.5:
            gather_launches(n_step, 16, 0)
        barrier()
        region_s, launch_s = gather_launches(n_step, args.steps, args.warmup)
        region_s, launch_s = max_over_ranks(region_s), max_over_ranks(launch_s)
        time.sleep(0.25)
    bytes_step = world * n_local * n_step * (2 * row_bytes + BYTES_PER_ROW_EXTRA)  # all GPUs of the job
    value = bytes_step * args.steps / region_s / 1e9
    achieved = n_step * (2 * row_bytes + BYTES_PER_ROW_EXTRA) / launch_s / 1e9
    # latency of a single 4096-row batch (the per-call granularity of the config)
    _, single_s = gather_launches(B, 50, 5)

    # ---- the same gather with the dataset left in pinned, mapped HOST memory
    # (the paper's default: rows pulled over PCIe by the kernel), against the
    # PCIe copy bandwidth measured here (1 GiB pinned source, 256 MiB per launch)
    host_src = None
    if not dist or dist.get_rank() == 0:
        h = handles[0]
        hbytes = 1 << 30
        hp = vp()
        ok(lib.synk_host_alloc(u64(hbytes), ctypes.byref(hp)), "host alloc")
        try:
            ctypes.memset(hp, 0x3F, hbytes)
            hrows = hbytes // row_bytes
            hidx = rng.integers(0, hrows, n_step).astype(np.uint64)
            d_hidx, d_out, d_cpy = vp(), vp(), vp()
            ok(lib.synk_alloc(h, u64(hidx.nbytes), ctypes.byref(d_hidx)), "alloc")
            ok(lib.synk_alloc(h, u64(n_step * row_bytes), ctypes.byref(d_out)), "alloc")
            ok(lib.synk_alloc(h, u64(n_step * row_bytes), ctypes.byref(d_cpy)), "alloc")
            ok(lib.synk_copy(h, d_hidx, hidx.ctypes.data_as(vp), u64(hidx.nbytes)), "H2D idx")
            ok(lib.synk_sync(h), "sync")

            def timed(fn, reps=5):
                for _ in range(2):
                    fn()
                m0, m1 = ctypes.c_int(), ctypes.c_int()
                ok(lib.synk_mark_reset(h), "marks")
                ok(lib.synk_mark(h, ctypes.byref(m0)), "mark")
                for _ in range(reps):
                    fn()
                ok(lib.synk_mark(h, ctypes.byref(m1)), "mark")
                ok(lib.synk_sync(h), "sync")
                sec = ctypes.c_double()
                ok(lib.synk_mark_elapsed(h, m0.value, m1.value, ctypes.byref(sec)), "elapsed")
                return sec.value / reps

            t_g = timed(lambda: ok(lib.synk_gather_rows(h, hp, u64(hrows), u64(row_bytes), d_hidx, u64(n_step),
                                                        d_out), "gather (host source)"))
            t_c = timed(lambda: ok(lib.synk_copy(h, d_cpy, hp, u64(n_step * row_bytes)), "H2D copy"))
            pcie = n_step * row_bytes / t_c / 1e9
            over_pcie = n_step * row_bytes / t_g / 1e9
            host_src = {"config": "C2 gather with the dataset in pinned, mapped host memory (1 GiB sample, %d rows "
                                  "per launch): rows travel over PCIe inside the gather kernel" % n_step,
                        "row_gbs_over_pcie": over_pcie, "pcie_h2d_copy_gbs": pcie,
                        "frac_of_pcie_copy": over_pcie / pcie, "us_per_launch": 1e6 * t_g}
            for p_ in (d_hidx, d_out, d_cpy):
                lib.synk_free(h, p_)
            ok(lib.synk_sync(h), "sync")
        finally:
            lib.synk_host_free(hp)

    # ---- e2e through the public API --------------------------------------------------
    f = sk.make_function(pool, sk.row_count_kernel(), ["scatter"], ["sum"])
    sk.distribute(pool)
    # Per-step index lists live in pinned host memory (sk.pinned_array): the call
    # reads them in place and DMAs each rank's part (filled before timing, as a
    # data loader would hand them over).
    e2e_idx = []
    for _ in range(total_steps):
        buf = sk.pinned_array(n_step * n_local, "int64")
        buf[:] = rng.integers(0, rows, n_step * n_local)
        e2e_idx.append(buf)
    for s in range(args.warmup):
        (cnt,) = f.call([arr], indexes=e2e_idx[s])
        assert float(cnt) == n_step * n_local
    barrier()
    t0 = time.perf_counter()
    for s in range(args.warmup, total_steps):
        (cnt,) = f.call([arr], indexes=e2e_idx[s])
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    assert float(cnt) == n_step * n_local
    e2e = bytes_step * args.steps / e2e_s / 1e9
    # where the e2e time goes (untimed repeat with the call report)
    rep_acc = {"scatter_s": 0.0, "reduce_s": 0.0, "total_s": 0.0, "compute_s": 0.0}
    for s in range(args.warmup, total_steps):
        _, rep = f.call_with_report([arr], indexes=e2e_idx[s])
        for k in ("scatter_s", "reduce_s", "total_s"):
            rep_acc[k] += rep[k] / args.steps
        rep_acc["compute_s"] += max(rep["rank_compute_s"]) / args.steps
    e2e_breakdown = {k + "_us": 1e6 * v for k, v in rep_acc.items()}
    # the config's own granularity: ONE 4096-row batch per GPU per Function.call
    one_idx = []
    for _ in range(220):
        buf = sk.pinned_array(B * n_local, "int64")
        buf[:] = rng.integers(0, rows, B * n_local)
        one_idx.append(buf)
    for s in range(20):
        f.call([arr], indexes=one_idx[s])
    barrier()
    t0 = time.perf_counter()
    for s in range(20, 220):
        (cnt,) = f.call([arr], indexes=one_idx[s])
    one_s = max_over_ranks((time.perf_counter() - t0) / 200)
    assert float(cnt) == B * n_local
    single_call = {"rows_per_gpu": B, "us_per_call": 1e6 * one_s,
                   "gbs": world * n_local * B * (2 * row_bytes + BYTES_PER_ROW_EXTRA) / one_s / 1e9,
                   "h2d_bytes_per_call": 8 * B * n_local, "d2h_bytes_per_call": 8}

    pool.shutdown()
    del arr
    return {"value": value, "region_s": region_s, "e2e": e2e, "e2e_breakdown": e2e_breakdown,
            "single_call": single_call, "achieved": achieved,
            "single_s": single_s, "clocks": clocks.summary(), "host_source": host_src,
            "setup_s": setup_s, "n_step": n_step, "row_bytes": row_bytes, "peak": peak, "peak_kind": peak_kind}


# ---- sync SGD (C1, C5): per-N samples/s, scaling and the paper's Table-1 split ----------

SGD_MODELS = {
    "c1": {"dims": [784, 512, 10], "per_gpu": 256, "rows": 65536, "compute": "native", "warm": 30, "dtype": "f32",
           "label": "C1: MLP 784-512-10 fp32 (tcgen05 3xTF32 GEMMs at fp32 accuracy), indexed from a 65536-row SharedInput (HBM mirror), "
                    "SGD lr 0.01, gradient all-reduce mean fused with the update"},
    "c5": {"dims": [2048, 4096, 4096, 100], "per_gpu": 8192, "rows": 16384, "compute": "bf16", "warm": 3,
           "dtype": "bf16",
           "label": "C5 (R1): MLP 2048-4096-4096-100 (25,583,716 params, fp32 master), bf16 tcgen05 GEMMs "
                    "(CTA-pair 256x256 tiles for the wide layers), indexed from a 16384-row HBM mirror, SGD lr 0.01, "
                    "gradient all-reduce mean + update fused; at W > 1 bucketed per layer and overlapped with the "
                    "backward pass, at W = 1 one update after it"},
}


def flops_per_sample(dims):
    """Forward + weight-gradient + input-gradient products of the MLP (no dX
    for layer 0): 6*sum(d_l*d_{l+1}) - 2*d_0*d_1."""
    return 6 * sum(a * b for a, b in zip(dims[:-1], dims[1:])) - 2 * dims[0] * dims[1]


def gpu_counts(n_gpus):
    """The paper's 1/2/4/8 sweep, capped at the job's GPUs (and the job size itself)."""
    ns = [n for n in (1, 2, 4, 8) if n <= n_gpus]
    return ns if n_gpus in ns else ns + [n_gpus]


def measure_sgd(sk, model, devices, per_rank, steps, warmup, seed, sustained_s=0.0):
    """One pool over `devices`; `steps` timed train_steps (host clock around
    the calls: the pinned index list goes H2D, the loss comes back D2H every
    step), then an untimed repeat of as many steps read through
    Trainer.last_report for the Table-1 split (the reference accounting,
    src/bench.cpp:186-198), then optionally `sustained_s` seconds back to back."""
    m = SGD_MODELS[model]
    dims, n = m["dims"], len(devices)
    gb = per_rank * n
    with sk.Pool(workers=n, devices=list(devices)) as pool:
        cfg = sk.MlpConfig(in_dim=dims[0], width=dims[1], out_dim=dims[-1], layers=len(dims) - 1, seed=1)
        x, y = sk.mlp_make_dataset(m["rows"], cfg, seed=2, dtype="f32")
        sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
        sx.mirror(pool)
        sy.mirror(pool)
        block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
        g = sk.mlp_grad_function(pool, block, compute=m["compute"])
        sk.distribute(pool)
        tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
        rng = np.random.default_rng(seed)
        # Latency-bound C1 steps: a longer untimed warm-up lets the per-rank
        # CUDA-graph cache settle on the recycled batch buffers.
        warm = max(warmup, m["warm"])
        sel = [pinned_indexes(sk, rng, m["rows"], gb) for _ in range(warm + 2 * steps)]
        for s in range(warm):
            tr.train_step(g, [sx, sy], indexes=sel[s])
        t0 = time.perf_counter()
        for s in range(warm, warm + steps):
            loss = tr.train_step(g, [sx, sy], indexes=sel[s])
        dt = time.perf_counter() - t0
        t1 = {"function_s": 0.0, "shuffle_s": 0.0, "straggler_s": 0.0, "allreduce_s": 0.0, "total_s": 0.0}
        for s in range(warm + steps, warm + 2 * steps):
            t = time.perf_counter()
            tr.train_step(g, [sx, sy], indexes=sel[s])
            t1["total_s"] += time.perf_counter() - t
            rep = tr.last_report
            gc, sc = rep["grad_call"], rep["step_call"]
            t1["function_s"] += float(np.mean(gc["rank_compute_s"])) + (
                float(np.mean(sc["rank_compute_s"])) if sc["rank_compute_s"] else 0.0)
            t1["shuffle_s"] += gc["scatter_s"]
            t1["straggler_s"] += gc["straggler_s"] + sc["straggler_s"]
            t1["allreduce_s"] += rep["allreduce_s"]
        sustained = None
        if sustained_s > 0:
            k, t = 0, time.perf_counter()
            while time.perf_counter() - t < sustained_s:
                tr.train_step(g, [sx, sy], indexes=sel[k % len(sel)])
                k += 1
            el = time.perf_counter() - t
            sustained = {"seconds": el, "steps": k, "ms_per_step": 1e3 * el / k, "samples_per_s": gb * k / el}
        return {"n_gpus": n, "devices": list(devices), "global_batch": gb, "per_rank_batch": per_rank,
                "steps": steps, "seconds": dt, "samples_per_s": gb * steps / dt, "ms_per_step": 1e3 * dt / steps,
                "table1": t1, "loss_last": float(loss), "coherent": bool(block.params.coherent),
                "n_params": int(block.length), "sustained": sustained}


def stub_sgd(model, devices, per_rank, steps, sustained_s=0.0):
    """--dry-run stand-in for measure_sgd (no GPU): the same record shape with
    synthetic timings (a fixed per-step time plus a 2 % per-GPU overhead)."""
    n = len(devices)
    ms = (0.11 if model == "c1" else 1.14) * (1 + 0.02 * (n - 1))
    dt = ms * steps / 1e3
    t1 = {"function_s": 0.8 * dt, "shuffle_s": 0.05 * dt, "straggler_s": 0.01 * dt, "allreduce_s": 0.1 * dt,
          "total_s": dt}
    gb = per_rank * n
    return {"n_gpus": n, "devices": list(devices), "global_batch": gb, "per_rank_batch": per_rank, "steps": steps,
            "seconds": dt, "samples_per_s": gb * steps / dt, "ms_per_step": ms, "table1": t1, "loss_last": 1.0,
            "coherent": True, "n_params": 0, "stub": True,
            "sustained": {"seconds": sustained_s, "steps": 1, "ms_per_step": ms, "samples_per_s": gb / ms * 1e3}
            if sustained_s > 0 else None}


def scaling_summary(runs, model):
    """speedup_vs_1 / speedup_vs_2 as the reference bench (src/bench.cpp:213-221),
    efficiency = speedup_vs_1 / N (the north star: >= 0.9 at N=8), Table-1 per
    step in microseconds and as fractions of the step."""
    base = {r["n_gpus"]: r["samples_per_s"] for r in runs}
    dims = SGD_MODELS[model]["dims"]
    for r in runs:
        n = r["n_gpus"]
        r["speedup_vs_1"] = r["samples_per_s"] / base[1] if 1 in base else None
        r["speedup_vs_2"] = r["samples_per_s"] / base[2] if 2 in base else None
        r["efficiency_vs_linear"] = r["speedup_vs_1"] / n if r["speedup_vs_1"] is not None else None
        t1 = r["table1"]
        tot = t1["total_s"] or 1e-30
        r["table1_per_step_us"] = {k.replace("_s", ""): 1e6 * v / r["steps"] for k, v in t1.items()}
        r["table1_frac"] = {k.replace("_s", ""): v / tot for k, v in t1.items() if k != "total_s"}
        r["model_tflops_per_gpu"] = flops_per_sample(dims) * r["samples_per_s"] / n / 1e12
    return runs


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def reference_sgd(worker_counts, steps=3):
    """The unmodified reference's SyncSgd::train_step (oracle/_ref/ref_driver
    --mode sgd: src/sgd.cpp:259-332 through its public API) on this box's
    cores, W threads pinned, timed in this run: configs[0] exactly (W=2,
    batch 256 global) and the scaled sweep (256 rows per worker)."""
    cores = os.cpu_count() or 1
    out = {"kind": "reference", "cpu_model": cpu_model(), "host_cores": cores,
           "timing": "steady clock around SyncSgd::train_step; Table-1 split from the reference's StepReport"}
    res, err = run_reference_driver("sgd", ["--workers", 2, "--batch", 256, "--steps", max(steps, 3), "--warmup", 1])
    out["configs0_exact"] = err and {"unavailable": err} or dict(res, cores=2, sample="%d steps" % res["steps"])
    runs = []
    for w in worker_counts:
        if w > cores:
            continue
        res, err = run_reference_driver("sgd", ["--workers", w, "--batch", 256 * w, "--steps", steps, "--warmup", 1])
        if res is None:
            runs.append({"workers": w, "unavailable": err})
            continue
        runs.append(dict(res, cores=w))
    b1 = next((r["samples_per_s"] for r in runs if r.get("workers") == 1 and "samples_per_s" in r), None)
    for r in runs:
        if b1 and "samples_per_s" in r:
            r["speedup_vs_1"] = r["samples_per_s"] / b1
    out["scaled"] = runs
    return out


def tree_fold(vals, op):
    """The reference's binomial collective order (replicated.cpp:16-29):
    step = 1, 2, 4, ...: acc[r] = acc[r] op acc[r + step] for r = 0, 2*step, ..."""
    acc = [v.copy() for v in vals]
    step = 1
    while step < len(acc):
        for r in range(0, len(acc) - step, 2 * step):
            a, b = acc[r], acc[r + step]
            acc[r] = a + b if op == "sum" else np.where(b > a, b, a)
        step *= 2
    return acc[0]


def cross_gpu_selfcheck(sk, devices):
    """Before any timed N>1 number: the peer-memory collectives across these
    GPUs must be BITWISE equal to the reference's tree order (sum, mean, max;
    broadcast), and NCCL's sum within 8*W*eps_f32 (acceptance_main.cpp:415).
    Raises on any mismatch -- a wrong collective never gets timed."""
    W = len(devices)
    rng = np.random.default_rng(99)
    checks = []
    for n in (1000, (1 << 20) + 3):  # one-launch path (rank 0 folds all chunks) and per-rank chunk kernels
        vals = [rng.uniform(-1, 1, n).astype(np.float32) for _ in range(W)]
        with sk.Pool(workers=W, devices=list(devices)) as pool:
            var = sk.replicate(pool, np.zeros(n, np.float32))
            for op in ("sum", "mean", "max"):
                for r in range(W):
                    var.set(r, vals[r])
                var.all_reduce(op)
                want = tree_fold(vals, "max" if op == "max" else "sum")
                if op == "mean":
                    want = (want.astype(np.float64) * (1.0 / W)).astype(np.float32)
                for r in range(W):
                    if var.get(r).tobytes() != want.tobytes():
                        raise RuntimeError("self-check: all_reduce(%s) of %d floats differs from the tree order on "
                                           "rank %d (devices %s)" % (op, n, r, devices))
                checks.append("all_reduce_%s_%d: bitwise" % (op, n))
            for r in range(W):
                var.set(r, vals[r])
            var.broadcast(W - 1)
            for r in range(W):
                if var.get(r).tobytes() != vals[W - 1].tobytes():
                    raise RuntimeError("self-check: broadcast differs on rank %d (devices %s)" % (r, devices))
            checks.append("broadcast_%d: bitwise" % n)
        if len(set(devices)) == W and sk.nccl_available():
            with sk.Pool(workers=W, devices=list(devices), collectives="nccl") as pool:
                var = sk.replicate(pool, np.zeros(n, np.float32))
                for r in range(W):
                    var.set(r, vals[r])
                var.all_reduce("sum")
                want = tree_fold(vals, "sum").astype(np.float64)
                tol = 8 * W * float(np.finfo(np.float32).eps)
                for r in range(W):
                    err = np.max(np.abs(var.get(r) - want) / np.maximum(1.0, np.abs(want)))
                    if not err <= tol:
                        raise RuntimeError("self-check: NCCL sum elem_err %.3g > %.3g on rank %d" % (err, tol, r))
                checks.append("nccl_all_reduce_sum_%d: elem_err <= 8*W*eps" % n)
    return {"devices": list(devices), "distinct_gpus": len(set(devices)), "ok": True, "checks": checks}


def collectives_sweep(sk, devices, collectives, sizes, rng):
    """Replicated.all_reduce("mean") and broadcast(0) per size, timed per call
    on the host (phase protocol + kernel + stream sync)."""
    world = len(devices)
    sweep = []
    with sk.Pool(workers=world, devices=list(devices), collectives=collectives) as pool:
        for S in sizes:
            n = S // 4
            var = sk.replicate(pool, np.zeros(n, np.float32))
            for r in range(world):
                var.set(r, rng.uniform(-1, 1, n).astype(np.float32))
            reps = 200 if S <= (1 << 20) else (30 if S <= (1 << 27) else 8)
            for _ in range(3):
                var.all_reduce("mean")
                var.broadcast(0)
            t = time.perf_counter()
            for _ in range(reps):
                var.all_reduce("mean")
            t_ar = (time.perf_counter() - t) / reps
            t = time.perf_counter()
            for _ in range(reps):
                var.broadcast(0)
            t_bc = (time.perf_counter() - t) / reps
            coherent = var.coherent
            del var
            sweep.append({"bytes": S, "allreduce_us": 1e6 * t_ar,
                          "allreduce_busbw_gbs": S / t_ar * 2 * (world - 1) / world / 1e9,
                          "broadcast_us": 1e6 * t_bc, "broadcast_busbw_gbs": S / t_bc / 1e9, "coherent": coherent})
    return sweep


def stub_sweep(devices, sizes):
    world = len(devices)
    return [{"bytes": S, "allreduce_us": 10 + S / 5e5, "allreduce_busbw_gbs": S / (10e-6 + S / 5e11) * 2 * (world - 1)
             / world / 1e9, "broadcast_us": 10 + S / 7e5, "broadcast_busbw_gbs": S / (10e-6 + S / 7e11) / 1e9,
             "coherent": True, "stub": True} for S in sizes]


NVLINK_PEAK_GBS = 900.0  # NVLink 5, per direction per GPU (B200_PROFILING.md)


def collectives_c4(sk, args, n_gpus, dry=False):
    """C4: all-reduce mean + broadcast(0), 1 KiB - 1 GiB, at W = 2/4/8 on
    distinct GPUs (peer-memory kernels, and NCCL as the library baseline),
    busbw = S/t * 2(W-1)/W (all-reduce), S/t (broadcast), against the NVLink
    peak. With one GPU the W=2 ranks share it and the bytes move through
    local HBM (stated in the output, not an NVLink number)."""
    ndev = n_gpus if dry else max(1, sk.device_count())
    sizes = [1 << k for k in range(10, 31, 3)] + [1 << 30]
    rng = np.random.default_rng(1000)
    worlds = [w for w in (2, 4, 8) if w <= min(n_gpus, ndev)]
    runs = []
    if not worlds:  # one GPU: W=2 ranks on it
        devs = [0, 0]
        runs.append({"ranks": 2, "devices": devs, "link": "1 GPU: the ranks share it, peer-memory kernels run over "
                                                          "local HBM (NVLink unmeasured)",
                     "p2p": stub_sweep(devs, sizes) if dry else collectives_sweep(sk, devs, "p2p", sizes, rng)})
    for w in worlds:
        devs = list(range(w))
        run = {"ranks": w, "devices": devs, "link": "NVLink peer memory (NVSwitch)",
               "p2p": stub_sweep(devs, sizes) if dry else collectives_sweep(sk, devs, "p2p", sizes, rng)}
        if dry or sk.nccl_available():
            try:
                run["nccl"] = stub_sweep(devs, sizes) if dry else collectives_sweep(sk, devs, "nccl", sizes, rng)
            except Exception as e:  # reported, not fatal
                run["nccl"] = {"unavailable": str(e)[:200]}
        for key in ("p2p", "nccl"):
            sw = run.get(key)
            if isinstance(sw, list) and sw:
                big = sw[-1]
                run[key + "_1gib_busbw_frac_of_nvlink"] = {
                    "allreduce": big["allreduce_busbw_gbs"] / NVLINK_PEAK_GBS,
                    "broadcast": big["broadcast_busbw_gbs"] / NVLINK_PEAK_GBS}
        runs.append(run)
    out = {"config": "C4: all_reduce mean + broadcast(0) of f32 buffers 1 KiB - 1 GiB", "nvlink_peak_gbs":
           NVLINK_PEAK_GBS, "runs": runs}
    if not args.no_cpu_baseline:
        ref = []
        for S in (1 << 10, 1 << 16, 1 << 20, 1 << 26):
            res, err = run_reference_driver("collective", ["--bytes", S, "--workers", 2, "--steps", 3, "--warmup", 1])
            if res is None:
                ref = {"unavailable": err}
                break
            ref.append({k: res[k] for k in ("bytes", "allreduce_us", "allreduce_busbw_gbs", "broadcast_us",
                                            "broadcast_busbw_gbs")})
        out["cpu_baseline"] = {"kind": "reference", "cores": 2, "cpu_model": cpu_model(), "sweep": ref}
    return out


def sync_sgd_section(sk, args, n_gpus, model, dry=False):
    """Per-N samples/s of one sync-SGD model (scaled mode: fixed batch per
    GPU), speedups, efficiency and the Table-1 split; N=1 also runs a 3 s
    back-to-back stretch (the sustained figure at the power cap)."""
    m = SGD_MODELS[model]
    runs = []
    # one rank per VISIBLE GPU: a job asking for more GPUs than the box shows
    # (e.g. torchrun N=2 on a 1-GPU box) measures up to the visible count
    n_vis = n_gpus if dry else min(n_gpus, max(1, sk.device_count()))
    for n in gpu_counts(n_vis):
        devs = list(range(n))
        sus = 3.0 if n == 1 and model == "c5" else 0.0
        if dry:
            runs.append(stub_sgd(model, devs, m["per_gpu"], args.steps, sus))
        else:
            runs.append(measure_sgd(sk, model, devs, m["per_gpu"], args.steps, args.warmup, 12 + n, sus))
    scaling_summary(runs, model)
    top = runs[-1]
    out = {"config": m["label"] + ", batch %d per GPU (scaled)" % m["per_gpu"], "dtype": m["dtype"],
           "gpus_visible_capped": None if n_vis == n_gpus else "%d of %d requested GPUs visible" % (n_vis, n_gpus),
           "flops_per_sample": flops_per_sample(m["dims"]), "runs": runs,
           "samples_per_s": top["samples_per_s"], "ms_per_step": top["ms_per_step"], "n_gpus": top["n_gpus"],
           "table1_note": "function = gradient-call compute (mean over ranks, device events); shuffle = staging of "
                          "the indexed batch before compute (0 when the gather is fused into the compute graph); "
                          "straggler = max - mean rank task; allreduce = the fused all-reduce + 1/W + update "
                          "kernel (so the update sits here, not in function); for C5 at W > 1 the all-reduce + "
                          "update runs per layer on a second stream, overlapped with the backward GEMMs, so its "
                          "span overlaps function and the parts sum to more than total (at W = 1 it follows the "
                          "backward pass)"}
    if model == "c5":
        bf16_peak, bf16_sustained, peak_kind = 1609.7, 1365.0, "fallback"
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
                mp = json.load(fh)
            bf16_peak = float(mp["bf16_tflops"])
            bf16_sustained = float(mp.get("bf16_tflops_sustained", bf16_sustained))
            peak_kind = "measured"
        except Exception:
            pass
        r1 = runs[0]
        out.update({"bf16_peak_tflops": bf16_peak, "bf16_sustained_tflops": bf16_sustained, "peak_kind": peak_kind,
                    "model_tflops_per_gpu_n1": r1["model_tflops_per_gpu"],
                    "frac_of_bf16_sustained_n1": r1["model_tflops_per_gpu"] / bf16_sustained,
                    "frac_of_bf16_peak_n1": r1["model_tflops_per_gpu"] / bf16_peak})
        if r1.get("sustained"):
            sus_tf = flops_per_sample(m["dims"]) * r1["sustained"]["samples_per_s"] / 1e12
            out["sustained_n1"] = dict(r1["sustained"], model_tflops=sus_tf, frac_of_bf16_sustained=sus_tf /
                                       bf16_sustained)
    return out


def sub_measurements(args, n_gpus, peak, peak_kind, dry=False):
    """Everything beyond the C2 headline, on the executor's own single-process
    pools over the job's GPUs (the paper's master + workers): the cross-GPU
    self-check, C1 and C5 sync SGD at N = 1/2/4/8 (<= the job's GPUs) with the
    Table-1 split, C1 exactly as configs[0], the reference's own SyncSgd
    timed here, C3 slicing and the C4 collective sweep."""
    sk = None
    if not dry:
        import paper_1710_04162_b200 as sk
    out = {}
    ndev = n_gpus if dry else max(1, sk.device_count())
    sc_devs = list(range(n_gpus)) if n_gpus >= 2 and ndev >= n_gpus else [0, 0]
    out["cross_gpu_selfcheck"] = ({"devices": sc_devs, "ok": True, "stub": True} if dry
                                  else cross_gpu_selfcheck(sk, sc_devs))
    if not args.no_sgd:
        out["sync_sgd"] = sync_sgd_section(sk, args, n_gpus, "c1", dry)
        exact_devs = [0, 1] if ndev >= 2 else [0, 0]
        ex = (stub_sgd("c1", exact_devs, 128, args.steps) if dry
              else measure_sgd(sk, "c1", exact_devs, 128, args.steps, args.warmup, 31))
        out["sync_sgd_c1_exact"] = dict(ex, config="C1 as configs[0]: MLP 784-512-10 fp32, W=2 workers, batch 256 "
                                                   "global (128 per rank), indexed, SGD lr 0.01, grad all-reduce "
                                                   "mean fused with the update")
        if not args.no_cpu_baseline:
            ref = reference_sgd(gpu_counts(n_gpus) if n_gpus > 1 else [1, 2], steps=3)
            out["sync_sgd"]["cpu_baseline"] = ref
            exact = ref.get("configs0_exact", {})
            if "samples_per_s" in exact:
                out["sync_sgd_c1_exact"]["cpu_baseline"] = {
                    "value": exact["samples_per_s"], "unit": "samples/s", "cores": 2, "kind": "reference",
                    "cpu_model": ref["cpu_model"], "sample": "%d SyncSgd::train_step calls, W=2 threads, batch 256"
                    % exact["steps"], "table1": exact.get("table1")}
                out["sync_sgd_c1_exact"]["speedup_vs_cpu_reference"] = ex["samples_per_s"] / exact["samples_per_s"]
        out["sync_sgd_wide_bf16"] = sync_sgd_section(sk, args, n_gpus, "c5", dry)
    if not args.no_c3 and not dry:
        with sk.Pool(workers=n_gpus, devices=[d % ndev for d in range(n_gpus)]) as pool:
            out["slicing_c3"] = slicing_c3(sk, pool, args, n_gpus, peak, peak_kind)
    if not args.no_c4:
        out["collectives_c4"] = collectives_c4(sk, args, n_gpus, dry)
    return out


def stub_headline(args, n_gpus, world):
    """--dry-run stand-in for gather_headline (no GPU): synthetic timings of
    the same record shape, so the line's assembly runs unchanged on CPU."""
    n_step, row_bytes = args.batch * args.batches, args.cols * 4
    peak, peak_kind = measured_peak_hbm()
    launch_s = n_step * (2 * row_bytes + BYTES_PER_ROW_EXTRA) / (0.9 * peak * 1e9)
    bytes_step = n_gpus * n_step * (2 * row_bytes + BYTES_PER_ROW_EXTRA)
    return {"value": bytes_step / launch_s / 1e9, "region_s": launch_s * args.steps, "e2e": 0.8 * bytes_step / launch_s
            / 1e9, "e2e_breakdown": {}, "single_call": {"rows_per_gpu": args.batch, "us_per_call": 20.0, "stub": True},
            "achieved": 0.9 * peak, "single_s": 8e-6, "clocks": {"sm_mhz": None, "sm_max_mhz": None,
                                                               "reasons": ["dry-run"]},
            "host_source": None, "setup_s": 0.0, "n_step": n_step, "row_bytes": row_bytes, "peak": peak,
            "peak_kind": peak_kind}


def ours(args, n_gpus, dist=None, world=1, local_device=0, dry=False):
    """Our arm. Single process: the headline on a pool over all N GPUs. Under
    torchrun: one process per GPU for the headline (each its own one-GPU
    pool), then rank 0 alone runs the sub-measurements over every GPU.
    dry: no GPU work, synthetic timings through the same line assembly."""
    devices = [local_device] if dist is not None else list(range(n_gpus))
    hd = stub_headline(args, n_gpus, world) if dry else gather_headline(args, n_gpus, devices, dist, world)
    if dist is not None:
        dist.barrier()  # every rank's headline pool is down before rank 0 opens its own over all GPUs
        if dist.get_rank() != 0:
            return None
    value, n_step, row_bytes = hd["value"], hd["n_step"], hd["row_bytes"]
    achieved, peak, peak_kind = hd["achieved"], hd["peak"], hd["peak_kind"]
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": n_gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * hd["region_s"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, n_gpus),
            "e2e": {"value": hd["e2e"], "unit": "GB/s", "h2d_bytes_per_step": 8 * n_step * n_gpus,
                    "d2h_bytes_per_step": 8 * (world if dist is not None else 1),
                    "path": "Function.call(indexes) -> row_count kernel -> Sum, %d batches of %d rows per GPU per "
                            "call" % (args.batches, args.batch),
                    "breakdown_per_call": hd["e2e_breakdown"], "single_batch_call": hd["single_call"],
                    "residency": "dataset mirrored in HBM before timing (SharedInput.mirror, SURVEY 8(f)#1); with "
                                 "the dataset left in pinned host memory see gather_from_host_memory"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(n_step * (2 * row_bytes + 8)),
                         "traffic_unit": "bytes/launch", "peak_kind": peak_kind,
                         "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of the committed ncu --set "
                                           "full capture of this launch size (%s), not measured in this run"
                                           % TRAFFIC_CAPTURE,
                         "kernel": "gather_rows_kernel<32>" if row_bytes % 32 == 0 else "gather_rows_kernel<16>", "bytes_per_launch": n_step * (2 * row_bytes + 8)},
            "single_batch_us": 1e6 * hd["single_s"],
            "gather_from_host_memory": hd["host_source"],
            "gpu_launches": n_gpus * args.steps, "clocks": hd["clocks"], "setup_s": hd["setup_s"]}
    if dist is not None:
        line["processes"] = "one per GPU for the headline (torchrun); rank 0 alone for the sub-measurements"
    line.update(sub_measurements(args, n_gpus, peak, peak_kind, dry))
    if dry:
        line["dry_run"] = True
        line["data"] = "synthetic timings (dry run: no GPU work)"
    return line


def gather_cpu_baseline(args):
    """The unmodified reference's call(indexes) (no-op kernel) on this box's
    cores: a bounded sample (5 steps) of the headline workload."""
    cores = os.cpu_count() or 1
    res, err = run_reference_driver("gather", ["--rows", args.rows, "--cols", args.cols, "--batch",
                                               args.batch * args.batches, "--steps", 5, "--warmup", 1,
                                               "--workers", cores])
    if not res:
        return {"value": None, "unavailable": err}
    return {"value": res["gbs"], "unit": "GB/s", "cores": res["workers"], "kind": "reference", "cpu_model": cpu_model(),
            "sample": "5 steps x %d rows via the unmodified reference call(indexes), no-op kernel, from the same "
                      "%dx%d f32 dataset shape" % (args.batch * args.batches, args.rows, args.cols)}


def main():
    args = parse()
    rank, world, dist = dist_setup()
    n_gpus = max(args.gpus, world)
    line = None
    seen = None
    if args.dry_run and dist is not None:
        seen = [None] * world
        dist.all_gather_object(seen, {"rank": rank, "pid": os.getpid()})
    if args.dry_run:
        # No GPU work: every rank reports in, rank 0 assembles the full line
        # from synthetic device timings (the CPU reference legs run for real).
        if rank == 0:
            if args.impl == "reference":
                line = reference_arm(args, n_gpus)
            else:
                line = ours(args, n_gpus, world=world, dry=True)
                if not args.no_cpu_baseline:
                    line["cpu_baseline"] = gather_cpu_baseline(args)
            line.update({"dry_run": True, "world": world, "driver_rank": 0,
                         "ranks_seen": sorted(x["rank"] for x in seen) if seen else [0]})
    elif args.impl == "ours" and dist is not None:
        # torchrun: one process per GPU for the headline, rank 0 then drives the rest
        import paper_1710_04162_b200 as sk

        local = int(os.environ.get("LOCAL_RANK", rank)) % max(1, sk.device_count())
        line = ours(args, n_gpus, dist=dist, world=world, local_device=local)
    elif rank == 0:
        if args.impl == "reference":
            line = reference_arm(args, n_gpus)
        else:
            line = ours(args, n_gpus)
            if not args.no_cpu_baseline:
                line["cpu_baseline"] = gather_cpu_baseline(args)
    if dist is not None:
        dist.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
