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


def ncu_traffic(bytes_per_launch, path="profiles/r01_gather_ncu_full_raw.csv"):
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
                                  "sample": "%d steps x %d rows gathered through call(indexes) with a no-op kernel "
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
            "value": res["gbs"], "unit": "GB/s", "cores": res["workers"], "kind": "reference",
            "sample": "2 calls over %dx%d f32 (explicit scatter input), num_slices=%d, Sum+Max+Gather" % (
                sample, cols, slices)}
    return out


def collectives_c4(sk, args, n_gpus):
    """C4: Replicated.all_reduce("mean") and broadcast(0) of f32 buffers from
    1 KiB to 1 GiB, timed per call on the host (phase protocol + peer-memory
    kernel + stream sync). busbw = S/t * 2(W-1)/W (all-reduce), S/t (broadcast).
    With one GPU the W=2 ranks share it, so the peer-memory kernels move the
    bytes through local HBM instead of NVLink (stated in the output)."""
    world = n_gpus if n_gpus >= 2 else 2
    ndev = max(1, sk.device_count())
    devices = [d % ndev for d in range(n_gpus)] if n_gpus >= 2 else [0, 0]
    sizes = [1 << k for k in range(10, 31, 3)] + [1 << 30]
    rng = np.random.default_rng(1000)

    def sweep_with(collectives):
        sweep = []
        with sk.Pool(workers=world, devices=devices, collectives=collectives) as pool:
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
                              "broadcast_us": 1e6 * t_bc, "broadcast_busbw_gbs": S / t_bc / 1e9,
                              "coherent": coherent})
        return sweep

    sweep = sweep_with("p2p")
    out = {"config": "C4: all_reduce mean + broadcast(0) of f32 buffers 1 KiB - 1 GiB, W=%d ranks" % world,
           "ranks": world, "devices": devices,
           "link": "NVLink peer memory" if len(set(devices)) >= 2 else "1 GPU: the ranks share it, peer-memory "
                                                                         "kernels run over local HBM (NVLink unmeasured)",
           "sweep": sweep}
    # Library baseline on distinct GPUs: the same sweep through NCCL (busbw vs
    # the NVLink peak, next to the peer-memory kernels above).
    if len(set(devices)) >= 2 and sk.nccl_available():
        try:
            out["nccl_sweep"] = sweep_with("nccl")
        except Exception as e:  # reported, not fatal
            out["nccl_sweep"] = {"unavailable": str(e)[:200]}
    if not args.no_cpu_baseline:
        ref = []
        for S in (1 << 10, 1 << 16, 1 << 20, 1 << 26):
            res, err = run_reference_driver("collective", ["--bytes", S, "--workers", world, "--steps", 3,
                                                           "--warmup", 1])
            if res is None:
                ref = {"unavailable": err}
                break
            ref.append({k: res[k] for k in ("bytes", "allreduce_us", "allreduce_busbw_gbs", "broadcast_us",
                                            "broadcast_busbw_gbs")})
        out["cpu_baseline"] = {"kind": "reference", "cores": world, "sweep": ref}
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

    pool.shutdown()
    del arr
    return {"value": value, "region_s": region_s, "e2e": e2e, "e2e_breakdown": e2e_breakdown, "achieved": achieved,
            "single_s": single_s, "clocks": clocks.summary(), "host_source": host_src,
            "setup_s": setup_s, "n_step": n_step, "row_bytes": row_bytes, "peak": peak, "peak_kind": peak_kind}


def sub_measurements(args, n_gpus, peak, peak_kind):
    """C1, C5 (sync SGD through Trainer), C3 (slicing), C4 (collectives): the
    executor's own single-process pool over the job's GPUs (the paper's
    master + workers; collectives are peer-memory kernels across them)."""
    import paper_1710_04162_b200 as sk

    ndev = max(1, sk.device_count())
    pool = sk.Pool(workers=n_gpus, devices=[d % ndev for d in range(n_gpus)])
    rng = np.random.default_rng(12)
    total_steps = args.warmup + args.steps
    # ---- sync SGD (C1) sub-measurement ------------------------------------------------
    sgd = None
    if not args.no_sgd:
        cfg = sk.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
        x, y = sk.mlp_make_dataset(65536, cfg, seed=2, dtype="f32")
        sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
        sx.mirror(pool)
        sy.mirror(pool)
        block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
        g = sk.mlp_grad_function(pool, block)
        sk.distribute(pool)
        tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
        # Latency-bound steps: a longer untimed warm-up lets the per-rank CUDA-graph
        # cache settle on the recycled batch buffers (captures cost ~0.5 ms each).
        warm1 = max(args.warmup, 30)
        sel = [pinned_indexes(sk, rng, 65536, 256 * n_gpus) for _ in range(warm1 + args.steps)]
        for s in range(warm1):
            tr.train_step(g, [sx, sy], indexes=sel[s])
        t0 = time.perf_counter()
        for s in range(warm1, warm1 + args.steps):
            loss = tr.train_step(g, [sx, sy], indexes=sel[s])
        dt = time.perf_counter() - t0
        rep = tr.last_report
        sgd = {"config": "C1: MLP 784-512-10 fp32, batch 256 per GPU (scaled), indexed from a 65536-row SharedInput "
                         "(HBM mirror), SGD lr 0.01, grad all-reduce mean fused with the update",
               "samples_per_s": 256 * n_gpus * args.steps / dt, "ms_per_step": 1e3 * dt / args.steps,
               "allreduce_ms_last": 1e3 * rep["allreduce_s"], "loss_last": loss, "coherent": block.params.coherent}

    # ---- wide MLP (C5) sync SGD on tcgen05 bf16 -------------------------------------------
    sgd5 = None
    if not args.no_sgd:
        dims = [2048, 4096, 4096, 100]
        cfg = sk.MlpConfig(in_dim=dims[0], width=dims[1], out_dim=dims[-1], layers=3, seed=1)
        x, y = sk.mlp_make_dataset(16384, cfg, seed=2, dtype="f32")
        sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
        sx.mirror(pool)
        sy.mirror(pool)
        block = sk.ParamBlock.create(pool, sk.mlp_init_params(cfg, "f32"))
        g = sk.mlp_grad_function(pool, block, compute="bf16")
        sk.distribute(pool)
        tr = sk.Trainer(pool, block, sk.SgdRule(), lr=0.01)
        per_gpu = 8192
        sel = [pinned_indexes(sk, rng, 16384, per_gpu * n_gpus) for _ in range(total_steps)]
        for s in range(args.warmup):
            tr.train_step(g, [sx, sy], indexes=sel[s])
        t0 = time.perf_counter()
        for s in range(args.warmup, total_steps):
            loss = tr.train_step(g, [sx, sy], indexes=sel[s])
        dt = time.perf_counter() - t0
        flops_per_sample = 6 * sum(a * b for a, b in zip(dims[:-1], dims[1:])) - 2 * dims[0] * dims[1]
        # Roofline denominators (MEASURED_PEAKS.json): the sustained bf16 figure
        # applies to a long back-to-back GEMM stream like this step (power
        # management lowers the clocks under sustained tensor load); burst kept too.
        bf16_peak, bf16_sustained, peak_kind = 1609.7, 1365.0, "fallback"
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
                mp = json.load(fh)
            bf16_peak = float(mp["bf16_tflops"])
            bf16_sustained = float(mp.get("bf16_tflops_sustained", bf16_sustained))
            peak_kind = "measured"
        except Exception:
            pass
        tflops = flops_per_sample * per_gpu * n_gpus * args.steps / dt / 1e12 / n_gpus
        sgd5 = {"config": "C5 (R1): MLP 2048-4096-4096-100 (25,583,716 params, fp32 master), bf16 tcgen05 GEMMs, "
                          "batch %d per GPU indexed from a 16384-row HBM mirror, SGD lr 0.01, fused grad "
                          "all-reduce mean + update" % per_gpu,
                "n_params": int(block.length), "samples_per_s": per_gpu * n_gpus * args.steps / dt,
                "ms_per_step": 1e3 * dt / args.steps, "model_tflops_per_gpu": tflops,
                "frac_of_bf16_peak": tflops / bf16_peak, "frac_of_bf16_sustained": tflops / bf16_sustained,
                "bf16_peak_tflops": bf16_peak, "bf16_sustained_tflops": bf16_sustained, "peak_kind": peak_kind,
                "loss_last": loss, "coherent": block.params.coherent}

    # ---- slicing + aggregation (C3) sub-measurement ----------------------------------
    c3 = None
    if not args.no_c3:
        c3 = slicing_c3(sk, pool, args, n_gpus, peak, peak_kind)

    pool.shutdown()
    # ---- C1 exactly as BASELINE configs[0] states it: W=2 workers, batch 256
    # global (128 per rank), the CPU reference's own configuration -------------
    sgd_exact = None
    if not args.no_sgd:
        ndev = max(1, sk.device_count())
        devices = [0, 1 % ndev]
        with sk.Pool(workers=2, devices=devices) as pool2:
            cfg = sk.MlpConfig(in_dim=784, width=512, out_dim=10, layers=2, seed=1)
            x, y = sk.mlp_make_dataset(65536, cfg, seed=2, dtype="f32")
            sx, sy = sk.SharedInput.from_array(x), sk.SharedInput.from_array(y)
            sx.mirror(pool2)
            sy.mirror(pool2)
            block = sk.ParamBlock.create(pool2, sk.mlp_init_params(cfg, "f32"))
            g = sk.mlp_grad_function(pool2, block)
            sk.distribute(pool2)
            tr = sk.Trainer(pool2, block, sk.SgdRule(), lr=0.01)
            warm1 = max(args.warmup, 30)
            sel = [pinned_indexes(sk, rng, 65536, 256) for _ in range(warm1 + args.steps)]
            for s in range(warm1):
                tr.train_step(g, [sx, sy], indexes=sel[s])
            t0 = time.perf_counter()
            for s in range(warm1, warm1 + args.steps):
                loss = tr.train_step(g, [sx, sy], indexes=sel[s])
            dt = time.perf_counter() - t0
            sgd_exact = {"config": "C1 as configs[0]: MLP 784-512-10 fp32, W=2 workers, batch 256 global (128 per "
                                   "rank), indexed, SGD lr 0.01, grad all-reduce mean fused with the update",
                         "devices": devices, "samples_per_s": 256 * args.steps / dt,
                         "ms_per_step": 1e3 * dt / args.steps, "loss_last": loss, "coherent": block.params.coherent,
                         "reference_cpu_samples_per_s": 2048,
                         "reference_note": "BASELINE/SURVEY probe of the unmodified reference, W=2, 8-core box"}
    # ---- shared-variable sync sweep (C4): its own pool (one live pool per process) ----
    c4 = None
    if not args.no_c4:
        c4 = collectives_c4(sk, args, n_gpus)
    out = {}
    if sgd:
        out["sync_sgd"] = sgd
    if sgd_exact:
        out["sync_sgd_c1_exact"] = sgd_exact
    if sgd5:
        out["sync_sgd_wide_bf16"] = sgd5
    if c3:
        out["slicing_c3"] = c3
    if c4:
        out["collectives_c4"] = c4
    return out


def ours(args, n_gpus, dist=None, world=1, local_device=0):
    """Our arm. Single process: the headline on a pool over all N GPUs. Under
    torchrun: one process per GPU for the headline (each its own one-GPU
    pool), then rank 0 alone runs the sub-measurements over every GPU."""
    devices = [local_device] if dist is not None else list(range(n_gpus))
    hd = gather_headline(args, n_gpus, devices, dist, world)
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
                    "path": "Function.call(indexes) -> row_count kernel -> Sum",
                    "breakdown_per_call": hd["e2e_breakdown"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(n_step * (2 * row_bytes + 8)),
                         "traffic_unit": "bytes/launch", "peak_kind": peak_kind,
                         "kernel": "gather_rows_kernel<32>" if row_bytes % 32 == 0 else "gather_rows_kernel<16>", "bytes_per_launch": n_step * (2 * row_bytes + 8)},
            "single_batch_us": 1e6 * hd["single_s"],
            "gather_from_host_memory": hd["host_source"],
            "gpu_launches": n_gpus * args.steps, "clocks": hd["clocks"], "setup_s": hd["setup_s"]}
    if dist is not None:
        line["processes"] = "one per GPU for the headline (torchrun); rank 0 alone for the sub-measurements"
    line.update(sub_measurements(args, n_gpus, peak, peak_kind))
    return line


def main():
    args = parse()
    rank, world, dist = dist_setup()
    n_gpus = max(args.gpus, world)
    line = None
    if args.dry_run:
        # Coordination only: every rank reports in, rank 0 alone prints.
        if dist is not None:
            import torch

            seen = [None] * world
            dist.all_gather_object(seen, {"rank": rank, "pid": os.getpid()})
        else:
            seen = [{"rank": 0, "pid": os.getpid()}]
        line = {"metric": METRIC, "dry_run": True, "n_gpus": n_gpus, "world": world,
                "ranks_seen": sorted(s["rank"] for s in seen), "driver_rank": 0}
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
                cores = os.cpu_count() or 1
                res, err = run_reference_driver("gather", ["--rows", args.rows, "--cols", args.cols, "--batch",
                                                           args.batch * args.batches, "--steps", 5, "--warmup", 1,
                                                           "--workers", cores])
                line["cpu_baseline"] = (
                    {"value": res["gbs"], "unit": "GB/s", "cores": res["workers"], "kind": "reference",
                     "sample": "5 steps x %d rows via the unmodified reference call(indexes), no-op kernel, from the "
                               "same %dx%d f32 dataset shape" % (args.batch * args.batches, args.rows, args.cols)}
                    if res else {"value": None, "unavailable": err})
    if dist is not None:
        dist.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
