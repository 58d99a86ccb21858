"""CPU coverage of the N>1 path (no GPU).

1. bench.py under torchrun with world_size 2 (gloo): every rank joins, exactly
   one JSON line (rank 0) is printed, all ranks exit 0 — for both arms.
2. The collective work split of the device layer (synk_chunk_range, the same
   function the peer-memory kernels use) tiles [0, n) exactly, in rank order,
   with 16-element-aligned boundaries, for every world size the executor
   accepts — so W ranks never touch the same element and never miss one.
3. The rank-order fold semantics the master applies across ranks match the
   reference (oracle) for uneven shards: partition_rows + weighted left fold.
"""

import ctypes
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("impl", ["ours", "reference"])
def test_bench_torchrun_world2_gloo(impl):
    """bench.py under torchrun, world 2 (gloo), --dry-run: synthetic device
    timings, the CPU reference legs for real (small dataset), and the whole
    line assembled as on an N=2 box: per-N sync-SGD runs with speedups and the
    Table-1 split, the reference's own SyncSgd timed here, C4 at W=2 through
    peer memory and NCCL, the cross-GPU self-check record."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--impl", impl, "--dry-run",
           "--rows", "100000", "--batches", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["world"] == 2 and rec["n_gpus"] == 2 and rec["ranks_seen"] == [0, 1]
    if impl == "reference":
        assert rec["impl"] == "reference" and rec["value"] > 0 and rec["e2e"]["h2d_bytes_per_step"] == 0
        return
    for key in ("value", "e2e", "roofline", "cpu_baseline", "clocks", "gpu_launches"):
        assert key in rec, key
    assert rec["cpu_baseline"]["value"] > 0 and rec["cpu_baseline"]["cpu_model"]
    for sec in ("sync_sgd", "sync_sgd_wide_bf16"):
        runs = rec[sec]["runs"]
        assert [r["n_gpus"] for r in runs] == [1, 2]
        for r in runs:
            assert r["speedup_vs_1"] > 0 and r["efficiency_vs_linear"] > 0
            assert set(r["table1_per_step_us"]) == {"function", "shuffle", "straggler", "allreduce", "total"}
    ref = rec["sync_sgd"]["cpu_baseline"]
    assert ref["configs0_exact"]["samples_per_s"] > 0 and ref["configs0_exact"]["workers"] == 2
    assert [r["workers"] for r in ref["scaled"]] == [1, 2]
    assert set(ref["scaled"][1]["table1"]) == {"total_s", "function_s", "shuffle_s", "straggler_s", "allreduce_s"}
    assert rec["sync_sgd_c1_exact"]["cpu_baseline"]["value"] > 0
    c4 = rec["collectives_c4"]["runs"]
    assert c4[0]["ranks"] == 2 and c4[0]["devices"] == [0, 1] and "nccl" in c4[0]
    assert "p2p_1gib_busbw_frac_of_nvlink" in c4[0]
    assert rec["cross_gpu_selfcheck"]["devices"] == [0, 1]


def test_tree_fold_matches_oracle(oracle):
    """bench.py's self-check fold (the numpy binomial tree it compares the
    cross-GPU collectives with) is the oracle's tree fold, bit for bit."""
    sys.path.insert(0, ROOT)
    import bench

    rng = np.random.default_rng(4)
    for world in (2, 3, 5, 8):
        vals = [rng.uniform(-1, 1, 1001).astype(np.float32) for _ in range(world)]
        vals[0][3] = np.nan
        vals[-1][7] = -0.0
        for op in ("sum", "max"):
            got = bench.tree_fold(vals, op)
            want = oracle.tree_fold(vals, op)
            assert got.tobytes() == np.asarray(want, np.float32).tobytes(), (world, op)


def test_chunk_ranges_tile_exactly():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1710_04162_b200", "_lib", "libsynk_cuda.so"))
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    for world in (1, 2, 3, 4, 5, 7, 8, 16, 64):
        for n in (0, 1, 15, 16, 17, 1000, 407050, 25583716):
            covered = 0
            prev_hi = 0
            for r in range(world):
                assert lib.synk_chunk_range(ctypes.c_uint64(n), world, r, ctypes.byref(lo), ctypes.byref(hi)) == 0
                assert lo.value == prev_hi or lo.value == hi.value  # contiguous, in rank order
                if lo.value < n:
                    assert lo.value % 16 == 0
                covered += hi.value - lo.value
                prev_hi = max(prev_hi, hi.value)
            assert covered == n and prev_hi == n
    assert lib.synk_chunk_range(ctypes.c_uint64(10), 2, 2, ctypes.byref(lo), ctypes.byref(hi)) != 0


def test_uneven_shard_rank_fold(oracle):
    # function.cpp:515-527: rank outputs folded left in rank order, Mean weighted
    # by effective rows; partition gives the first n % W ranks one extra row.
    rng = np.random.default_rng(3)
    data = rng.uniform(-1, 1, (10, 4))
    parts = oracle.partition_rows(10, 4)
    assert [b - a for a, b in parts] == [3, 3, 2, 2]
    shard_means = [data[a:b].mean(axis=0) for a, b in parts]
    folded = oracle.left_fold(shard_means, "mean", [b - a for a, b in parts])
    np.testing.assert_allclose(folded, data.mean(axis=0), rtol=0, atol=1e-15)
