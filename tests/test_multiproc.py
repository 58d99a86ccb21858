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
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--impl", impl, "--dry-run"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["world"] == 2 and rec["n_gpus"] == 2 and rec["ranks_seen"] == [0, 1]


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
