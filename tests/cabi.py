"""Minimal ctypes driver of libsynk_cuda.so for kernel-level parity tests.

Device memory, copies and kernels all go through the C-ABI itself (no torch),
so these tests exercise exactly the entry points a reference-side FFI would
bind."""

import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(ROOT, "paper_1710_04162_b200", "_lib", "libsynk_cuda.so")

F32, F64 = 1, 2
OPS = {"sum": 0, "mean": 1, "max": 2, "min": 3, "prod": 4}
RULES = {"sgd": 0, "momentum": 1, "rmsprop": 2, "adam": 3}
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64


def lib():
    if not hasattr(lib, "h"):
        h = ctypes.CDLL(LIB_PATH)
        h.synk_last_error.restype = ctypes.c_char_p
        h.synk_dev_stream.restype = _vp
        lib.h = h
    return lib.h


def check(rc, what=""):
    if rc != 0:
        raise RuntimeError("%s failed (%d): %s" % (what, rc, lib().synk_last_error().decode()))


def dt(a):
    return F32 if np.dtype(a) == np.float32 else F64


class Ranks:
    """`world` rank contexts on the given devices (default: all on GPU 0)."""

    def __init__(self, world=1, devices=None):
        devices = devices or [0] * world
        self.world = world
        self.h = (_vp * world)()
        ids = (ctypes.c_int * world)(*devices)
        check(lib().synk_open(world, ids, self.h), "synk_open")
        self.bufs = []

    def __getitem__(self, r):
        return _vp(self.h[r])

    def close(self):
        for r in range(self.world):
            lib().synk_sync(self[r])
        for ptr, r in self.bufs:
            lib().synk_free(self[r], _vp(ptr))
        for r in range(self.world):
            lib().synk_sync(self[r])
            lib().synk_close(self[r])

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- memory ----
    def alloc(self, nbytes, rank=0):
        p = _vp()
        check(lib().synk_alloc(self[rank], _u64(max(nbytes, 16)), ctypes.byref(p)), "synk_alloc")
        check(lib().synk_sync(self[rank]), "sync")
        self.bufs.append((p.value, rank))
        return p.value

    def upload(self, arr, rank=0):
        arr = np.ascontiguousarray(arr)
        p = self.alloc(arr.nbytes, rank)
        if arr.nbytes:
            check(lib().synk_copy(self[rank], _vp(p), arr.ctypes.data_as(_vp), _u64(arr.nbytes)), "H2D")
        check(lib().synk_sync(self[rank]), "sync")
        return p

    def download(self, ptr, shape, dtype, rank=0):
        out = np.empty(shape, dtype)
        if out.nbytes:
            check(lib().synk_copy(self[rank], out.ctypes.data_as(_vp), _vp(ptr), _u64(out.nbytes)), "D2H")
        check(lib().synk_sync(self[rank]), "sync")
        return out

    def sync(self, rank=0):
        return lib().synk_sync(self[rank])


def ptr_array(ptrs):
    return (_vp * len(ptrs))(*ptrs)
