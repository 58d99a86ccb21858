"""ctypes/numpy front of the C restatement (oracle/synk_oracle.c).

TEST INFRASTRUCTURE ONLY — the parity checker for tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg. The product (paper_1710_04162_b200) never
imports this module.

Also exposes the unmodified reference build (oracle/_ref/_synkpar_ref, built
from /root/reference by oracle/Makefile) when it is present.
"""

import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
_LIB = os.path.join(REF_DIR, "libsynk_oracle.so")

F32, F64 = 1, 2
OPS = {"sum": 0, "mean": 1, "max": 2, "min": 3, "prod": 4, "gather": 5}
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p


def build(with_reference=None):
    """Compile the restatement (and, when /root/reference exists, the reference)."""
    targets = ["restatement"]
    if with_reference is None:
        with_reference = os.path.isdir("/root/reference/proj")
    if with_reference:
        targets.append("ref")
    subprocess.run(["make", "-s", "-j8", *targets], cwd=HERE, check=True)


def _lib():
    if not hasattr(_lib, "h"):
        if not os.path.exists(_LIB):
            build(with_reference=False)
        h = ctypes.CDLL(_LIB)
        h.so_gather_rows.restype = ctypes.c_int
        h.so_combine.restype = ctypes.c_int
        h.so_weighted_mean.restype = ctypes.c_int
        h.so_tree_fold.restype = ctypes.c_int
        h.so_left_fold.restype = ctypes.c_int
        h.so_mlp_loss_grad.restype = ctypes.c_int
        _lib.h = h
    return _lib.h


def _dt(a):
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.float64:
        return F64
    raise TypeError("oracle handles f32/f64 only, got %s" % a.dtype)


def _p(a):
    return a.ctypes.data_as(_vp)


def partition_rows(n, parts):
    s = np.zeros(parts, np.uint64)
    e = np.zeros(parts, np.uint64)
    _lib().so_partition_rows(ctypes.c_uint64(n), ctypes.c_uint64(parts), s.ctypes.data_as(_u64p), e.ctypes.data_as(_u64p))
    return [(int(a), int(b)) for a, b in zip(s, e)]


def gather_rows(src, idx):
    src = np.ascontiguousarray(src)
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.empty((len(idx),) + src.shape[1:], src.dtype)
    row_bytes = src.dtype.itemsize * int(np.prod(src.shape[1:], dtype=np.int64))
    rc = _lib().so_gather_rows(_p(src), ctypes.c_uint64(src.shape[0]), ctypes.c_uint64(row_bytes),
                               idx.ctypes.data_as(_u64p), ctypes.c_uint64(len(idx)), _p(out))
    if rc != 0:
        raise IndexError("gather_rows: index out of range")
    return out


def combine(acc, other, op):
    acc = np.array(acc, copy=True)
    other = np.ascontiguousarray(other, dtype=acc.dtype)
    rc = _lib().so_combine(_dt(acc), OPS[op], _p(acc), _p(other), ctypes.c_uint64(acc.size))
    if rc != 0:
        raise ValueError("combine: %s is not elementwise" % op)
    return acc


def weighted_mean(acc, wa, other, wb):
    acc = np.array(acc, copy=True)
    other = np.ascontiguousarray(other, dtype=acc.dtype)
    rc = _lib().so_weighted_mean(_dt(acc), _p(acc), ctypes.c_double(wa), _p(other), ctypes.c_double(wb),
                                 ctypes.c_uint64(acc.size))
    if rc != 0:
        raise ValueError("weighted_mean: zero weights")
    return acc


def scale(buf, factor):
    buf = np.array(buf, copy=True)
    _lib().so_scale(_dt(buf), _p(buf), ctypes.c_double(factor), ctypes.c_uint64(buf.size))
    return buf


def tree_fold(parts, op):
    parts = [np.ascontiguousarray(p) for p in parts]
    out = np.empty_like(parts[0])
    arr = (_vp * len(parts))(*[p.ctypes.data for p in parts])
    rc = _lib().so_tree_fold(_dt(out), OPS[op], arr, ctypes.c_uint64(len(parts)), ctypes.c_uint64(out.size), _p(out))
    if rc != 0:
        raise ValueError("tree_fold failed")
    return out


def left_fold(parts, op, weights=None):
    parts = [np.ascontiguousarray(p) for p in parts]
    out = np.empty_like(parts[0])
    arr = (_vp * len(parts))(*[p.ctypes.data for p in parts])
    w = None if weights is None else np.ascontiguousarray(weights, np.uint64)
    rc = _lib().so_left_fold(_dt(out), OPS[op], arr, None if w is None else w.ctypes.data_as(_u64p),
                             ctypes.c_uint64(len(parts)), ctypes.c_uint64(out.size), _p(out))
    if rc != 0:
        raise ValueError("left_fold failed")
    return out


def sgd(p, g, lr):
    p = np.array(p, copy=True)
    _lib().so_sgd(_dt(p), _p(p), _p(np.ascontiguousarray(g, p.dtype)), ctypes.c_double(lr), ctypes.c_uint64(p.size))
    return p


def momentum(p, v, g, mu, lr):
    p, v = np.array(p, copy=True), np.array(v, copy=True)
    _lib().so_momentum(_dt(p), _p(p), _p(v), _p(np.ascontiguousarray(g, p.dtype)), ctypes.c_double(mu),
                       ctypes.c_double(lr), ctypes.c_uint64(p.size))
    return p, v


def rmsprop(p, a, g, rho, eps, lr):
    p, a = np.array(p, copy=True), np.array(a, copy=True)
    _lib().so_rmsprop(_dt(p), _p(p), _p(a), _p(np.ascontiguousarray(g, p.dtype)), ctypes.c_double(rho),
                      ctypes.c_double(eps), ctypes.c_double(lr), ctypes.c_uint64(p.size))
    return p, a


def adam(p, m, v, g, b1, b2, eps, lr, t):
    p, m, v = (np.array(x, copy=True) for x in (p, m, v))
    _lib().so_adam(_dt(p), _p(p), _p(m), _p(v), _p(np.ascontiguousarray(g, p.dtype)), ctypes.c_double(b1),
                   ctypes.c_double(b2), ctypes.c_double(eps), ctypes.c_double(lr), ctypes.c_uint64(t),
                   ctypes.c_uint64(p.size))
    return p, m, v


def mlp_loss_grad(params, dims, x, y):
    """Flat params [W0 b0 W1 b1 ...]; returns (f64 loss, flat grad in params' dtype)."""
    params = np.ascontiguousarray(params)
    x = np.ascontiguousarray(x, params.dtype)
    y = np.ascontiguousarray(y, params.dtype)
    d = np.ascontiguousarray(dims, np.uint64)
    grad = np.empty_like(params)
    loss = ctypes.c_double(0.0)
    rc = _lib().so_mlp_loss_grad(_dt(params), d.ctypes.data_as(_u64p), ctypes.c_uint64(len(dims) - 1), _p(params),
                                 _p(x), _p(y), ctypes.c_uint64(x.shape[0]), ctypes.byref(loss), _p(grad))
    if rc != 0:
        raise ValueError("mlp_loss_grad: empty batch")
    return loss.value, grad


def column_fold(x, kind):
    """kind: 'sum' | 'max' | 'min' (acceptance_main.cpp:86-133 kernels)."""
    x = np.ascontiguousarray(x)
    rows, cols = x.shape[0], int(np.prod(x.shape[1:], dtype=np.int64))
    out = np.empty(cols, x.dtype)
    _lib().so_column_fold(_dt(x), {"sum": 0, "max": 1, "min": 2}[kind], _p(x), ctypes.c_uint64(rows),
                          ctypes.c_uint64(cols), _p(out))
    return out


def fill_uniform(n, seed, first=0, dtype=np.float32):
    """Synthetic U[-1,1) stream (synk_fill_uniform's formula)."""
    out = np.empty(n, dtype)
    _lib().so_fill_uniform(_dt(out), _p(out), ctypes.c_uint64(n), ctypes.c_uint64(seed), ctypes.c_uint64(first))
    return out


def elem_err(a, b):
    """support.hpp:17-30: max |a-b| / max(1, |b|)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        return float("inf")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


def reference_module():
    """The unmodified reference pybind module (oracle/_ref/_synkpar_ref), or None."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import _synkpar_ref  # noqa: F401
        return _synkpar_ref
    except ImportError:
        return None
