"""ctypes front-end of the CPU checkers (TEST INFRASTRUCTURE ONLY).

Two checkers live under oracle/_ref/ (built by oracle/Makefile):

* ``liboracle.so``  -- our plain-C restatement (fastnn_oracle.c), and
* ``_fastnn_ref``   -- the unmodified reference compiled from /root/reference.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package never
does; it runs on the GPU or raises.
"""
from __future__ import annotations

import ctypes
import importlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(REF_DIR, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run `make -C oracle`)")
        L = ctypes.CDLL(path)
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
        L.orc_float_to_half_bits.restype = ctypes.c_uint16
        L.orc_float_to_half_bits.argtypes = [ctypes.c_float, ctypes.POINTER(ctypes.c_int)]
        L.orc_half_bits_to_float.restype = ctypes.c_float
        L.orc_half_bits_to_float.argtypes = [ctypes.c_uint16]
        L.orc_pair_distance.restype = ctypes.c_float
        L.orc_pair_distance.argtypes = [f32p, f32p, ctypes.c_uint32, ctypes.c_int]
        L.orc_nn_scan.restype = None
        L.orc_nn_scan.argtypes = [f32p, ctypes.c_uint32, f32p, ctypes.c_uint32, ctypes.c_uint32,
                                  ctypes.c_int, ctypes.c_int, u32p, f32p,
                                  ctypes.POINTER(ctypes.c_uint64)]
        L.orc_top2.restype = None
        L.orc_top2.argtypes = [f32p, ctypes.c_uint32, f32p, ctypes.c_uint32, ctypes.c_uint32,
                               ctypes.c_int, f32p, u32p, f32p]
        L.orc_grid_subsample.restype = ctypes.c_uint32
        L.orc_grid_subsample.argtypes = [ctypes.c_uint32] * 4 + [ctypes.c_void_p]
        L.orc_reciprocal_match.restype = ctypes.c_uint32
        L.orc_reciprocal_match.argtypes = [
            f32p, ctypes.c_uint32, ctypes.c_uint32, f32p, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_int, u32p,
            ctypes.POINTER(OrcReport)]
        _lib = L
    return _lib


class OrcReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_uint32), ("samples", ctypes.c_uint32),
                ("converged", ctypes.c_uint32), ("matches_emitted", ctypes.c_uint32),
                ("duplicates_dropped", ctypes.c_uint32),
                ("a_block_fetches", ctypes.c_uint64), ("b_block_fetches", ctypes.c_uint64),
                ("half_saturation_events", ctypes.c_uint64), ("history_len", ctypes.c_uint32),
                ("active_history", ctypes.c_uint32 * 64)]


def reference():
    """The compiled, unmodified reference pybind module (``_fastnn_ref``)."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    return importlib.import_module("_fastnn_ref")


def _rows(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a.reshape(-1, a.shape[-1]) if a.ndim != 2 else a


def to_half_round(x: float):
    sat = ctypes.c_int(0)
    bits = lib().orc_float_to_half_bits(ctypes.c_float(x), ctypes.byref(sat))
    return float(lib().orc_half_bits_to_float(bits)), bool(sat.value)


def half_bits(x: float) -> int:
    return int(lib().orc_float_to_half_bits(ctypes.c_float(x), None))


def half_round_array(a):
    """Vectorised binary16 RNE with the reference's saturation rule."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = a.astype(np.float16).astype(np.float32)  # IEEE RNE, overflow -> inf
    big = np.abs(a) >= 65520.0
    out[big] = np.copysign(np.float32(65504.0), a[big])
    return out


def nn_scan(queries, targets, metric="l2", hybrid=False):
    q, t = _rows(queries), _rows(targets)
    n = q.shape[0]
    nearest = np.zeros(n, np.uint32)
    md = np.zeros(n, np.float32)
    sat = ctypes.c_uint64(0)
    lib().orc_nn_scan(q, n, t, t.shape[0], q.shape[1], int(metric == "l2"), int(hybrid),
                      nearest, md, ctypes.byref(sat))
    return {"nearest": nearest, "min_dist": md, "half_saturation_events": sat.value}


def top2(queries, targets, metric="l2"):
    q, t = _rows(queries), _rows(targets)
    n = q.shape[0]
    b = np.zeros(n, np.float32)
    s = np.zeros(n, np.float32)
    bi = np.zeros(n, np.uint32)
    lib().orc_top2(q, n, t, t.shape[0], q.shape[1], int(metric == "l2"), b, bi, s)
    return bi, b, s


def grid_subsample(h, w, k=0, stride=8):
    n = lib().orc_grid_subsample(h, w, k, stride, None)
    out = np.zeros(max(n, 1), np.uint32)
    lib().orc_grid_subsample(h, w, k, stride, out.ctypes.data_as(ctypes.c_void_p))
    return out[:n]


_BACKENDS = {"bruteforce": 0, "double": 1, "single": 2, "hybrid": 3}


def reciprocal_match(D1, D2, backend="single", k=0, stride=8, max_iters=10, convergence=0.99,
                     metric="l2", precision="full", block_size=4096):
    D1 = np.ascontiguousarray(D1, np.float32)
    D2 = np.ascontiguousarray(D2, np.float32)
    h1, w1, d = D1.shape
    h2, w2, _ = D2.shape
    stride = 0 if k > 0 else stride
    ns = lib().orc_grid_subsample(h1, w1, k, stride, None)
    pairs = np.zeros(3 * max(ns, 1), np.uint32)
    rep = OrcReport()
    n = lib().orc_reciprocal_match(D1, h1, w1, D2, h2, w2, d, k, stride, max_iters, convergence,
                                   int(metric == "l2"), int(precision == "hybrid"), block_size,
                                   _BACKENDS[backend], pairs, ctypes.byref(rep))
    report = {f: getattr(rep, f) for f, _ in OrcReport._fields_ if f != "active_history"}
    report["active_history"] = list(rep.active_history[: rep.history_len])
    return pairs[: 3 * n].reshape(n, 3), report
