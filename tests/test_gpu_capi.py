"""GPU: the C-ABI called directly through ctypes (the binding INTEGRATION.md
shows a reference maintainer), compared with the compiled reference."""
import ctypes
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class MatchConfig(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("grid_stride", ctypes.c_uint32), ("max_iters", ctypes.c_uint32),
                ("convergence_fraction", ctypes.c_double), ("metric", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("block_size", ctypes.c_uint32)]


class RunStats(ctypes.Structure):
    _fields_ = [("samples", ctypes.c_uint32), ("iterations", ctypes.c_uint32), ("converged", ctypes.c_uint32),
                ("duplicates_dropped", ctypes.c_uint32), ("matches", ctypes.c_uint32),
                ("history_len", ctypes.c_uint32), ("active_history", ctypes.c_uint32 * 64),
                ("a_block_fetches", ctypes.c_uint64), ("b_block_fetches", ctypes.c_uint64),
                ("half_saturation_events", ctypes.c_uint64), ("near_tie_rows", ctypes.c_uint64),
                ("query_rows", ctypes.c_uint64), ("subsample_us", ctypes.c_double),
                ("forward_nn_us", ctypes.c_double), ("reverse_nn_us", ctypes.c_double),
                ("harvest_us", ctypes.c_double), ("rescan_rows", ctypes.c_uint64),
                ("tensor_route", ctypes.c_uint32), ("computed_query_rows", ctypes.c_uint64)]


@pytest.fixture(scope="module")
def capi():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2503_10017_b200", "libfastnn_b200.so"))
    lib.fnl_last_error.restype = ctypes.c_char_p
    ctx = ctypes.c_void_p()
    assert lib.fnl_context_create(0, ctypes.byref(ctx)) == 0, lib.fnl_last_error()
    yield lib, ctx
    lib.fnl_context_destroy(ctx)


def _match(lib, ctx, D1, D2, backend, metric, stride=8):
    f32p = ctypes.POINTER(ctypes.c_float)
    cfg = MatchConfig(0, stride, 10, 0.99, metric, 0, 4096)
    cap = -(-D1.shape[0] // stride) * -(-D1.shape[1] // stride)
    pairs = np.zeros((cap, 3), np.uint32)
    n = ctypes.c_uint32()
    st = RunStats()
    rc = lib.fnl_reciprocal_match(ctx, D1.ctypes.data_as(f32p), D1.shape[0], D1.shape[1], D2.ctypes.data_as(f32p),
                                  D2.shape[0], D2.shape[1], D1.shape[2], ctypes.byref(cfg), backend,
                                  pairs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), ctypes.byref(n),
                                  ctypes.byref(st))
    return rc, pairs[: n.value], st


def test_capi_reciprocal_single_and_tensor(capi, ref):
    lib, ctx = capi
    from oracle import oracle
    D1 = ref.gen_random(64, 48, 24, 21)
    D2 = ref.gen_random(64, 48, 24, 121)
    rc, m, st = _match(lib, ctx, D1, D2, backend=2, metric=1)  # single, dot
    assert rc == 0, lib.fnl_last_error()
    want, rep = ref.reciprocal_match(D1, D2, backend="single", metric="dot")
    assert np.array_equal(m, want)
    assert list(st.active_history[: st.history_len]) == json.loads(rep)["active_history"]
    rc, m, st = _match(lib, ctx, D1, D2, backend=4, metric=1)  # tensor, dot
    assert rc == 0, lib.fnl_last_error()
    want, _ = ref.reciprocal_match(oracle.half_round_array(D1), oracle.half_round_array(D2), backend="single",
                                   metric="dot")
    assert np.array_equal(m, want)
    assert st.query_rows > 0


def test_capi_errors(capi):
    lib, ctx = capi
    D = np.zeros((4, 4, 4), np.float32)
    D[1, 1, 1] = np.inf
    rc, _, _ = _match(lib, ctx, D, np.zeros((4, 4, 4), np.float32), backend=2, metric=0)
    assert rc == 1 and b"non-finite value at flat index 21" in lib.fnl_last_error()
    rc, _, _ = _match(lib, ctx, np.zeros((4, 4, 4), np.float32), np.zeros((4, 4, 4), np.float32), backend=9, metric=0)
    assert rc == 1


def test_kernel_profile_classes(fnl):
    """Per-kernel-class device time (fnl_kernel_profile): every class the
    tensor matcher launches is timed, and the score class equals
    fnl_kernel_timing's number."""
    D1 = fnl.gen_random(128, 96, 24, 5)
    D2 = fnl.gen_random(128, 96, 24, 6)
    fnl.kernel_timing(reset=True)
    fnl.kernel_profile(enable=1, reset=True)
    fnl.reciprocal_match(D1, D2, backend="tensor", metric="dot")
    prof = fnl.kernel_profile(enable=0, reset=True)
    timing = fnl.kernel_timing(reset=True)
    for cls in ("score", "pack", "gather", "merge", "rescan", "harvest"):
        assert prof[cls]["launches"] > 0 and prof[cls]["ms"] > 0.0, cls
    assert prof["score"]["launches"] == timing["score_launches"]
    assert abs(prof["score"]["ms"] - timing["score_ms"]) < 1e-6
