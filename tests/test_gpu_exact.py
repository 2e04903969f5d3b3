"""GPU parity of the reference backends against the unmodified reference
compiled from /root/reference (oracle/_ref/_fastnn_ref).

Bar: bit-exact nearest indices AND min_dist values, identical fetch counters,
saturation counts, MatchSets (order included) and RunReports except the four
*_us timing fields -- the reference's own equivalence contract
(tests/acceptance.cpp:47-118, tests/test_reciprocal.cpp:167-178).

Every test runs twice: on the default route (tcgen05 scores + certified
resolution in the backend's arithmetic, where the inputs allow it) and with
FNL_EXACT_KERNEL=cuda_core (the CUDA-core exact scan K4 everywhere).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TIMING = ("subsample_us", "forward_nn_us", "reverse_nn_us", "harvest_us")


@pytest.fixture(autouse=True, params=["tensor_route", "cuda_core"])
def exact_kernel(request, monkeypatch):
    if request.param == "cuda_core":
        monkeypatch.setenv("FNL_EXACT_KERNEL", "cuda_core")
    else:
        monkeypatch.delenv("FNL_EXACT_KERNEL", raising=False)
    return request.param


def same_f32(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


def strip(report_json):
    r = json.loads(report_json)
    for k in TIMING:
        r.pop(k)
    return r


@pytest.mark.parametrize("dim", [1, 3, 8, 16, 24, 64, 100])
@pytest.mark.parametrize("metric", ["l2", "dot"])
def test_nn_backends_bitwise(fnl, ref, dim, metric):
    rng = np.random.default_rng(dim * 7 + (metric == "dot"))
    for trial in range(3):
        h, w = int(rng.integers(2, 24)), int(rng.integers(2, 40))
        A = ref.gen_random(h, w, dim, 100 + trial, normalize=bool(trial % 2))
        B = ref.gen_random(h + 1, w, dim, 200 + trial, normalize=bool(trial % 2))
        bs = int(rng.integers(1, 2 * h * w))
        for name, kw in [("nn_single_loop", dict(block_size=bs, precision="full")),
                         ("nn_single_loop", dict(block_size=bs, precision="hybrid")),
                         ("nn_double_loop", dict(block_size=bs, precision="full")),
                         ("nn_double_loop", dict(block_size=bs, precision="hybrid")),
                         ("nn_hybridcast", dict(block_size=bs)),
                         ("nn_bruteforce", dict())]:
            ours = getattr(fnl, name)(A, B, metric=metric, **kw)
            theirs = getattr(ref, name)(A, B, metric=metric, **kw)
            assert np.array_equal(ours["nearest"], theirs["nearest"]), (name, kw)
            assert same_f32(ours["min_dist"], theirs["min_dist"]), (name, kw)
            for k in ("a_block_fetches", "b_block_fetches", "half_saturation_events"):
                assert ours[k] == theirs[k], (name, kw, k)


def test_ties_resolve_to_lowest_index(fnl, ref):
    # quantised descriptors produce many exact distance ties
    rng = np.random.default_rng(5)
    A = (np.round(rng.uniform(-2, 2, (9, 11, 4)) * 2) / 2).astype(np.float32)
    B = (np.round(rng.uniform(-2, 2, (13, 17, 4)) * 2) / 2).astype(np.float32)
    for metric in ("l2", "dot"):
        ours = fnl.nn_single_loop(A, B, metric=metric)
        theirs = ref.nn_bruteforce(A, B, metric=metric)
        assert np.array_equal(ours["nearest"], theirs["nearest"])
        assert same_f32(ours["min_dist"], theirs["min_dist"])


def test_known_answers(fnl):
    # reference tests/test_nn.cpp:53-61 and tests/python/test_smoke.py:23-29
    A = np.array([[[0, 0], [10, 10]]], np.float32)
    B = np.array([[[9, 9], [1, 1]]], np.float32)
    r = fnl.nn_bruteforce(A, B)
    assert r["nearest"].tolist() == [1, 0] and r["min_dist"].tolist() == [2.0, 2.0]
    q = np.zeros((1, 2), np.float32)
    t = np.array([[3.0, 4.0], [1.0, 0.0]], np.float32)
    assert fnl.block_distances(q, t, metric="l2", precision="full").tolist() == [[25.0, 1.0]]
    assert fnl.block_distances(q, t, metric="l2", precision="hybrid").tolist() == [[25.0, 1.0]]
    A = fnl.gen_random(8, 8, 6, seed=1)
    B = fnl.gen_random(8, 8, 6, seed=2)
    assert fnl.nn_double_loop(A, B, block_size=16)["b_block_fetches"] == 16
    assert fnl.nn_single_loop(A, B, block_size=16)["b_block_fetches"] == 4
    A = fnl.gen_random(6, 6, 8, seed=3)
    r = fnl.nn_hybridcast(A, A, block_size=8)
    assert np.array_equal(r["nearest"], np.arange(36, dtype=np.uint32))
    assert r["min_dist"].max() == 0.0


@pytest.mark.parametrize("metric", ["l2", "dot"])
@pytest.mark.parametrize("precision", ["full", "hybrid"])
def test_block_distances_bitwise(fnl, ref, metric, precision):
    for nt in (1, 7, 8, 9, 64, 213):
        for dim in (1, 3, 24):
            Q = ref.gen_random(1, 5, dim, nt + dim, normalize=False).reshape(5, dim)
            T = ref.gen_random(1, nt, dim, nt * dim + 1, normalize=False).reshape(nt, dim)
            assert same_f32(fnl.block_distances(Q, T, metric, precision),
                            ref.block_distances(Q, T, metric, precision))


def test_hybrid_saturation_counted(fnl, ref):
    # reference tests/test_kernels.cpp:212-221: beyond-range values clamp, counted, finite
    A = np.zeros((1, 1, 4), np.float32)
    B = np.array([[[70000.0, -70000.0, 300.0, -300.0]]], np.float32)
    for metric in ("l2", "dot"):
        ours = fnl.nn_hybridcast(A, B, metric=metric)
        theirs = ref.nn_hybridcast(A, B, metric=metric)
        assert ours["half_saturation_events"] == theirs["half_saturation_events"] > 0
        assert same_f32(ours["min_dist"], theirs["min_dist"])
    big = (np.random.default_rng(1).normal(0, 300, (6, 7, 5))).astype(np.float32)
    for name in ("nn_single_loop", "nn_double_loop"):
        for metric in ("l2", "dot"):
            o = getattr(fnl, name)(big, big[::-1].copy(), block_size=5, metric=metric, precision="hybrid")
            t = getattr(ref, name)(big, big[::-1].copy(), block_size=5, metric=metric, precision="hybrid")
            assert o["half_saturation_events"] == t["half_saturation_events"] > 0
            assert np.array_equal(o["nearest"], t["nearest"])
            assert same_f32(o["min_dist"], t["min_dist"])


def _match_cases(ref):
    yield ref.gen_random(64, 48, 24, 21), ref.gen_random(64, 48, 24, 121)
    p = ref.gen_matched_pair(64, 48, 24, 7, 0.05)
    yield p["d1"], p["d2"]
    yield ref.gen_random(12, 9, 8, 2111), ref.gen_random(12, 9, 8, 2112)
    yield ref.gen_random(10, 10, 6, 31337), ref.gen_random(10, 10, 6, 31338)


@pytest.mark.parametrize("backend", ["single", "hybrid", "double", "bruteforce"])
@pytest.mark.parametrize("metric", ["l2", "dot"])
@pytest.mark.parametrize("precision", ["full", "hybrid"])
def test_reciprocal_match_identical(fnl, ref, backend, metric, precision):
    for n, (D1, D2) in enumerate(_match_cases(ref)):
        for kw in (dict(stride=8, block_size=100), dict(stride=2, block_size=13, convergence=1.0),
                   dict(k=20, max_iters=3, block_size=7)):
            if D1.shape[0] * D1.shape[1] > 1000 and kw.get("stride") == 2:
                continue
            m1, r1 = fnl.reciprocal_match(D1, D2, backend=backend, metric=metric, precision=precision, **kw)
            m2, r2 = ref.reciprocal_match(D1, D2, backend=backend, metric=metric, precision=precision, **kw)
            assert np.array_equal(m1, m2), (n, kw)
            assert strip(r1) == strip(r2), (n, kw)


def test_reciprocal_identity_and_errors(fnl):
    D = fnl.gen_random(12, 12, 8, seed=4)
    matches, rep = fnl.reciprocal_match(D, D, backend="single", stride=4)
    assert matches.shape == (9, 3)
    assert np.array_equal(matches[:, 0], matches[:, 1]) and (matches[:, 2] == 1).all()
    rep = json.loads(rep)
    assert rep["iterations"] == 1 and rep["converged_fraction"] == 1.0 and rep["backend"] == "single"
    A = fnl.gen_random(4, 4, 4, seed=1)
    B = fnl.gen_random(4, 4, 5, seed=2)
    with pytest.raises(ValueError):
        fnl.nn_bruteforce(A, B)
    with pytest.raises(ValueError):
        fnl.reciprocal_match(A, B)
    bad = A.copy()
    bad[1, 2, 3] = np.nan
    with pytest.raises(ValueError, match="non-finite value at flat index 27"):
        fnl.reciprocal_match(bad, A)
    with pytest.raises(ValueError):
        fnl.reciprocal_match(A, A, stride=0, k=0)
    with pytest.raises(ValueError):
        fnl.reciprocal_match(A, A, backend="nope")


@pytest.mark.parametrize("metric", ["l2", "dot"])
def test_mutual_nn_identical(fnl, ref, metric):
    for seed in range(4):
        D1 = ref.gen_random(5 + seed, 6, 4, 10 * seed, normalize=False)
        D2 = ref.gen_random(6, 5 + seed, 4, 10 * seed + 1, normalize=False)
        assert np.array_equal(fnl.mutual_nn_exact(D1, D2, metric), ref.mutual_nn_exact(D1, D2, metric))
    p = ref.gen_matched_pair(10, 10, 8, 5, 0.0)
    m = fnl.mutual_nn_exact(p["d1"], p["d2"])
    assert m.shape[0] == 100 and np.array_equal(p["truth"][m[:, 0]], m[:, 1])


@pytest.mark.slow
@pytest.mark.parametrize("backend", ["single", "hybrid"])
def test_c2_full_size_identical(fnl, ref, backend):
    """BASELINE config C2: 512x384 d=24, stride 8, seeds 606/607, dot metric."""
    D1 = ref.gen_random(512, 384, 24, 606)
    D2 = ref.gen_random(512, 384, 24, 607)
    threads = os.cpu_count() or 1
    m1, r1 = fnl.reciprocal_match(D1, D2, backend=backend, metric="dot", block_size=384)
    m2, r2 = ref.reciprocal_match(D1, D2, backend=backend, metric="dot", block_size=384, threads=threads)
    assert np.array_equal(m1, m2)
    assert strip(r1) == strip(r2)
