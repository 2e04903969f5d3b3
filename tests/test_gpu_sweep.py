"""Randomised parity sweep in the style of the reference acceptance criteria
(tests/acceptance.cpp AC1 / AC3 / AC4): many small instances with ragged
shapes, several descriptor dims, both metrics, different D1 / D2 sizes and
matcher settings.  Every backend must reproduce the compiled reference bit for
bit: the reference backends on the maps as given, the tensor backend on
binary16-rounded maps."""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu


def _instances(n, seed):
    rng = np.random.default_rng(seed)
    for i in range(n):
        h1, w1 = int(rng.integers(3, 70)), int(rng.integers(3, 70))
        if rng.random() < 0.5:
            h2, w2 = h1, w1
        else:
            h2, w2 = int(rng.integers(3, 70)), int(rng.integers(3, 70))
        d = int(rng.choice([2, 8, 16, 24, 30]))
        metric = str(rng.choice(["dot", "l2"]))
        stride = int(rng.choice([1, 2, 3, 4, 8]))
        k = int(rng.choice([0, 0, 0, 17]))
        iters = int(rng.choice([1, 3, 10]))
        conv = float(rng.choice([0.5, 0.99, 1.0]))
        yield i, (h1, w1, h2, w2, d, metric, stride, k, iters, conv, 5000 + 2 * i)


@pytest.mark.parametrize("i,cfg", list(_instances(120, 7)))
def test_reciprocal_sweep_tensor(fnl, ref, i, cfg):
    h1, w1, h2, w2, d, metric, stride, k, iters, conv, seed = cfg
    if metric == "l2" and d > 30:
        pytest.skip("tensor l2 carries the norm in 2 extra channels (d <= 30)")
    D1 = oracle.half_round_array(fnl.gen_random(h1, w1, d, seed))
    D2 = oracle.half_round_array(fnl.gen_random(h2, w2, d, seed + 1))
    kw = dict(metric=metric, stride=stride, k=k, max_iters=iters, convergence=conv)
    got, _ = fnl.reciprocal_match(D1, D2, backend="tensor", **kw)
    want, _ = ref.reciprocal_match(D1, D2, backend="single", **kw)
    assert np.array_equal(got, want), cfg


@pytest.mark.parametrize("i,cfg", list(_instances(60, 11)))
@pytest.mark.parametrize("backend", ["single", "hybrid"])
def test_reciprocal_sweep_exact(fnl, ref, backend, i, cfg):
    h1, w1, h2, w2, d, metric, stride, k, iters, conv, seed = cfg
    D1 = fnl.gen_random(h1, w1, d, seed)
    D2 = fnl.gen_random(h2, w2, d, seed + 1)
    kw = dict(metric=metric, stride=stride, k=k, max_iters=iters, convergence=conv)
    got, rep = fnl.reciprocal_match(D1, D2, backend=backend, **kw)
    want, rep_ref = ref.reciprocal_match(D1, D2, backend=backend, **kw)
    assert np.array_equal(got, want), cfg


@pytest.mark.parametrize("seed", [11, 12, 13])
@pytest.mark.parametrize("backend", ["tensor", "single"])
def test_permutation_recovered_at_iteration_one(fnl, seed, backend):
    """AC4 (tests/acceptance.cpp:185-225): a noise-free permuted pair is
    recovered completely at iteration 1, in sample order."""
    rng = np.random.default_rng(seed)
    H, W, d = 48, 40, 24
    D1 = oracle.half_round_array(fnl.gen_random(H, W, d, seed))
    perm = rng.permutation(H * W)
    D2 = np.ascontiguousarray(D1.reshape(-1, d)[perm].reshape(H, W, d))
    m, _ = fnl.reciprocal_match(D1, D2, backend=backend, metric="dot", stride=8)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(H * W)
    samples = fnl.grid_subsample(H, W, stride=8)
    assert m.shape[0] == len(samples)
    assert np.array_equal(m[:, 0], samples)
    assert np.array_equal(m[:, 1], inv[m[:, 0]])
    assert (m[:, 2] == 1).all()


def _nn_instances(n, seed):
    rng = np.random.default_rng(seed)
    for i in range(n):
        hq, wq = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        ht, wt = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        d = int(rng.choice([1, 5, 7, 24, 30, 31, 33, 64]))
        metric = str(rng.choice(["dot", "l2"]))
        bs = int(rng.choice([1, 3, 64, 100000]))
        yield i, (hq, wq, ht, wt, d, metric, bs, 9000 + 2 * i)


@pytest.mark.parametrize("i,cfg", list(_nn_instances(60, 3)))
def test_nn_sweep_all_backends(fnl, ref, i, cfg):
    """AC1 (tests/acceptance.cpp:47-118): bruteforce == double == single (and
    hybrid) bitwise on nearest AND min_dist, ragged shapes, odd dims, block
    sizes from 1 to beyond the map."""
    hq, wq, ht, wt, d, metric, bs, seed = cfg
    Q = fnl.gen_random(hq, wq, d, seed)
    T = fnl.gen_random(ht, wt, d, seed + 1)
    for name in ("nn_single_loop", "nn_double_loop"):
        got = getattr(fnl, name)(Q, T, metric=metric, block_size=bs)
        want = getattr(ref, name)(Q, T, metric=metric, block_size=bs)
        for key in ("nearest", "min_dist", "a_block_fetches", "b_block_fetches"):
            assert np.array_equal(np.asarray(got[key]), np.asarray(want[key])), (name, key, cfg)
    got = fnl.nn_bruteforce(Q, T, metric=metric)
    want = ref.nn_bruteforce(Q, T, metric=metric)
    assert np.array_equal(got["nearest"], want["nearest"]) and np.array_equal(got["min_dist"], want["min_dist"])
    got = fnl.nn_hybridcast(Q, T, metric=metric, block_size=bs)
    want = ref.nn_hybridcast(Q, T, metric=metric, block_size=bs)
    for key in ("nearest", "min_dist", "half_saturation_events"):
        assert np.array_equal(np.asarray(got[key]), np.asarray(want[key])), ("hybrid", key, cfg)
    if d + (2 if metric == "l2" else 0) <= 32:
        Qh, Th = oracle.half_round_array(Q), oracle.half_round_array(T)
        got = fnl.nn_tensor(Qh, Th, metric=metric)
        want = ref.nn_single_loop(Qh, Th, metric=metric)
        assert np.array_equal(got["nearest"], want["nearest"]), ("tensor", cfg)
        assert np.array_equal(got["min_dist"], want["min_dist"]), ("tensor min_dist", cfg)
