"""GPU parity of the tcgen05 tensor backend (HybridCast).

Contract: binary16 cast-in, fp32 tensor-core accumulation, fp32 compare, near
ties re-decided by the reference FMA chain.  The result must equal the
reference `single` backend run on binary16-rounded maps -- nearest indices and
min_dist bit for bit, MatchSets in order -- and every row whose tensor-core
top-2 gap is inside the certified error band is counted (near_tie_rows).
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu
TIMING = ("subsample_us", "forward_nn_us", "reverse_nn_us", "harvest_us")


def h16(a):
    return oracle.half_round_array(a)


def strip(rep):
    r = json.loads(rep)
    for k in TIMING + ("precision", "backend", "block_size", "a_block_fetches", "b_block_fetches",
                       "half_saturated", "half_saturation_events"):
        r.pop(k)
    return r


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("metric", ["dot", "l2"])
@pytest.mark.parametrize("dim", [24, 8, 30])
def test_umma_layout_and_accumulation_error(fnl, metric, dim, mode):
    """Raw TMEM scores vs float64 on the same binary16 values: pins the UMMA
    descriptor / canonical-layout encoding and measures the accumulation error
    the certification margin has to cover (margin uses 2^-16 * sum|products|)."""
    rng = np.random.default_rng(dim)
    q = h16(rng.normal(size=(256, dim)).astype(np.float32))
    t = h16(rng.normal(size=(128, dim)).astype(np.float32))
    q /= np.linalg.norm(q, axis=1, keepdims=True).astype(np.float32)
    t /= np.linalg.norm(t, axis=1, keepdims=True).astype(np.float32)
    q, t = h16(q), h16(t)
    got = fnl._tensor_selftest(q, t, metric, mode).astype(np.float64)
    exact = q.astype(np.float64) @ t.astype(np.float64).T
    if metric == "l2":
        n2 = (t.astype(np.float64) ** 2).sum(1)
        exact = exact - n2[None, :] / 2
        bound = (np.abs(q.astype(np.float64)) @ np.abs(t.astype(np.float64)).T + n2[None, :]) * 2.0**-16 \
            + n2[None, :] * 2.0**-19
    else:
        bound = (np.abs(q.astype(np.float64)) @ np.abs(t.astype(np.float64)).T) * 2.0**-16
    err = np.abs(got - exact)
    assert np.all(err <= bound), float((err / bound).max())
    # the margin has headroom: observed error far inside it
    assert (err / bound).max() < 0.25


@pytest.mark.parametrize("metric", ["dot", "l2"])
def test_nn_tensor_equals_reference_on_half_inputs(fnl, ref, metric):
    for seed in range(3):
        A = ref.gen_random(40 + seed, 33, 24, 300 + seed)
        B = ref.gen_random(37, 41 + 3 * seed, 24, 400 + seed)
        ours = fnl.nn_tensor(A, B, metric)
        theirs = ref.nn_single_loop(h16(A), h16(B), metric=metric, precision="full")
        assert np.array_equal(ours["nearest"], theirs["nearest"])
        assert np.array_equal(ours["min_dist"].view(np.uint32), theirs["min_dist"].view(np.uint32))


@pytest.mark.parametrize("nq", [1, 63, 64, 65, 127, 192, 255, 256, 257, 321, 513])
def test_nn_tensor_merge_slice_boundaries(fnl, ref, nq):
    """Query counts around the merge kernel's 64-row slices and 256-row tile
    pairs (ragged last slice, empty trailing slices, multi-tile-pair)."""
    A = ref.gen_random(1, nq, 24, 500 + nq)
    B = ref.gen_random(48, 40, 24, 600 + nq)
    ours = fnl.nn_tensor(A, B, "dot")
    theirs = ref.nn_single_loop(h16(A), h16(B), metric="dot", precision="full")
    assert np.array_equal(ours["nearest"], theirs["nearest"])
    assert np.array_equal(ours["min_dist"].view(np.uint32), theirs["min_dist"].view(np.uint32))


def test_nn_tensor_ties_and_duplicates(fnl, ref):
    # duplicated targets force exact ties: lowest index must win via the rescan
    rng = np.random.default_rng(3)
    base = h16(rng.normal(size=(1, 200, 16)).astype(np.float32))
    B = np.concatenate([base, base[:, ::-1]], axis=1).copy()
    A = base[:, :150].copy()
    for metric in ("dot", "l2"):
        ours = fnl.nn_tensor(A, B, metric)
        theirs = ref.nn_single_loop(A, B, metric=metric)
        assert np.array_equal(ours["nearest"], theirs["nearest"])


def _cases(ref):
    yield ref.gen_random(64, 48, 24, 21), ref.gen_random(64, 48, 24, 121)
    p = ref.gen_matched_pair(64, 48, 24, 7, 0.05)
    yield p["d1"], p["d2"]
    yield ref.gen_random(100, 70, 24, 5), ref.gen_random(90, 80, 24, 6)
    yield ref.gen_random(12, 9, 16, 2111), ref.gen_random(12, 9, 16, 2112)


@pytest.mark.parametrize("metric", ["dot", "l2"])
def test_reciprocal_tensor_equals_reference_on_half_inputs(fnl, ref, metric):
    for D1, D2 in _cases(ref):
        for kw in (dict(stride=8), dict(stride=3, convergence=1.0), dict(k=50, max_iters=4)):
            m1, r1 = fnl.reciprocal_match(D1, D2, backend="tensor", metric=metric, **kw)
            m2, r2 = ref.reciprocal_match(h16(D1), h16(D2), backend="single", metric=metric, **kw)
            assert np.array_equal(m1, m2)
            assert strip(r1) == strip(r2)


@pytest.mark.slow
@pytest.mark.parametrize("metric", ["dot", "l2"])
def test_c2_tensor_full_size(fnl, ref, metric):
    """C2 512x384 d=24 stride 8, random (606/607) and matched (7, sigma 0.05) pairs."""
    threads = os.cpu_count() or 1
    p = ref.gen_matched_pair(512, 384, 24, 7, 0.05)
    for D1, D2 in ((ref.gen_random(512, 384, 24, 606), ref.gen_random(512, 384, 24, 607)), (p["d1"], p["d2"])):
        m1, r1 = fnl.reciprocal_match(D1, D2, backend="tensor", metric=metric)
        m2, r2 = ref.reciprocal_match(h16(D1), h16(D2), backend="single", metric=metric,
                                      block_size=384, threads=threads)
        assert np.array_equal(m1, m2)
        assert strip(r1) == strip(r2)


def test_batch_api_matches_single(fnl, ref):
    D1 = np.stack([ref.gen_random(64, 48, 24, 1000 + 2 * k) for k in range(5)])
    D2 = np.stack([ref.gen_random(64, 48, 24, 1001 + 2 * k) for k in range(5)])
    pairs, counts, stats = fnl.reciprocal_match_batch(D1, D2, backend="tensor", metric="dot")
    for k in range(5):
        m, rep = fnl.reciprocal_match(D1[k], D2[k], backend="tensor", metric="dot")
        assert counts[k] == m.shape[0]
        assert np.array_equal(pairs[k, : counts[k]], m)
        assert stats[k]["active_history"] == json.loads(rep)["active_history"]
    pairs_e, counts_e, _ = fnl.reciprocal_match_batch(D1, D2, backend="single", metric="dot")
    for k in range(5):
        m, _ = ref.reciprocal_match(D1[k], D2[k], backend="single", metric="dot")
        assert np.array_equal(pairs_e[k, : counts_e[k]], m)


@pytest.mark.parametrize("metric", ["dot", "l2"])
def test_mutual_nn_tensor_equals_reference_on_half_maps(fnl, ref, metric):
    """dense mutual NN on the tensor cores equals the
    reference mutual_nn_exact on binary16-rounded maps (index pairs, order)."""
    from oracle import oracle
    D1 = fnl.gen_random(64, 48, 24, 31)
    D2 = fnl.gen_random(64, 48, 24, 131)
    got = fnl.mutual_nn_tensor(D1, D2, metric=metric)
    want = ref.mutual_nn_exact(oracle.half_round_array(D1), oracle.half_round_array(D2), metric=metric)
    assert np.array_equal(got, np.asarray(want, dtype=np.uint32))


@pytest.mark.slow
def test_mutual_nn_tensor_full_resolution(fnl):
    """512x384 dense mutual NN (2 x 3.87e10 scores) on the tensor path equals
    the exact CUDA-core path on binary16-rounded maps."""
    from oracle import oracle
    D1 = oracle.half_round_array(fnl.gen_random(512, 384, 24, 606))
    D2 = oracle.half_round_array(fnl.gen_random(512, 384, 24, 607))
    got = fnl.mutual_nn_tensor(D1, D2, metric="dot")
    want = fnl.mutual_nn_exact(D1, D2, metric="dot")
    assert np.array_equal(got, want)


@pytest.mark.parametrize("metric", ["dot", "l2"])
def test_confidence_compaction_equals_post_filter(fnl, ref, metric):
    """Confidence-thresholded compaction (fnl_confidence_compact_device): the
    kept matches are exactly the unthresholded MatchSet filtered by the
    reference dist_scalar <= threshold, in emission order."""
    import torch
    B, H, W, D = 3, 96, 64, 24
    maps1 = [fnl.gen_random(H, W, D, 70 + p) for p in range(B)]
    maps2 = [fnl.gen_random(H, W, D, 170 + p) for p in range(B)]
    d1 = torch.from_numpy(np.stack(maps1)).cuda()
    d2 = torch.from_numpy(np.stack(maps2)).cuda()
    S = len(fnl.grid_subsample(H, W, stride=8))
    out = torch.zeros((B, S, 3), dtype=torch.int32, device="cuda")
    cnt = torch.zeros((B,), dtype=torch.int32, device="cuda")

    def run(**kw):
        fnl.reciprocal_match_device(d1.data_ptr(), d2.data_ptr(), B, H, W, D, out.data_ptr(), cnt.data_ptr(),
                                    backend="tensor", stride=8, metric=metric, **kw)
        torch.cuda.synchronize()
        return [out[p, :int(cnt[p])].cpu().numpy().astype(np.uint32) for p in range(B)]

    full = run()
    dists = [np.array([ref.dist_scalar(maps1[p].reshape(-1, D)[i], maps2[p].reshape(-1, D)[j], metric=metric)
                       for i, j, _ in full[p]], dtype=np.float32) for p in range(B)]
    thr = float(np.median(np.concatenate(dists)))
    kept = run(max_distance=thr)
    for p in range(B):
        assert np.array_equal(kept[p], full[p][dists[p] <= np.float32(thr)])
    assert 0 < sum(len(k) for k in kept) < sum(len(f) for f in full)


def test_batch_over_1024_pairs(fnl, ref):
    """More pairs than one plan-kernel chunk (1024): the device-built work
    lists (K2p) must scan across chunks; every pair equals the exact CUDA
    `single` backend on the same binary16-rounded maps."""
    P = 1100
    base1 = [h16(ref.gen_random(16, 12, 24, 3000 + k)) for k in range(8)]
    base2 = [h16(ref.gen_random(16, 12, 24, 4000 + k)) for k in range(8)]
    D1 = np.stack([base1[k % 8] for k in range(P)])
    D2 = np.stack([base2[(k // 8) % 8] for k in range(P)])
    pt, ct, st = fnl.reciprocal_match_batch(D1, D2, backend="tensor", metric="dot", stride=2)
    ps, cs, ss = fnl.reciprocal_match_batch(D1, D2, backend="single", metric="dot", stride=2)
    assert np.array_equal(ct, cs)
    for k in range(P):
        assert np.array_equal(pt[k, : ct[k]], ps[k, : cs[k]])
        assert st[k]["active_history"] == ss[k]["active_history"]
