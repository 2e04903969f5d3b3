"""CPU: host-side logic of the product (no GPU needed) against the reference:
seeded generators, grid subsample, binary16, scalar distance, .fmap IO, report
formats; plus the C-ABI library's exported symbols and its no-GPU behaviour."""
import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


def test_generators_bit_identical_to_reference(fnl, golden):
    for g in golden["gen_random"]:
        h, w, d, seed, norm = g["args"]
        assert sha(fnl.gen_random(h, w, d, seed, normalize=norm)) == g["sha256"], g["args"]
    for g in golden["gen_matched_pair"]:
        h, w, d, seed, sigma, perm = g["args"]
        p = fnl.gen_matched_pair(h, w, d, seed, sigma, perm)
        assert (sha(p["d1"]), sha(p["d2"]), sha(p["truth"])) == (g["d1"], g["d2"], g["truth"])


def test_grid_subsample(fnl, golden):
    for case in golden["grid"]:
        h, w, k, s = case["args"]
        assert fnl.grid_subsample(h, w, k=k, stride=s).tolist() == case["ids"]
    assert fnl.grid_subsample(8, 8, stride=4).tolist() == [18, 22, 50, 54]
    assert fnl.grid_subsample(480, 640, stride=8).shape[0] == 60 * 80
    with pytest.raises(ValueError):
        fnl.grid_subsample(5, 7, k=0, stride=0)


def test_half_round(fnl, orc):
    g = np.load(os.path.join(GOLD, "half.npz"))
    got = np.array([fnl.to_half_round(float(x)) for x in g["probes"]], np.float32)
    assert np.array_equal(got.view(np.uint32), g["rounded"].view(np.uint32))
    assert fnl.to_half_round(2049.0) == 2048.0 and fnl.to_half_round(2048.0) == 2048.0


def test_dist_scalar(fnl, orc, ref):
    rng = np.random.default_rng(3)
    for _ in range(200):
        d = int(rng.integers(1, 40))
        a = rng.normal(size=d).astype(np.float32)
        b = rng.normal(size=d).astype(np.float32)
        for metric in ("l2", "dot"):
            want = ref.dist_scalar(a.tolist(), b.tolist(), metric)
            assert np.float32(fnl.dist_scalar(a.tolist(), b.tolist(), metric)) == np.float32(want)
    assert fnl.dist_scalar([1, 0], [0, 1], "l2") == 2.0
    with pytest.raises(ValueError):
        fnl.dist_scalar([1.0, 2.0], [1.0], "l2")


def test_fmap_round_trip_and_cross_read(fnl, ref, tmp_path):
    m = fnl.gen_random(5, 4, 3, seed=9)
    p1, p2 = str(tmp_path / "ours.fmap"), str(tmp_path / "ref.fmap")
    fnl.write_fmap(m, p1)
    ref.write_fmap(m, p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    assert np.array_equal(fnl.read_fmap(p2), m)
    bad = bytearray(open(p1, "rb").read())
    bad[0] = ord("X")
    open(p1, "wb").write(bytes(bad))
    with pytest.raises(RuntimeError, match="bad magic"):
        fnl.read_fmap(p1)


def test_report_golden_formats(fnl):
    # reference tests/acceptance.cpp:354-397 (golden zero report, CSV header)
    zero = fnl._render_report({}, "json")
    lines = zero.splitlines()
    assert lines[0] == "{" and lines[-1] == "}" and zero.endswith("}\n")
    keys = [l.split(":")[0].strip().strip('"') for l in lines[1:-1]]
    assert keys == ["backend", "metric", "precision", "height1", "width1", "height2", "width2", "dim", "k",
                    "grid_stride", "max_iters", "convergence_fraction", "block_size", "seed", "subsample_us",
                    "forward_nn_us", "reverse_nn_us", "harvest_us", "a_block_fetches", "b_block_fetches",
                    "iterations", "samples", "converged", "converged_fraction", "half_saturated",
                    "half_saturation_events", "hybrid_full_argmin_agreement", "matches_emitted",
                    "duplicates_dropped", "active_history"]
    assert '"convergence_fraction": 0.0,' in zero and '"hybrid_full_argmin_agreement": null,' in zero
    assert '"active_history": []' in zero and '"half_saturated": false,' in zero
    csv = fnl._render_report({}, "csv").splitlines()
    assert csv[0] == ("backend,metric,precision,height1,width1,height2,width2,dim,k,grid_stride,max_iters,"
                      "convergence_fraction,block_size,seed,subsample_us,forward_nn_us,reverse_nn_us,"
                      "harvest_us,a_block_fetches,b_block_fetches,iterations,samples,converged,"
                      "converged_fraction,half_saturated,half_saturation_events,"
                      "hybrid_full_argmin_agreement,matches_emitted,duplicates_dropped")
    rep = {"backend": "single", "metric": "dot", "precision": "full", "samples": 3072, "converged": 3066,
           "converged_fraction": 0.998046875, "active_history": [1549, 123, 6], "iterations": 3}
    js = fnl._render_report(rep, "json")
    assert fnl._parse_report(js) == js


def test_report_matches_reference_rendering(fnl, golden):
    # every golden reciprocal report (rendered by the reference) re-renders identically
    for case in golden["reciprocal_c1"][:16]:
        r = dict(case["report"])
        r.update({k: 0.0 for k in ("subsample_us", "forward_nn_us", "reverse_nn_us", "harvest_us")})
        js = fnl._render_report(r, "json")
        assert json.loads(js) == r


def test_capi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "fastnn_b200.h")).read()
    declared = sorted(set(re.findall(r"\b(fnl_[a-z0-9_]+)\s*\(", header)))
    assert len(declared) >= 12
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2503_10017_b200", "libfastnn_b200.so"))
    for name in declared:
        assert hasattr(lib, name), name
    lib.fnl_abi_version.restype = ctypes.c_int
    assert lib.fnl_abi_version() == 1


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and False, reason="")
def test_no_cpu_fallback_without_gpu():
    from tests.conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("GPU present")
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2503_10017_b200", "libfastnn_b200.so"))
    lib.fnl_last_error.restype = ctypes.c_char_p
    ctx = ctypes.c_void_p()
    rc = lib.fnl_context_create(0, ctypes.byref(ctx))
    assert rc == 2  # FNL_ERUNTIME
    assert b"no CPU fallback" in lib.fnl_last_error()
    import paper_2503_10017_b200 as fnl
    A = fnl.gen_random(4, 4, 4, seed=1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fnl.nn_single_loop(A, A)
    with pytest.raises(RuntimeError):
        fnl.reciprocal_match(A, A)
