"""CPU: the C restatement (oracle/fastnn_oracle.c) pinned against the reference's
own known answers and against golden vectors produced by the compiled
reference (tests/golden/make_golden.py)."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


def test_half_known_answers(orc):
    # reference tests/test_half.cpp:14-84
    cases = {2048.0: 2048.0, 2049.0: 2048.0, 2051.0: 2052.0, 2050.5: 2050.0, 1.0: 1.0, -2049.0: -2048.0,
             65504.0: 65504.0, 65519.0: 65504.0, 2.0**-24: 2.0**-24, 2.0**-25: 0.0, 2.0**-14: 2.0**-14}
    for x, want in cases.items():
        got, sat = orc.to_half_round(x)
        assert got == want and not sat, x
    for x in (65520.0, -1e9, float("inf")):
        got, sat = orc.to_half_round(x)
        assert abs(got) == 65504.0 and sat
    got, _ = orc.to_half_round(-0.0)
    assert got == 0.0 and np.signbit(got)
    got, _ = orc.to_half_round(float(np.nextafter(np.float32(2.0**-25), np.float32(1))))
    assert got == 2.0**-24


def test_half_exhaustive_round_trip(orc):
    # every finite binary16 pattern widens and converts back to itself (test_half.cpp:43-51)
    lib = orc.lib()
    bits = np.arange(0, 0x10000, dtype=np.uint32)
    finite = ((bits >> 10) & 0x1F) != 0x1F
    vals = np.frombuffer(bits.astype(np.uint16).tobytes(), dtype=np.float16).astype(np.float32)
    for b, v in zip(bits[finite][::7], vals[finite][::7]):
        assert lib.orc_float_to_half_bits(float(v), None) == b


def test_half_golden(orc):
    g = np.load(os.path.join(GOLD, "half.npz"))
    got = np.array([orc.to_half_round(float(x))[0] for x in g["probes"]], np.float32)
    assert np.array_equal(got.view(np.uint32), g["rounded"].view(np.uint32))


def test_grid_golden(orc, golden):
    for case in golden["grid"]:
        h, w, k, s = case["args"]
        assert orc.grid_subsample(h, w, k, s).tolist() == case["ids"]


def test_nn_golden(orc, fnl):
    g = np.load(os.path.join(GOLD, "nn_c1.npz"))
    D1 = fnl.gen_random(64, 48, 24, 21)
    D2 = fnl.gen_random(64, 48, 24, 121)
    for metric in ("l2", "dot"):
        for prec in ("full", "hybrid"):
            r = orc.nn_scan(D1, D2, metric, hybrid=prec == "hybrid")
            assert np.array_equal(r["nearest"], g[f"{metric}_{prec}_nearest"])
            assert np.array_equal(r["min_dist"].view(np.uint32), g[f"{metric}_{prec}_min_dist"].view(np.uint32))
            assert r["half_saturation_events"] == g[f"{metric}_{prec}_counters"][2]


def test_reciprocal_golden(orc, fnl, golden):
    D1 = fnl.gen_random(64, 48, 24, 21)
    D2 = fnl.gen_random(64, 48, 24, 121)
    mp = fnl.gen_matched_pair(64, 48, 24, 7, 0.05, "random")
    maps = {"random": (D1, D2), "matched": (mp["d1"], mp["d2"])}
    for case in golden["reciprocal_c1"]:
        A, B = maps[case["pair"]]
        m, rep = orc.reciprocal_match(A, B, backend=case["backend"], metric=case["metric"],
                                      precision=case["precision"], **case["kwargs"])
        assert m.tolist() == case["matches"], case["backend"]
        want = case["report"]
        for key in ("iterations", "samples", "converged", "duplicates_dropped", "matches_emitted",
                    "a_block_fetches", "b_block_fetches", "half_saturation_events", "active_history"):
            assert rep[key] == want[key], key


def test_tensor_semantics_golden(orc, fnl, golden):
    D1 = orc.half_round_array(fnl.gen_random(64, 48, 24, 21))
    D2 = orc.half_round_array(fnl.gen_random(64, 48, 24, 121))
    for case in golden["tensor_semantics_c1"]:
        m, _ = orc.reciprocal_match(D1, D2, backend="single", metric=case["metric"])
        assert m.tolist() == case["matches"]


def test_oracle_matches_compiled_reference(orc, ref):
    """Random small instances: restatement vs the compiled reference itself."""
    rng = np.random.default_rng(7)
    for n in range(12):
        h, w, d = int(rng.integers(3, 12)), int(rng.integers(3, 12)), int(rng.choice([2, 8, 24]))
        A = ref.gen_random(h, w, d, 100 + n, normalize=bool(n % 2))
        B = ref.gen_random(h, w + 1, d, 200 + n, normalize=bool(n % 2))
        metric = "dot" if n % 3 == 0 else "l2"
        for prec in ("full", "hybrid"):
            mine = orc.nn_scan(A, B, metric, hybrid=prec == "hybrid")
            theirs = ref.nn_single_loop(A, B, metric=metric, precision=prec)
            assert np.array_equal(mine["nearest"], theirs["nearest"])
            assert np.array_equal(mine["min_dist"].view(np.uint32), theirs["min_dist"].view(np.uint32))
        for backend in ("single", "hybrid", "double", "bruteforce"):
            kw = dict(stride=int(rng.integers(1, 4)), block_size=int(rng.integers(1, 40)), metric=metric)
            m1, r1 = orc.reciprocal_match(A, B, backend=backend, **kw)
            m2, r2 = ref.reciprocal_match(A, B, backend=backend, **kw)
            assert np.array_equal(m1, m2)
            r2 = json.loads(r2)
            assert r1["active_history"] == r2["active_history"]
            assert (r1["a_block_fetches"], r1["b_block_fetches"]) == (r2["a_block_fetches"], r2["b_block_fetches"])


def test_attention_oracle_pinned_by_loop():
    """The vectorised FlashMatch oracle agrees with its two-pass loop form."""
    import numpy as np
    from oracle import attention
    rng = np.random.default_rng(5)
    q = rng.standard_normal((7, 64)).astype(np.float16)
    k = rng.standard_normal((11, 64)).astype(np.float16)
    v = rng.standard_normal((11, 64)).astype(np.float16)
    a = attention.attention(q, k, v)
    b = attention.attention_loop(q.tolist(), k.tolist(), v.tolist())
    assert np.abs(a - b).max() < 1e-12
