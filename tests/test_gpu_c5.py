"""BASELINE config C5 (one 1536x1152 d=24 pair, 27,648 samples, gen_random
seeds 2606/2607, dot, stride 8) against the reference's own MatchSet
(tests/golden/recip_c5.npz, generated from the unmodified reference by
tests/golden/make_golden_c5.py): unsharded, and target-sharded over 2 ranks
(both sharing the box's one GPU) with either key transport."""
import hashlib
import os
import socket

import numpy as np
import pytest

from tests.test_gpu_shard import _worker

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "recip_c5.npz")


def _maps(fnl, z):
    D1 = fnl.gen_random(1536, 1152, 24, 2606)
    D2 = fnl.gen_random(1536, 1152, 24, 2607)
    assert hashlib.sha256(D1.tobytes()).digest() == z["sha_d1"].tobytes()
    assert hashlib.sha256(D2.tobytes()).digest() == z["sha_d2"].tobytes()
    return D1, D2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("backend", ["single", "hybrid"])
def test_c5_unsharded_equals_reference(fnl, gold, backend):
    D1, D2 = _maps(fnl, gold)
    got, _ = fnl.reciprocal_match(D1, D2, backend=backend, metric="dot", stride=8)
    assert np.array_equal(got, gold[f"matches_{backend}"])


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_c5_sharded_two_ranks_equals_reference(fnl, gold, transport):
    import torch.multiprocessing as mp
    D1, D2 = _maps(fnl, gold)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), D1, D2, "dot", out, transport, 1, "single"), nprocs=2, join=True)
    for r in range(2):
        got, _ = out[r]
        assert np.array_equal(got.astype(np.uint32), gold["matches_single"]), f"rank {r}"
