"""Native NCCL in the C-ABI (fnl_comm_*): config C5's per-pass key reduction
issued by the library itself (ncclAllReduce(int64, MIN) on the matcher's
stream).  The box has one GPU, so the communicator has one rank here -- the
sharded key path still runs end to end (encode, NCCL all-reduce, decode) and
must reproduce the unsharded MatchSet; multi-rank runs use the same code with
one process per GPU (tests/cpp/c5_sharded with FNL_RANK / FNL_NRANKS)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("backend,metric", [("single", "dot"), ("hybrid", "dot"), ("tensor", "l2"),
                                            ("single", "l2")])
def test_cpp_c5_sharded_over_native_nccl(backend, metric):
    exe = os.path.join(ROOT, "tests", "cpp", "c5_sharded")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/c5_sharded not built (make testbins)")
    out = subprocess.run([exe, "192", "144", backend, metric], cwd=ROOT, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and "IDENTICAL" in out.stdout, out.stdout + out.stderr[-2000:]


def test_python_native_comm_single_rank(fnl, ref):
    import torch

    from paper_2503_10017_b200.shard import NativeComm, match_sharded
    D1 = fnl.gen_random(128, 96, 24, 606)
    D2 = fnl.gen_random(128, 96, 24, 607)
    comm = NativeComm()
    try:
        n, r, ver = comm.info()
        assert (n, r) == (1, 0) and ver >= 21800
        for backend in ("single", "tensor"):
            pairs, counts, _ = match_sharded(torch.from_numpy(D1).cuda(), torch.from_numpy(D2).cuda(),
                                             backend=backend, transport="nccl-native", comm=comm)
            got = pairs[0, : int(counts[0])].cpu().numpy().astype(np.uint32)
            want, _ = fnl.reciprocal_match(D1, D2, backend=backend, metric="dot")
            assert np.array_equal(got, want), backend
        want_ref, _ = ref.reciprocal_match(D1, D2, backend="single", metric="dot")
        pairs, counts, _ = match_sharded(torch.from_numpy(D1).cuda(), torch.from_numpy(D2).cuda(),
                                         backend="single", transport="nccl-native", comm=comm)
        assert np.array_equal(pairs[0, : int(counts[0])].cpu().numpy().astype(np.uint32), want_ref)
    finally:
        comm.close()
