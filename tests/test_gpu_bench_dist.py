"""bench.py's B200 arm at N=2 (the driver launches N>1 under torchrun, one
rank per GPU).  The GPU box has one GPU, so both ranks share it and talk over
gloo (FNL_BENCH_DIST_BACKEND=gloo): timings are meaningless here, but the
sharding is real -- each rank matches its own contiguous range of pairs with
no data-path collective, rank 0 alone prints one JSON line, and the matches
rank 1 reports are exactly those of pairs [B, 2B) matched directly."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_b200_arm_two_ranks(fnl):
    B = 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29563", "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--pairs", str(B), "--e2e-steps", "1", "--no-c3", "--no-c5", "--no-cpu-baseline",
           "--no-other-backends"]
    env = dict(os.environ, FNL_BENCH_DIST_BACKEND="gloo")
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["steps"] == 2
    c = d["config"]
    assert c["global_batch"] == 2 * B and c["pairs_per_gpu_per_step"] == B
    assert c["pairs_by_rank"] == [[0, B], [B, 2 * B]]
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    # rank 1's matches == pairs [B, 2B) matched here directly (same maps)
    sys.path.insert(0, ROOT)
    import bench
    maps = {}

    def m(i):
        if i not in maps:
            maps[i] = fnl.gen_random(bench.H, bench.W, bench.D, 1000 + i)
        return maps[i]
    for rank in (0, 1):
        idx = [bench.pair_maps(k) for k in range(rank * B, (rank + 1) * B)]
        D1 = np.stack([m(a) for a, _ in idx])
        D2 = np.stack([m(b) for _, b in idx])
        _, counts, _ = fnl.reciprocal_match_batch(D1, D2, backend=c["backend"], stride=bench.STRIDE,
                                                  metric=bench.METRIC)
        assert int(counts.sum()) == c["matches_by_rank"][rank], rank
