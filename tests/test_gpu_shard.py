"""Config C5 on the device: the target-sharded matcher (fnl_reciprocal_match_
sharded_device) run as 2 or 3 processes on the one B200 with a real int64 MIN
all-reduce (gloo on CUDA tensors; NCCL on a multi-GPU box) must give every
rank the MatchSet of the unsharded tensor backend, bit for bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, D1, D2, metric, out, transport="nccl", calls=1, backend="tensor"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2503_10017_b200.shard import match_sharded
    d1 = torch.from_numpy(D1).cuda()
    d2 = torch.from_numpy(D2).cuda()
    if transport == "p2p":
        # one transport reused over several calls (barrier counters carry over)
        from paper_2503_10017_b200.shard import PeerTransport
        samples = ((D1.shape[0] + 7) // 8) * ((D1.shape[1] + 7) // 8)
        peers = PeerTransport(samples, None)
        for _ in range(calls):
            pairs, counts, stats = match_sharded(d1, d2, metric=metric, transport="p2p", peers=peers,
                                                 backend=backend)
        torch.cuda.synchronize()
        dist.barrier()
        peers.close()
    else:
        pairs, counts, stats = match_sharded(d1, d2, metric=metric, backend=backend)
    torch.cuda.synchronize()
    n = int(counts[0].item())
    out[rank] = (pairs[0, :n].cpu().numpy().copy(), stats[0]["iterations"])
    dist.destroy_process_group()


@pytest.mark.parametrize("H,W,world,metric", [(128, 96, 2, "dot"), (128, 96, 3, "l2"), (512, 384, 2, "dot")])
def test_sharded_equals_unsharded(fnl, H, W, world, metric):
    import torch.multiprocessing as mp
    D1 = fnl.gen_random(H, W, 24, 606)
    D2 = fnl.gen_random(H, W, 24, 607)
    want, _ = fnl.reciprocal_match(D1, D2, backend="tensor", metric=metric)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), D1, D2, metric, out), nprocs=world, join=True)
    for r in range(world):
        got, _ = out[r]
        assert np.array_equal(got.astype(np.uint32), want), f"rank {r}"


@pytest.mark.parametrize("H,W,world,metric,calls", [(128, 96, 2, "dot", 3), (128, 96, 3, "l2", 1)])
def test_sharded_peer_memory_equals_unsharded(fnl, H, W, world, metric, calls):
    """The peer-memory transport (CUDA IPC mapped key buffers, system-scope
    atomicMin pushes from the merge epilogues, peer-memory barrier) -- here
    between processes sharing the one GPU -- gives the same MatchSet."""
    import torch.multiprocessing as mp
    D1 = fnl.gen_random(H, W, 24, 606)
    D2 = fnl.gen_random(H, W, 24, 607)
    want, _ = fnl.reciprocal_match(D1, D2, backend="tensor", metric=metric)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), D1, D2, metric, out, "p2p", calls), nprocs=world, join=True)
    for r in range(world):
        got, _ = out[r]
        assert np.array_equal(got.astype(np.uint32), want), f"rank {r}"


@pytest.mark.parametrize("backend,metric", [("single", "dot"), ("single", "l2"), ("hybrid", "dot")])
def test_sharded_reference_backends_equal_reference(fnl, ref, backend, metric):
    """The reference backends shard too (tensor route, winner keys in the
    backend's own arithmetic): 2 ranks == the reference on the same maps."""
    import torch.multiprocessing as mp
    D1 = fnl.gen_random(128, 96, 24, 606)
    D2 = fnl.gen_random(128, 96, 24, 607)
    want, _ = ref.reciprocal_match(D1, D2, backend=backend, metric=metric, stride=8)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), D1, D2, metric, out, "nccl", 1, backend), nprocs=2, join=True)
    for r in range(2):
        got, _ = out[r]
        assert np.array_equal(got.astype(np.uint32), want), f"rank {r}"
