"""Target-column sharding of one oversized pair over N GPUs (config C5).

Every rank holds both descriptor maps.  In each NN pass rank r scans only its
contiguous range of 256-target tiles of the target map and produces, per
query, the exact winner of that range as a signed 64-bit key

    key = ((orderable(dist) << 32) | index) ^ 2**63

so that an int64 MIN all-reduce over the ranks (NCCL over NVLink, or gloo)
selects the global reference winner -- smallest distance, lowest index on an
exact tie (src/kernels.cpp:202-229, 287-300) -- and every rank continues the
reciprocal loop (harvest, convergence: src/reciprocal.cpp:142-185) with
identical state.  The MatchSet is therefore bit-identical to the unsharded
run.  This is the only collective on the path: 8 B per active query per pass
(221 KB for 27,648 queries).

The device work is in libfastnn_b200.so (fnl_reciprocal_match_sharded_device);
this module only supplies the key buffer and the all-reduce callback.

``transport="nccl-native"`` keeps NCCL but drops the Python callback: the
library owns an NCCL communicator (fnl_comm_create, NativeComm) and issues
ncclAllReduce(int64, MIN) on the matcher's stream itself.

``transport="p2p"`` replaces the NCCL all-reduce with peer memory: every
rank's key buffers and barrier counter are CUDA-IPC-mapped into every other
rank (NVLink / NVSwitch peer access), the merge and near-tie epilogues push
each winner key straight into all ranks' buffers with a system-scope
atomicMin, and a one-thread peer-memory barrier kernel closes the pass -- the
collective is fused into the kernels that produce the keys.
"""
import numpy as np

TILE = 256                 # targets per K3 tile (kTargetTileRows)
KEY_NONE = (1 << 63) - 1   # INT64_MAX: no candidate in this shard


def shard_tiles(ntargets, rank, count):
    """Target tile range [begin, end) of shard `rank` (same split as capi.cu)."""
    tiles = (ntargets + TILE - 1) // TILE
    return tiles * rank // count, tiles * (rank + 1) // count


def orderable(dist):
    """float32 -> u32 with the same total order as <, -0 == +0 (fnl_common.cuh)."""
    b = np.asarray(dist, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = np.where(b == 0x80000000, 0, b)
    return np.where(b & 0x80000000, (~b) & 0xFFFFFFFF, b | 0x80000000).astype(np.uint64)


def encode_keys(dist, index):
    """(dist, global index) -> signed shard keys (int64)."""
    k = (orderable(dist) << np.uint64(32)) | np.asarray(index, dtype=np.uint64)
    return (k ^ np.uint64(1 << 63)).view(np.int64)


def decode_index(keys):
    return (np.asarray(keys, dtype=np.int64).view(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)


class PeerTransport:
    """Key buffers (two NN-pass parities) and a barrier counter per rank,
    mapped into every rank of `group` with CUDA IPC.  Reusable across calls
    with at most `nkeys` keys per pass; close() unmaps and frees."""

    def __init__(self, nkeys, group=None):
        import torch.distributed as dist

        from . import _fastnn
        self._fnl = _fastnn
        self.nkeys = nkeys
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.keys = _fastnn.p2p_alloc(2 * nkeys * 8, True)
        self.flag = _fastnn.p2p_alloc(4, False)
        mine = (_fastnn.ipc_handle(self.keys), _fastnn.ipc_handle(self.flag))
        handles = [None] * world
        if world > 1:
            dist.all_gather_object(handles, mine, group=group)
        else:
            handles = [mine]
        self.opened = []
        self.peer_keys, self.peer_flags = [], []
        ok, err = True, ""
        try:
            for r, (hk, hf) in enumerate(handles):
                if r == self.rank:
                    self.peer_keys.append(self.keys)
                    self.peer_flags.append(self.flag)
                    continue
                k = _fastnn.ipc_open(hk)
                self.opened.append(k)
                f = _fastnn.ipc_open(hf)
                self.opened.append(f)
                self.peer_keys.append(k)
                self.peer_flags.append(f)
        except Exception as e:  # e.g. no peer access between these GPUs
            ok, err = False, str(e)
        # every rank learns whether every rank mapped every buffer (and no rank
        # pushes before all have): all succeed or all raise, nobody hangs
        verdicts = [(ok, err)]
        if world > 1:
            verdicts = [None] * world
            dist.all_gather_object(verdicts, (ok, err), group=group)
        bad = [e for good, e in verdicts if not good]
        if bad:
            self.close()
            raise RuntimeError("peer-memory transport unavailable: " + bad[0])
        self.seq = 0
        self.broken = None

    def close(self):
        for p in self.opened:
            self._fnl.ipc_close(p)
        self.opened = []
        self._fnl.p2p_free(self.keys)
        self._fnl.p2p_free(self.flag)


class NativeComm:
    """A native NCCL communicator inside libfastnn_b200 (fnl_comm_create) over
    the ranks of `group`: the library runs ncclAllReduce(int64, MIN) on the
    keys itself, on the matcher's stream -- no Python callback per pass.
    Rank 0's NCCL id reaches the others through torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist

        from . import _fastnn
        self._fnl = _fastnn
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        ids = [_fastnn.nccl_unique_id() if self.rank == 0 else None]
        if self.world > 1:
            dist.broadcast_object_list(ids, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
        self.handle = _fastnn.comm_create(ids[0], self.world, self.rank)

    def info(self):
        return self._fnl.comm_info(self.handle)

    def close(self):
        if self.handle:
            self._fnl.comm_destroy(self.handle)
            self.handle = 0


def match_sharded(d1, d2, stride=8, metric="dot", group=None, backend="tensor", transport="nccl",
                  peers=None, comm=None, **kw):
    """Reciprocal matching of one pair (or a stack) with the target columns
    sharded over the ranks of `group` (torch.distributed; NCCL on GPUs).

    d1, d2: float32 CUDA tensors [P, H, W, d] (or [H, W, d]) on this rank's
    device, identical on every rank.  Returns (matches [P, samples, 3] int32
    device tensor, counts [P] int32 device tensor, per-pair stats) -- equal on
    every rank and to the unsharded result.
    """
    import torch
    import torch.distributed as dist

    from . import _fastnn

    if d1.dim() == 3:
        d1, d2 = d1.unsqueeze(0), d2.unsqueeze(0)
    P, H, W, D = d1.shape
    samples = ((H + stride - 1) // stride) * ((W + stride - 1) // stride)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    pairs = torch.empty((P, samples, 3), dtype=torch.int32, device=d1.device)
    counts = torch.empty((P,), dtype=torch.int32, device=d1.device)
    stream = torch.cuda.current_stream(d1.device).cuda_stream
    if transport == "p2p":
        own = peers is None
        if own:
            peers = PeerTransport(P * samples, group)
        if peers.broken:
            raise RuntimeError("PeerTransport unusable after a failed call (" + peers.broken +
                               "); its barrier counters are out of step: create a new one")
        try:
            stats, peers.seq = _fastnn.reciprocal_match_p2p_device(
                d1.data_ptr(), d2.data_ptr(), P, H, W, D, pairs.data_ptr(), counts.data_ptr(),
                2 * peers.nkeys, rank, peers.peer_keys, peers.peer_flags, peers.seq, backend=backend,
                stride=stride, metric=metric, stream=stream, **kw)
        except Exception as e:
            # the device counters advanced but barrier_seq did not come back:
            # a reused transport would compute stale barrier targets
            peers.broken = str(e)[:200]
            raise
        finally:
            if own:
                torch.cuda.synchronize(d1.device)
                if world > 1:
                    dist.barrier(group=group)  # nobody unmaps while a peer may still push
                peers.close()
        return pairs, counts, stats
    keys = torch.empty((P * samples,), dtype=torch.int64, device=d1.device)
    if transport == "nccl-native":
        # the library all-reduces with its own NCCL communicator
        own = comm is None
        if own:
            comm = NativeComm(group)
        try:
            stats = _fastnn.reciprocal_match_sharded_device(
                d1.data_ptr(), d2.data_ptr(), P, H, W, D, pairs.data_ptr(), counts.data_ptr(), keys.data_ptr(),
                keys.numel(), comm.rank, comm.world, None, backend=backend, stride=stride, metric=metric,
                stream=stream, comm=comm.handle, **kw)
        finally:
            if own:
                torch.cuda.synchronize(d1.device)
                comm.close()
        return pairs, counts, stats

    def reduce(count):
        dist.all_reduce(keys[:count], op=dist.ReduceOp.MIN, group=group)

    stats = _fastnn.reciprocal_match_sharded_device(
        d1.data_ptr(), d2.data_ptr(), P, H, W, D, pairs.data_ptr(), counts.data_ptr(), keys.data_ptr(),
        keys.numel(), rank, world, reduce, backend=backend, stride=stride, metric=metric, stream=stream, **kw)
    return pairs, counts, stats
