"""torchrun --nproc-per-node N tools/shard_check.py [H W metric]: the sharded
matcher on N ranks (gloo if all ranks share one GPU, else NCCL) vs the
unsharded tensor backend."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    H, W = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (128, 96)
    metric = sys.argv[3] if len(sys.argv) > 3 else "dot"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    ngpu = torch.cuda.device_count()
    dev = rank % ngpu
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl" if ngpu >= world else "gloo")
    import paper_2503_10017_b200 as fnl
    from paper_2503_10017_b200.shard import match_sharded
    fnl.set_device(dev)
    D1 = fnl.gen_random(H, W, 24, 606)
    D2 = fnl.gen_random(H, W, 24, 607)
    want, _ = fnl.reciprocal_match(D1, D2, backend="tensor", metric=metric)
    pairs, counts, stats = match_sharded(torch.from_numpy(D1).cuda(), torch.from_numpy(D2).cuda(), metric=metric)
    torch.cuda.synchronize()
    n = int(counts[0].item())
    got = pairs[0, :n].cpu().numpy().astype(np.uint32)
    ok = np.array_equal(got, want)
    print(f"rank {rank}: {n} matches, equal={ok}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
