"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): tensor + exact reciprocal matching at C1,
dense tensor NN, the sharded pass (1 process, no-op reduce), FlashMatch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_10017_b200 as fnl
from paper_2503_10017_b200 import _fastnn
D1 = fnl.gen_random(64, 48, 24, 21)
D2 = fnl.gen_random(64, 48, 24, 121)
for be in ("tensor", "single", "hybrid", "double"):
    m, _ = fnl.reciprocal_match(D1, D2, backend=be, metric="dot")
    print(be, m.shape[0])
print("l2", fnl.reciprocal_match(D1, D2, backend="tensor", metric="l2")[0].shape[0])
# several 256-row tile pairs (merge slices 0..3, ragged last slice) and the
# dim-dependent exact kernels (33..64 channels: 2 / 1 queries per thread)
E1 = fnl.gen_random(128, 96, 24, 31)
E2 = fnl.gen_random(128, 96, 24, 131)
print("tensor 700q", fnl.reciprocal_match(E1, E2, backend="tensor", metric="dot", stride=4)[0].shape[0])
F1 = fnl.gen_random(32, 24, 48, 41)
F2 = fnl.gen_random(32, 24, 48, 141)
for be in ("single", "hybrid"):
    print(be, "d48", fnl.reciprocal_match(F1, F2, backend=be, metric="dot", stride=4)[0].shape[0])
# ragged target count (3,500 = 54 x 64 + 44): the last sub-tile's padding masks
G1 = fnl.gen_random(50, 70, 24, 51)
G2 = fnl.gen_random(50, 70, 24, 151)
for be in ("single", "tensor"):
    print(be, "ragged", fnl.reciprocal_match(G1, G2, backend=be, metric="dot", stride=4)[0].shape[0])
r = fnl.nn_tensor(D1, D2, metric="dot")
print("dense", len(r["nearest"]))
print("mutual", fnl.mutual_nn_exact(D1, D2, metric="dot").shape[0])
d1 = torch.from_numpy(D1).cuda(); d2 = torch.from_numpy(D2).cuda()
S = 48
keys = torch.empty(S, dtype=torch.int64, device="cuda")
pairs = torch.empty((1, S, 3), dtype=torch.int32, device="cuda"); cnt = torch.empty(1, dtype=torch.int32, device="cuda")
for rank in (0, 1):
    _fastnn.reciprocal_match_sharded_device(d1.data_ptr(), d2.data_ptr(), 1, 64, 48, 24, pairs.data_ptr(),
                                            cnt.data_ptr(), keys.data_ptr(), S, rank, 2, lambda c: None)
q = torch.randn((1, 2, 200, 64), device="cuda").half(); k = torch.randn((1, 2, 150, 64), device="cuda").half()
o = fnl.flashmatch(q, k, k)
torch.cuda.synchronize()
print("flashmatch", tuple(o.shape), bool(torch.isfinite(o.float()).all()))
# the device batch API without stats: host-driven first call, then the loop
# captured and replayed as a CUDA graph (WHILE node) on the same buffers
dd1 = torch.from_numpy(np.stack([D1, E1[:64, :48]])).cuda().contiguous()
dd2 = torch.from_numpy(np.stack([D2, E2[:64, :48]])).cuda().contiguous()
gp = torch.empty((2, S, 3), dtype=torch.int32, device="cuda"); gc = torch.empty(2, dtype=torch.int32, device="cuda")
for _ in range(3):
    fnl.reciprocal_match_device(dd1.data_ptr(), dd2.data_ptr(), 2, 64, 48, 24, gp.data_ptr(), gc.data_ptr(),
                                backend="single", metric="dot", with_stats=False)
torch.cuda.synchronize()
print("graph replay", gc.tolist())
