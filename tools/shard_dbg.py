import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2503_10017_b200 as fnl
from paper_2503_10017_b200 import _fastnn
D1 = fnl.gen_random(128, 96, 24, 606); D2 = fnl.gen_random(128, 96, 24, 607)
d1 = torch.from_numpy(D1).cuda(); d2 = torch.from_numpy(D2).cuda()
S = 16*12
keys = torch.empty(S, dtype=torch.int64, device='cuda')
pairs = torch.empty((1,S,3), dtype=torch.int32, device='cuda'); counts = torch.empty(1, dtype=torch.int32, device='cuda')
for rank in (0, 1):
    st = _fastnn.reciprocal_match_sharded_device(d1.data_ptr(), d2.data_ptr(), 1, 128, 96, 24, pairs.data_ptr(), counts.data_ptr(), keys.data_ptr(), S, rank, 2, lambda c: None, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    print(rank, counts.item(), st[0]["iterations"])
