import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2503_10017_b200 as fnl
q = torch.randn((2,16,768,64), device='cuda').half(); k = torch.randn_like(q); v = torch.randn_like(q)
for _ in range(3): fnl.flashmatch(q,k,v)
torch.cuda.synchronize()
