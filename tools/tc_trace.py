"""Summarise a K3 clock trace (FNL_TC_DEBUG=16) of CTA 0.

Rows (clock64 stamps per tile k): 0 loader issue; 1 issuer of query tile 0
before its "B landed" wait; 2 / 3 the same issuer after the "half 0 / half 1
drained" waits (= MMA issue of that half); 4 / 5 wake / release of each of the
four epilogue warps (TMEM lane quadrants) of chain (query tile 0, half 0),
[quad][1024]; 6 trees + key insert done (one warp)."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(7, 4096).astype(np.int64)
n = int((t[2] > 0).sum())
t0 = t[0][t[0] > 0].min()
L, M0, I0, I1, _, _, C = (t[i] - t0 for i in range(7))
W = t[4].reshape(4, 1024) - t0
R = t[5].reshape(4, 1024) - t0
nq = min(n, 1024)
print(f"tiles traced {n}")
for k in list(range(0, 6)) + list(range(nq // 2, nq // 2 + 8)):
    print(f"k={k:4d} load={L[k]:8d} iss_wait={M0[k]:8d} h0_issue={I0[k]:8d} h1_issue={I1[k]:8d} "
          f"wake={' '.join(f'{w:8d}' for w in W[:, k])} rel={' '.join(f'{r:8d}' for r in R[:, k])} done={C[k]:8d}")
s = slice(10, nq - 1)
k = np.arange(10, nq - 1)
d = np.diff(I0[10:nq])
wake_min, wake_max = W[:, s].min(0), W[:, s].max(0)
rel_max = R[:, s].max(0)
print(f"steady (k 10..{nq - 1}): h0 issue interval median {np.median(d):.0f} cyc; h1 - h0 issue {np.median(I1[s] - I0[s]):.0f}")
print(f"  h0 issue -> first quad wake {np.median(wake_min - I0[s]):.0f}; wake skew (last - first) {np.median(wake_max - wake_min):.0f}; "
      f"per-quad wake -> release {', '.join(f'{np.median(R[q, s] - W[q, s]):.0f}' for q in range(4))}")
print(f"  per-quad wake - h0 issue {', '.join(f'{np.median(W[q, s] - I0[s]):.0f}' for q in range(4))}")
print(f"  last release -> next h0 issue {np.median(I0[k + 1] - rel_max):.0f}; issuer reaches tile k+1 (after h1 of k) - last h0 release {np.median(M0[k + 1] - rel_max):.0f}")
print(f"  quad3 release -> trees done {np.median(C[s] - R[3, s]):.0f}; trees done -> next wake {np.median(W[3, 11:nq] - C[10:nq - 1]):.0f}")
