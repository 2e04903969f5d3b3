"""Summarise a K3 clock trace (FNL_TC_DEBUG=16): per-tile loader issue,
MMA wait start/end and epilogue wake times of CTA 0."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(6, 4096).astype(np.int64)
n = int((t[1] > 0).sum())
t0 = t[:, 0][t[:, 0] > 0].min()
L, M0, M1, E, R, C = (t[i, :n] - t0 for i in range(6))
print(f"tiles traced {n}")
for k in list(range(0, 12)) + list(range(n // 2, n // 2 + 6)):
    print(f"k={k:4d} load_issue={L[k]:8d} mma_wait={M0[k]:8d}..{M1[k]:8d} (waited {M1[k]-M0[k]:6d}) epi_wake={E[k]:8d} released={R[k]-E[k]:5d} computed={C[k]-R[k]:5d}")
d = np.diff(M1[10:n])
print(f"steady: MMA issue interval median {np.median(d):.0f} cyc, mean {d.mean():.0f}; "
      f"MMA wait median {np.median(M1[10:n]-M0[10:n]):.0f}; load lead (mma_ready - load_issue) median {np.median(M1[10:n]-L[10:n]):.0f}; "
      f"epi wake - mma issue median {np.median(E[10:n]-M1[10:n]):.0f}; epi load {np.median(R[10:n]-E[10:n]):.0f}, compute {np.median(C[10:n]-R[10:n]):.0f}, next wake wait {np.median(E[11:n]-C[10:n-1]):.0f}")
