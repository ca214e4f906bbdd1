"""Summarise an SSQA_TC_TRACE dump: per-row-tile durations of MMA, loader, epilogue (block 0)."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.int64).reshape(4, -1, 2)
n = int((a[0, :, 1] > 0).sum())
t0 = a[0, 0, 0]
mma_s, mma_e = a[0, :n, 0] - t0, a[0, :n, 1] - t0
ld_s, ld_e = a[1, :n, 0] - t0, a[1, :n, 1] - t0
ep_s, ep_e = a[2, :n, 0] - t0, a[2, :n, 1] - t0
ep_rdy = a[3, :n, 0] - t0
print(f"row tiles traced: {n}")
print("rt   mma[start,dur]   ld[start,dur]   epi[start, wait, work]   (cycles)")
for r in list(range(min(n, 45))):
    print(f"{r:4d} {mma_s[r]:9d} {mma_e[r]-mma_s[r]:6d} | {ld_s[r]:9d} {ld_e[r]-ld_s[r]:6d} | "
          f"{ep_s[r]:9d} {ep_rdy[r]-ep_s[r]:6d} {ep_e[r]-ep_rdy[r]:6d}")
if n > 4:
    w = slice(2, n)
    print("mean mma dur", np.mean(mma_e[w] - mma_s[w]), " mean epi work", np.mean(ep_e[w] - ep_rdy[w]),
          " mean epi wait", np.mean(ep_rdy[w] - ep_s[w]), " total", ep_e[n - 1])
