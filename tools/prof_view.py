"""Summarise a PNCE_DIAG_PROF cycle-accounting dump (tools/bin/libpnce_diag_prof*.so)."""
import sys
import numpy as np

d = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(1024, 16).astype(np.float64)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 148
d = d[:n]
lead = d[0::2]
tot = lead[:, 12].mean() or (lead[:, 2] + lead[:, 3] + lead[:, 4]).mean()
names = {0: "Bprod wait empty", 1: "Bprod issue", 2: "MMA wait tempty", 3: "MMA wait full", 4: "MMA issue",
         5: "raw wait empty", 6: "raw issue", 7: "conv wait empty", 8: "conv wait raw", 9: "conv convert",
         10: "epi wait tfull", 11: "epi drain", 13: "conv read+bar wait", 14: "conv store-done wait",
         15: "Bprod scratch wait"}
print(f"MMA-thread total cycles (mean over leaders): {tot:.3e}")
for i, nm in names.items():
    v = (lead if i in (2, 3, 4) else d)[:, i].mean()
    print(f"  {i:2d} {nm:18s} {v:12.4e}  {100 * v / tot:6.1f}%")
