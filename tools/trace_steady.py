"""Steady-state timeline of the fused kernel (trace build): jobs of tiles 4-7 of the first CTA pair.
Columns per job: raw issue (6), conv raw ok (7), conv empty ok (8), conv arrive (9), MMA full ok (2),
MMA issued (3); per tile: MMA tempty ok (1), epi tfull (10), epi done (11/12)."""
import sys
import numpy as np
S, MAXJ = 16, 512
t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(2, S, MAXJ).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1000.0, np.nan)
KB = 16
for tile in range(3, 8):
    print(f"tile {tile}: tempty ok {t[0,1,tile]:.2f}  epi tfull {t[0,10,tile]:.2f}  epi done {t[0,11,tile]:.2f}/{t[0,12,tile]:.2f}")
    for kb in range(KB):
        j = tile * KB + kb
        vals = " ".join(f"{n}={t[0,sl,j]:7.2f}" for n, sl in (("raw", 6), ("rawok", 7), ("emp", 8), ("arr", 9), ("full", 2), ("iss", 3)))
        print(f"   kb{kb:2d} {vals}")
