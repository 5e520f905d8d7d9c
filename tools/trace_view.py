import sys
import numpy as np
S, MAXJ = 16, 512
t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(2, S, MAXJ).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1000.0, np.nan)   # us
names = {0: "Bprod empty ok", 1: "MMA tempty ok(tile)", 2: "MMA full ok", 3: "MMA issued", 4: "fwd local full",
         5: "fwd arrived", 6: "raw issue", 7: "conv raw ok", 8: "conv empty ok", 9: "conv arrive",
         10: "epi tfull(tile)", 11: "epi w8 done(tile)", 12: "epi w15 done(tile)", 13: "kernel entry",
         14: "prologue done", 15: "roles done"}
KB = int(sys.argv[2]) if len(sys.argv) > 2 else 16
jobs = int(np.sum(~np.isnan(t[0, 2])))
print("jobs traced", jobs)
for j in list(range(0, 40)):
    row = []
    for cta in (0, 1):
        for sl in (0, 6, 7, 8, 9, 4, 5, 2, 3):
            v = t[cta, sl, j]
            if not np.isnan(v):
                row.append(f"c{cta}.{sl}={v:7.2f}")
    print(f"j{j:3d} kb{j%KB:2d} " + " ".join(row))
print("kernel:", " ".join(f"c{c}.{sl}={t[c, sl, 0]:7.2f}" for c in (0, 1) for sl in (13, 14, 15)
                          if not np.isnan(t[c, sl, 0])))
print("tiles:")
for ti in range(0, 6):
    print(ti, " ".join(f"c{c}.{sl}={t[c, sl, ti]:7.2f}" for c in (0, 1) for sl in (1, 10, 11, 12) if not np.isnan(t[c, sl, ti])))
d = np.diff(t[0, 3, :jobs])
print("MMA issue interval us: median %.3f mean %.3f" % (np.nanmedian(d), np.nanmean(d)))
print("MMA full-wait->issued us median %.3f" % np.nanmedian(t[0, 3, :jobs] - t[0, 2, :jobs]))
