"""Summarise ncu --page source (SASS) stall samples per instruction for each profiled kernel."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
kern = None
hdr = None
data = {}
for r in rows:
    if len(r) >= 2 and r[0] == "Kernel Name":
        kern = r[1]
        data[kern] = []
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and kern and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        data[kern].append(d)
for k, ins in data.items():
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in ins)
    print(f"=== {k[:80]}  samples={tot}")
    idx = sorted(range(len(ins)), key=lambda i: -int(ins[i]["Warp Stall Sampling (All Samples)"] or 0))[:top]
    for i in sorted(idx):
        d = ins[i]
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        reasons = {h[6:]: int(d[h] or 0) for h in d if h.startswith("stall_") and "Not Issued" not in h}
        topr = sorted(reasons.items(), key=lambda x: -x[1])[:2]
        print(f"{i:5d} {100*s/max(tot,1):5.1f}%  {d['Source'].strip()[:60]:60s} {topr}")
