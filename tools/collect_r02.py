"""Copy the final round-2 measurement (tools/gpu_final_r02.sh outputs in gpurun_out/) into
profiles/r02/ and refresh profiles/ncu_traffic.json (per-frame-set DRAM bytes at 4096)."""
import csv
import json
import os
import shutil
import subprocess
import sys

G, P = "gpurun_out", "profiles/r02"
os.makedirs(P, exist_ok=True)


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


bench = last_json(f"{G}/bench.log")
json.dump(bench, open(f"{P}/bench_final.json", "w"), indent=1)
ref = last_json(f"{G}/bench_ref.log")
json.dump(ref, open(f"{P}/bench_reference_arm.json", "w"), indent=1)
shutil.copy(f"{G}/host.txt", f"{P}/gpu_host.txt")
shutil.copy(f"{G}/launches.csv", f"{P}/ncu_launches.csv")
out = subprocess.run([sys.executable, "tools/ncu_launches.py", f"{G}/launches.csv",
                      "ncu launch list of `bench.py --frames 10000 --steps 2 --warmup 3 --no-e2e --no-cpu` "
                      "(cold-cache, serialised; compare shares)"], capture_output=True, text=True).stdout
open(f"{P}/ncu_launches.txt", "w").write(out)
# DRAM traffic at 4096 frame-sets
rows = list(csv.reader(open(f"{G}/traffic.csv")))
st = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[st]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[st + 1:]:
    per.setdefault((int(r[ii]), r[ki].split("(")[0].replace("void <unnamed>::", "")), {})[r[mi]] = \
        float(r[vi].replace(",", ""))
lines, traffic = [], {}
names = {"k_correlate<2, 0, 0, 0>": "fused", "k_correlate<2, 1, 1, 0>": "scored",
         "k_correlate<2, 0, 1, 1>": "tensor16", "k_correlate<0, 0, 1, 0>": "packed"}
F = 4096
for (i, k), m in sorted(per.items()):
    rd, wr = m.get("dram__bytes_read.sum", 0) / F, m.get("dram__bytes_write.sum", 0) / F
    lines.append(f"[{i}] {k:28s} read {rd/1e6:7.3f} MB  write {wr/1e6:7.3f} MB  total {(rd+wr)/1e6:7.3f} MB per frame-set"
                 f"  {m.get('gpu__time_duration.sum', 0)/F/1e3:6.3f} us  tensor {m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):5.1f} %")
    if k in names and names[k] not in traffic:
        traffic[names[k]] = (rd, wr)
open(f"{P}/ncu_traffic.txt", "w").write("ncu --metrics dram__bytes_read/write.sum at 4096 frame-sets per launch "
                                       "(bench.py --frames 4096 --gemm-frames 4096 --scored-frames 4096)\n" + "\n".join(lines) + "\n")
tj = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, bench.py at 4096 "
                "frame-sets per launch (r02 final, profiles/r02/ncu_traffic.txt)"}
for name, (rd, wr) in traffic.items():
    tj[f"k_correlate_{name}_dram_read_per_frame"] = rd
    tj[f"k_correlate_{name}_dram_write_per_frame"] = wr
    tj[f"k_correlate_{name}_dram_bytes_per_frame"] = rd + wr
json.dump(tj, open("profiles/ncu_traffic.json", "w"), indent=1)
if os.path.exists(f"{G}/prof_full.ncu-rep"):
    out = subprocess.run([sys.executable, "tools/ncu_summary.py", f"{G}/prof_full.ncu-rep"], capture_output=True,
                         text=True).stdout
    open(f"{P}/ncu_full_k_correlate.txt", "w").write(out)
print(open(f"{P}/ncu_traffic.txt").read())
print(open(f"{P}/ncu_launches.txt").read())
