"""Key ncu metrics per profiled kernel (details page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = rows[0]
ki, mi, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
idi = hdr.index("ID")
want = ["Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "L2 Hit Rate", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Cluster Size"]
seen = {}
for r in rows[1:]:
    if r[mi] in want:
        seen.setdefault((r[idi], r[ki][:60]), []).append(f"{r[mi]}={r[vi]} {r[ui]}")
for (i, k), v in seen.items():
    print(f"[{i}] {k}")
    for x in v:
        print("    " + x)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_tex.sum", "gpu__time_duration.sum"]
for vals in rr[2:]:
    print("  raw:", ", ".join(f"{k.split('.')[0]}={vals[h.index(k)]}" for k in keys if k in h))
