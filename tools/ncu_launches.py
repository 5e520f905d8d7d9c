"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel launches,
mean duration and share of this library's kernels (cold-cache, serialised: compare shares)."""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
k_i, v_i, m_i = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[m_i] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"<unnamed>::", "", r[k_i]).split("(")[0]
    if not any(k in name for k in ("k_lfsr", "k_build_circulant", "k_pack_iq", "k_correlate", "k_t16_finish",
                                   "k_sat_finish", "k_draw_channel", "k_synth", "k_h_split", "k_build_bsyn")):
        continue
    agg.setdefault(name, []).append(float(r[v_i].replace(",", "")) / 1000.0)
tot = sum(sum(v) for v in agg.values())
print(sys.argv[2] if len(sys.argv) > 2 else "")
for k, v in agg.items():
    print(f"{k:28s} launches={len(v):3d} mean={sum(v)/len(v):9.1f} us  share_of_our_kernels={100*sum(v)/tot:5.1f}%")
