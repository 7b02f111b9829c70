"""Summarise an ncu CSV (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum]) of a
bench.py run into (1) a per-kernel launch list (share of the step) and (2) per-launch DRAM traffic JSON keyed
by the bench's kernel ids.  Usage: ncu_summary.py <ncu.csv> <steps> <out_prefix> [command text]"""
import collections
import csv
import json
import sys

path, steps, prefix = sys.argv[1], int(sys.argv[2]), sys.argv[3]
cmd = sys.argv[4] if len(sys.argv) > 4 else ""
rows = [r for r in csv.reader(open(path)) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    per[r[ii]][r[mi]] = v
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for lid, m in per.items():
    a = agg[names[lid]]
    a[0] += 1
    t = m.get("gpu__time_duration.sum", 0.0)
    a[1] += t / 1e6 if t > 1e3 else t   # ns -> ms (ncu reports ns or ms depending on version)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
with open(prefix + "_launches.txt", "w") as f:
    f.write("ncu launch list (gpu__time_duration.sum, --clock-control none); launches are serialised and cold-cache\n")
    f.write("under ncu, so the SHARE of each kernel is the comparable figure, not the absolute time.\n")
    if cmd:
        f.write("command: " + cmd + "\n")
    f.write(f"\n{'kernel':40s} {'launches':>8s} {'ms total':>10s} {'ms/step':>9s} {'share':>6s}\n")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{k:40s} {a[0]:8d} {a[1]:10.2f} {a[1] / steps:9.2f} {100 * a[1] / tot:5.1f}%\n")
    f.write(f"total {tot:.1f} ms over {steps} steps = {tot / steps:.1f} ms/step\n")
ids = {"mg::k_bin_expand2": "bin_expand", "mg::k_bin_expand": "bin_expand", "mg::k_bin_big": "bin_big",
       "mg::k_bin_reduce": "bin_reduce", "mg::k_heavy_sym2": "sym_heavy", "mg::k_heavy_symbolic": "sym_heavy",
       "mg::k_rows_block<1>": "num_block", "mg::k_rows_block<0>": "sym_block"}
tj = {"source": prefix + "_launches.txt", "kernels": {}}
for k, a in agg.items():
    if k in ids and a[2] > 0:
        tj["kernels"][ids[k]] = {"dram_bytes_per_launch": int(a[2] / a[0]), "ms_per_launch_ncu": round(a[1] / a[0], 3),
                                 "launches": a[0]}
json.dump(tj, open(prefix + "_traffic.json", "w"), indent=1)
print(open(prefix + "_launches.txt").read())
print(json.dumps(tj, indent=1))
