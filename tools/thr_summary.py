"""Per-kernel totals (ms, warp instructions, DRAM GB) of the ncu CSVs written by tools/gpu/run_threshold_sweep.sh."""
import collections, csv, sys
for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict); names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi: continue
        try: v = float(r[vi].replace(",", ""))
        except ValueError: continue
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("mg::", "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1; a[1] += m.get("gpu__time_duration.sum", 0.0) / 1e6   # ns -> ms (ncu csv prints ns)
        a[2] += m.get("smsp__inst_executed.sum", 0.0); a[3] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    print(path.split("/")[-1])
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:8]:
        print(f"  {k[:34]:34s} launches {a[0]:3d}  {a[1]:8.2f} ms  {a[2]/1e9:7.2f} G warp-inst  {a[3]/1e9:7.1f} GB dram")
