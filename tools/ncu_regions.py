"""Instruction / stall-sample totals of an ncu report grouped by source-line ranges.
Usage: ncu_regions.py <rep> <file> <start:name,start:name,...> [kernel regex]"""
import csv, io, subprocess, sys, collections
rep, fsel, spec = sys.argv[1], sys.argv[2], sys.argv[3]
kf = ["-k", "regex:" + sys.argv[4]] if len(sys.argv) > 4 else []
regs = sorted((int(a.split(":")[0]), a.split(":")[1]) for a in spec.split(","))
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname, hdr = "?", None
agg = collections.defaultdict(lambda: [0, 0])
other = collections.defaultdict(lambda: [0, 0])
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or row[0] in ("", "Function Name"): continue
    try:
        smp = int(row[hdr.index("Warp Stall Sampling (All Samples)")]); inst = int(row[hdr.index("Instructions Executed")]); ln = int(row[0])
    except (ValueError, IndexError): continue
    if fname == fsel:
        name = "pre"
        for s, nm in regs:
            if ln >= s: name = nm
        agg[name][0] += inst; agg[name][1] += smp
    else:
        other[fname][0] += inst; other[fname][1] += smp
ti = sum(v[0] for v in agg.values()) + sum(v[0] for v in other.values()) or 1
ts = sum(v[1] for v in agg.values()) + sum(v[1] for v in other.values()) or 1
for s, nm in [(0, "pre")] + regs:
    v = agg[nm]; print(f"{nm:14s} {100*v[0]/ti:5.1f}% inst {100*v[1]/ts:5.1f}% smp")
for f, v in sorted(other.items(), key=lambda x: -x[1][0]): print(f"[{f}] {100*v[0]/ti:5.1f}% inst {100*v[1]/ts:5.1f}% smp")
