"""Shared-memory wavefronts (actual / ideal / excessive) per source line of one kernel in an ncu report."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, agg = "?", None, {}
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or row[0] in ("", "Function Name"): continue
    try:
        w = int(row[hdr.index("L1 Wavefronts Shared")] or 0); i = int(row[hdr.index("L1 Wavefronts Shared Ideal")] or 0)
        x = int(row[hdr.index("L1 Wavefronts Shared Excessive")] or 0)
    except (ValueError, IndexError): continue
    if w == 0: continue
    a = agg.setdefault((fname, row[0]), [0, 0, 0, row[1][:100]])
    a[0] += w; a[1] += i; a[2] += x
tw = sum(a[0] for a in agg.values()) or 1; tx = sum(a[2] for a in agg.values())
print(f"shared wavefronts {tw}, excessive {tx} ({100*tx/tw:.1f}%)")
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{100*a[2]/tw:5.1f}% excess  {100*a[0]/tw:5.1f}% of wavefronts  {f}:{ln:5s} {a[3]}")
