"""Per-source-line instruction and stall-sample totals from an ncu report (source page, cuda)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
fname = "?"
hdr = None
agg = []
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] == "" or row[0] == "Function Name":
        continue
    try:
        samples = int(row[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = int(row[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    agg.append((inst, samples, f"{fname}:{row[0]}", row[1][:90]))
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"total inst {ti}, samples {ts}")
print("--- by instructions")
for a in sorted(agg, reverse=True)[:top]:
    print(f"{100*a[0]/ti:5.1f}% inst {100*a[1]/ts:5.1f}% smp  {a[2]:24s} {a[3]}")
print("--- by stall samples")
for a in sorted(agg, key=lambda x: -x[1])[:top // 2]:
    print(f"{100*a[0]/ti:5.1f}% inst {100*a[1]/ts:5.1f}% smp  {a[2]:24s} {a[3]}")
