"""Summarise an ncu report: key metrics and the hottest SASS lines (by stall samples)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for v in vals:
    print("kernel:", v[hdr.index("Kernel Name")][:80])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:70s} {v[i]:>20s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = list(csv.reader(io.StringIO(src)))
h = lines[1] if lines and lines[0] and lines[0][0] == "Kernel Name" else lines[0]
body = lines[2:] if h is lines[1] else lines[1:]
si = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[si] or 0) for r in body if len(r) > si)
body = [r for r in body if len(r) > si]
body.sort(key=lambda r: -int(r[si] or 0))
print("total samples", tot)
for r in body[:top]:
    print(f"{int(r[si]):7d} {100.0 * int(r[si]) / max(tot, 1):5.1f}%  {r[0][-6:]}  {r[1].strip()[:90]}")
