"""Summarise an ncu report: key metrics, stall reasons and the hottest SASS lines (by stall samples), per kernel."""
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
        "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__occupancy_limit_registers",
        "sm__maximum_warps_per_active_cycle_pct"]
stall_prefix = "smsp__average_warp_latency_issue_stalled_"
for v in vals:
    print("kernel:", v[hdr.index("Kernel Name")][:80])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:70s} {v[i]:>20s} {units[i]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                st.append((float(v[i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1.0
    print("  stalls:", ", ".join(f"{n} {100 * x / tot:.1f}%" for x, n in sorted(st, reverse=True)[:8]))

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = list(csv.reader(io.StringIO(src)))
blocks, cur = [], None
for r in lines:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "?", "hdr": None, "body": []}
        blocks.append(cur)
    elif cur is not None and cur["hdr"] is None:
        cur["hdr"] = r
    elif cur is not None:
        cur["body"].append(r)
for b in blocks:
    h = b["hdr"]
    si = h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in b["body"] if len(r) > si and r[si].isdigit()]
    tot = sum(int(r[si]) for r in body)
    print("==", b["name"][:70], "samples", tot)
    body.sort(key=lambda r: -int(r[si]))
    for r in body[:top]:
        print(f"{int(r[si]):7d} {100.0 * int(r[si]) / max(tot, 1):5.1f}%  {r[0][-5:]}  {r[1].strip()[:90]}")
