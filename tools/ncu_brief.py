"""A few raw metrics of every kernel in an ncu report."""
import csv, sys, subprocess, io
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct', 'sm__inst_executed.avg.per_cycle_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'launch__grid_size', 'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct']
for r in rows[2:]:
    for w in want:
        if w in h: print(f"  {w}: {r[h.index(w)]} {rows[1][h.index(w)]}")
    for i, c in enumerate(h):
        if c.startswith('smsp__average_warps_issue_stalled') and c.endswith('per_issue_active.ratio') or c.startswith('smsp__average_warp_latency_issue_stalled'):
            try:
                if float(r[i]) > 0.3: print(f"    {c.replace('smsp__average_warps_issue_stalled_','').replace('smsp__average_warp_latency_issue_stalled_','lat_')}: {r[i]}")
            except ValueError: pass
