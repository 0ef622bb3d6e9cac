"""Headline metrics + stall reasons of the first kernel in an ncu report (developer tool)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, r = rows[0], rows[1], rows[2]
keys = ['gpu__time_duration.sum', 'smsp__issue_active.avg.pct', 'smsp__inst_executed.sum', 'thread_inst_executed_per_inst',
        'sm__warps_active.avg.pct', 'registers_per_thread', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'l1tex__t_sector_hit_rate', 'lts__t_sector_hit_rate', 'shared_mem_per_block', 'sass__inst_executed_local']
for i, h in enumerate(hdr):
    if 'issue_stalled' in h and 'per_issue_active' in h:
        if float(r[i]) > 0.05: print('  stall', h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), r[i])
    elif any(k in h for k in keys) and 'pct_of_peak_sustained_elapsed' not in h and 'per_second' not in h and 'Triage' not in h:
        print(h, units[i], r[i])
