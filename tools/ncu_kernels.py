"""Headline metrics + top stall reasons + hottest source lines of every kernel in an ncu report."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'launch__registers_per_thread', 'smsp__inst_executed.sum', 'l1tex__t_sector_hit_rate.pct',
        'lts__t_sector_hit_rate.pct', 'sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active',
        'lts__t_sectors.sum', 'l1tex__t_sectors.sum']
stall = [k for k in h if 'issue_stalled' in k and 'per_issue_active' in k]
names = []
for r in rows[2:]:
    d = dict(zip(h, r))
    names.append(d['Kernel Name'])
    print('=====', d['Kernel Name'][:60])
    for k in keys:
        print(f'  {k:66s} {d.get(k)} {rows[1][h.index(k)] if k in h else ""}')
    st = sorted(((float(d[k]), k.split("issue_stalled_")[1].split("_per")[0]) for k in stall), reverse=True)[:6]
    print('  stalls:', ' '.join(f'{n}={v:.2f}' for v, n in st))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
# the source page prints one table per kernel
blocks = src.split('"#","Source"')
for bi, blk in enumerate(blocks[1:]):
    rws = list(csv.reader(('"#","Source"' + blk).splitlines()))
    hh = rws[0]
    try:
        ci = hh.index("# Samples") if "# Samples" in hh else [i for i, x in enumerate(hh) if "Sampl" in x][0]
    except Exception:
        continue
    ii = [i for i, x in enumerate(hh) if x.startswith("Instructions Executed")]
    tot = 0; lines = []
    for r in rws[1:]:
        if len(r) <= ci: continue
        try: v = float(r[ci])
        except ValueError: continue
        tot += v; lines.append((v, r[0], r[1].strip()[:110]))
    print(f"----- kernel {bi} ({names[bi][:40] if bi < len(names) else '?'}): samples {tot:.0f}")
    for v, ln, txt in sorted(lines, reverse=True)[:top]:
        print(f"   {v/max(tot,1)*100:5.1f}%  L{ln}: {txt}")
