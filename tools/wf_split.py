"""Per-iteration / per-kernel split of the second frame in a raw ncu launch list (developer tool)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
frames = []; cur = []
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].split('::')[-1].replace('wf_', '').replace('_kernel', '')
    if 'wf_exact' in r[ki]: name = 'exact'
    v = float(r[vi].replace(',', '')); v = v / 1e3 if r[ui] == 'ns' else (v * 1e3 if r[ui] == 'ms' else v)
    if name == 'begin':
        if cur: frames.append(cur)
        cur = []
    cur.append((name, v))
frames.append(cur)
fi = int(sys.argv[2]) if len(sys.argv) > 2 else 1
f = frames[fi] if len(frames) > fi else frames[0]
print("frames:", len(frames), "showing", fi)
tot = collections.OrderedDict(); it = 0; line = []
for name, v in f:
    tot[name] = tot.get(name, 0) + v
    line.append(f"{name}={v:.0f}")
    if name == 'next':
        print(it, ' '.join(line)); it += 1; line = []
print('totals (us):', ' '.join(f"{k}={v:.0f}" for k, v in tot.items()), ' frame', round(sum(tot.values())))
