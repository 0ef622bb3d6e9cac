"""Per-kernel times of one wavefront frame from an ncu launch list (developer tool)."""
import csv, collections, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/wf_launches.csv"
which = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; kn = h.index("Kernel Name"); mv = h.index("Metric Value")
seq = []
for r in rows[hi + 1:]:
    if len(r) <= mv: continue
    name = r[kn].split("(")[0].split("::")[-1]
    if "wf_exact_kernel" in r[kn]:
        name = "wf_exact<%s>" % r[kn].split("<")[-1].split(">")[0]
    seq.append((name, float(r[mv]) / 1e3))
frames = []; cur = None
for k, t in seq:
    if k == "wf_begin_kernel":
        cur = []; frames.append(cur)
    if cur is not None and k.startswith("wf_"): cur.append((k, t))
f = frames[which] if len(frames) > which else frames[-1]
print("kernels in frame:", len(f), "sum ms %.3f" % (sum(t for _, t in f) / 1e3))
agg = collections.OrderedDict()
for k, t in f: agg.setdefault(k, []).append(t)
for k, v in agg.items():
    print(f"{k:22s} n={len(v):3d} total {sum(v):9.1f} us   per-iter:", " ".join(f"{x:.0f}" for x in v[:20]))
