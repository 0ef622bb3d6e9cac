"""Kernel-by-kernel table (time, dram read/write) of the last pipeline run in an ncu --csv launch log.
usage: python tools/launch_table.py gpurun_out/vox_launches.csv [first-kernel-substring]"""
import csv, collections, sys
path = sys.argv[1]; first = sys.argv[2] if len(sys.argv) > 2 else "mark_starts"
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; kn = h.index("Kernel Name"); mn = h.index("Metric Name"); mv = h.index("Metric Value"); idc = h.index("ID"); mu = h.index("Metric Unit")
d = collections.OrderedDict()
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
for r in rows[hi + 1:]:
    if len(r) <= mv: continue
    e = d.setdefault(r[idc], {"k": r[kn].split("(")[0][-44:]})
    e[r[mn]] = float(r[mv].replace(",", "")) * scale.get(r[mu], 1.0)
ks = list(d.values())
st = [i for i, e in enumerate(ks) if first in e["k"]][-1]
tot = 0
for e in ks[st:]:
    t = e.get("gpu__time_duration.sum", 0); tot += t
    print(f"{e['k']:46s} {t:8.1f} us  rd {e.get('dram__bytes_read.sum', 0):8.1f} MB  wr {e.get('dram__bytes_write.sum', 0):8.1f} MB")
print("total us %.1f" % tot)
