"""Hottest CUDA source lines of a kernel by instruction share AND by stall samples (developer tool).
usage: python tools/ncu_hot2.py report.ncu-rep <kernel regex> [top_n]"""
import csv, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; data = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) > 5 and r[0] == "Line No":
        hdr = r; ci = {n: i for i, n in enumerate(r)}; continue
    if hdr and len(r) >= 10 and r[0] != "":
        try:
            data.append((int(r[ci["Instructions Executed"]]), int(r[ci["# Samples"]]), int(r[ci["Thread Instructions Executed"]]), cur, r[0], r[1]))
        except Exception:
            pass
toti = sum(d[0] for d in data) or 1; tots = sum(d[1] for d in data) or 1
print(f"== {pat}: warp inst {toti}, samples {tots}, threads/inst {sum(d[2] for d in data) / toti:.1f}")
seen = set()
for key in (0, 1):
    print("  -- by " + ("instructions" if key == 0 else "stall samples"))
    for d in sorted(data, key=lambda d: -d[key])[:top]:
        print(f"  {100*d[0]/toti:5.1f}% inst {100*d[1]/tots:5.1f}% smp thr {d[2]/max(d[0],1):5.1f} {d[3]}:{d[4]}: {d[5].strip()[:105]}")
