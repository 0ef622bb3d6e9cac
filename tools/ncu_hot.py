"""Hottest CUDA source lines of ONE kernel of an ncu report captured with --import-source on (developer tool).
usage: python tools/ncu_hot.py report.ncu-rep <kernel regex> [top_n]"""
import csv, subprocess, sys, collections
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; data = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        ci = {n: i for i, n in enumerate(r)}
        continue
    if hdr and len(r) >= 10 and r[0] != "":
        try:
            data.append((int(r[ci["# Samples"]]), int(r[ci["Instructions Executed"]]), int(r[ci["Thread Instructions Executed"]]),
                         cur, r[0], r[1], int(r[ci["stall_long_sb"]]), int(r[ci["stall_math"]]) if "stall_math" in ci else 0))
        except Exception:
            pass
tot = sum(d[0] for d in data) or 1; toti = sum(d[1] for d in data) or 1; tott = sum(d[2] for d in data)
print(f"kernel ~ {pat}: samples {tot}, warp inst {toti}, avg threads/inst {tott / toti:.2f}")
for d in sorted(data, reverse=True)[:top]:
    print(f"{100*d[0]/tot:5.1f}% smp {100*d[1]/toti:5.1f}% inst thr/inst {d[2]/max(d[1],1):5.1f} longsb {100*d[6]/max(d[0],1):3.0f}% {d[3]}:{d[4]}: {d[5].strip()[:110]}")
