"""Hottest CUDA source lines of one kernel in an ncu report.
usage: python tools/ncu_src.py report.ncu-rep kernel-regex [top_n]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]; top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "-s", skip, "-c", "1", "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; data = []; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if len(r) > 5 and r[0] == 'Line No': hdr = r; continue
    if hdr and len(r) >= 10 and r[0] != '':
        try: data.append((int(r[6]), int(r[7]), int(r[8]), cur, r[0], r[1]))
        except Exception: pass
tot = sum(d[0] for d in data) or 1; toti = sum(d[1] for d in data) or 1; tott = sum(d[2] for d in data)
print(kre, 'samples', tot, 'warp inst', toti, 'avg thr/inst %.2f' % (tott / toti))
for d in sorted(data, reverse=True)[:top]:
    print(f"{100*d[0]/tot:5.1f}% smp {100*d[1]/toti:5.1f}% inst thr/inst {d[2]/max(d[1],1):5.1f} {d[3]}:{d[4]}: {d[5].strip()[:105]}")
