"""Executed code footprint of a kernel from an ncu report's SASS page (developer tool).
usage: python tools/ncu_footprint.py report.ncu-rep"""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("# Samples")
ins = []
for r in rows[2:]:
    if len(r) <= ie or not r[ia].startswith("0x"):
        continue
    ins.append((int(r[ia], 16), int(r[ie]), int(r[isamp]), r[1].strip()))
base = ins[0][0]
tot = sum(i[1] for i in ins)
print(f"{len(ins)} SASS instructions = {len(ins)*16/1024:.1f} KB; executed warp-inst {tot/1e9:.2f} G")
for thr in (0, 1e5, 1e6, 1e7, 3e7):
    sel = [i for i in ins if i[1] > thr]
    print(f"  executed > {thr:9.0f} times: {len(sel):5d} instr = {len(sel)*16/1024:6.1f} KB, carrying {100*sum(i[1] for i in sel)/tot:5.1f}% of the executed instructions")
# 2 KB pages: executed share and samples
page = {}
for a, e, s, t in ins:
    k = (a - base) // 2048
    p = page.setdefault(k, [0, 0, 0]); p[0] += e; p[1] += s; p[2] += 1
ts = sum(p[1] for p in page.values())
print("2KB page: %exec %samples")
for k in sorted(page):
    p = page[k]
    print(f"  {k*2:4d} KB  {100*p[0]/tot:5.1f}%  {100*p[1]/ts:5.1f}%")
