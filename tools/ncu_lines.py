"""Aggregate an ncu report's source page by CUDA source line (developer tool).
usage: python tools/ncu_lines.py report.ncu-rep [top_n]"""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; data = []; hdr = None; sass = []; cur_line = None
for r in rows:
    if len(r) > 8 and r[0] == '' and r[2].startswith('0x'):
        try: sass.append((cur, cur_line, int(r[7]), int(r[6])))
        except Exception: pass
        continue
    if len(r) == 2 and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if len(r) > 5 and r[0] == 'Line No': hdr = r; continue
    if hdr and len(r) >= 10 and r[0] != '':
        cur_line = r[0]
        try: data.append((int(r[6]), int(r[7]), int(r[8]), cur, r[0], r[1]))
        except Exception: pass
tot = sum(d[0] for d in data); toti = sum(d[1] for d in data); tott = sum(d[2] for d in data)
print('samples', tot, 'warp inst', toti, 'thread inst', tott, 'avg thr/inst %.2f' % (tott / toti))
for d in sorted(data, reverse=True)[:top]:
    print(f"{100*d[0]/tot:5.1f}% smp {100*d[1]/toti:5.1f}% inst thr/inst {d[2]/max(d[1],1):5.1f} {d[3]}:{d[4]}: {d[5].strip()[:100]}")
# per-file/region summary
import collections
reg = collections.Counter(); regi = collections.Counter()
for d in data:
    reg[d[3]] += d[0]; regi[d[3]] += d[1]
for k in reg: print(k, '%.1f%% samples %.1f%% inst' % (100*reg[k]/tot, 100*regi[k]/toti))
# stage shares (line ranges of the current lvx_render.cu / lvx_geom.cuh)
def stage(d):
    f, ln = d[3], int(d[4])
    if f == 'lvx_geom.cuh':
        if ln < 190: return 'exact tests (tube/sphere)'
        if ln < 292: return 'dda'
        return 'shade/AO/trilinear'
    if f == 'lvx_render.cu':
        rng = STAGES
        for name, lo, hi in rng:
            if lo <= ln <= hi: return name
    return 'other'
import re
src = open('paper_1801_01155_b200/csrc/lvx_render.cu').read().split('\n')
def find(pat):
    for i, l in enumerate(src):
        if pat in l: return i + 1
    return 0
STAGES = [('accumulate_hit (dedup+blend)', find('__device__ __forceinline__ double accumulate_hit'), find('// Conservative float32 test')),
          ('shade_hit', find('__device__ __forceinline__ void shade_hit'), find('// Returns the accumulated alpha')),
          ('may_enter', find('// Conservative float32 test'), find('// Instrumentation (lvx_render_footprint)')),
          ('prologue (ray setup)', find('render_kernel(const RenderArgs A) {'), find('= W: walk to the next')),
          ('W walk', find('= W: walk to the next'), find('= V: list the voxels')),
          ('V voxel headers', find('= V: list the voxels'), find('= C + E: pre-reject')),
          ('C pre-reject', find('= C + E: pre-reject'), find('---- E: exact')),
          ('E exact-test driver', find('---- E: exact'), find('---- each owner takes')),
          ('owner insert', find('---- each owner takes'), find('= S: composite, _kernels')),
          ('S composite', find('= S: composite, _kernels'), find('// tail: a terminated ray')),
          ('tail+output', find('// tail: a terminated ray'), find('__global__ void __launch_bounds__(256)'))]
agg = collections.defaultdict(lambda: [0, 0, 0])
for d in data:
    a = agg[stage(d)]; a[0] += d[0]; a[1] += d[1]; a[2] += d[2]
print()
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:32s} {100*a[0]/tot:5.1f}% samples {100*a[1]/toti:5.1f}% warp-inst {100*a[2]/tott:5.1f}% thread-inst  thr/inst {a[2]/max(a[1],1):5.1f}")

# static size of the code each stage actually runs (SASS instructions executed > 1e5 times)
hot = collections.Counter(); allc = collections.Counter()
for f, ln, ex, smp in sass:
    k = stage((0, 0, 0, f, ln, ''))
    allc[k] += 1
    if ex > 1e5: hot[k] += 1
print()
print("hot code (executed > 1e5 times): %.1f KB of %.1f KB" % (sum(hot.values()) * 16 / 1024, sum(allc.values()) * 16 / 1024))
for k, v in sorted(hot.items(), key=lambda kv: -kv[1]):
    print(f"  {k:32s} {v:5d} instr {v*16/1024:5.1f} KB   (all {allc[k]})")
