"""Static SASS instruction count per source region of render_kernel<false> (developer tool).
usage: python tools/sass_regions.py file.o|file.cubin"""
import collections, os, re, subprocess, sys, tempfile
src = sys.argv[1]
tmp = tempfile.mkdtemp()
if not src.endswith(".cubin"):
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(src)], cwd=tmp, capture_output=True)
    src = os.path.join(tmp, [f for f in os.listdir(tmp) if f.endswith(".cubin")][0])
sass = subprocess.run(["nvdisasm", "-g", "-c", src], capture_output=True, text=True).stdout
cur = None; fn = None
cnt = collections.Counter()
for l in sass.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m: fn = m.group(1); continue
    if fn and 'render_kernelILb0' in fn and re.match(r'\s+/\*[0-9a-f]{4,6}\*/', l):
        cnt[cur] += 1
print("total", sum(cnt.values()), "instr =", sum(cnt.values()) * 16 // 1024, "KB")
GEOM = [(82, 'tube_f32axis'), (150, 'tube_f64'), (190, 'sphere'), (292, 'dda'), (320, 'trilinear'), (357, 'cone'),
        (374, 'density_ray'), (403, 'orient'), (423, 'ao_point'), (439, 'shade'), (10**9, 'alpha')]
g = collections.Counter(); r = collections.Counter(); o = collections.Counter()
for (f, ln), c in cnt.items():
    if f == 'lvx_geom.cuh':
        g[[n for hi, n in GEOM if ln < hi][0]] += c
    elif f == 'lvx_render.cu':
        r[ln // 20 * 20] += c
    else:
        o[f] += c
print("geom:", dict(g)); print("other:", dict(o))
print("lvx_render.cu by 20-line block:", {k: r[k] for k in sorted(r)})
