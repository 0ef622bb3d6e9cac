"""Per-kernel table from an `ncu --page raw --csv` export (developer tool).

    python tools/ncu_table.py <raw.csv> [--by-launch] [--title "..."] [--out profiles/x.txt]
Aggregates launches by kernel name (time-weighted means) and prints: launches, total ms, share,
dram GB (read+write), dram GB/s and % of HBM peak, L2 GB (lts__t_bytes, or lts__t_sectors x 32 B) and lts %, issue %, achieved
warps %, lanes per instruction, fp64 / fma / alu / lsu pipe %, registers, top stall reasons.
"""
import argparse, collections, csv, json, os, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("csv"); ap.add_argument("--by-launch", action="store_true"); ap.add_argument("--title", default="")
ap.add_argument("--out", default=""); ap.add_argument("--json", default="")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
h, units = rows[0], rows[1]
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    PEAK = 6650.0

def scale(name):
    u = units[h.index(name)].lower()
    return {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3,
            "ms": 1.0, "msecond": 1.0, "second": 1e3, "s": 1e3}.get(u, 1)

M = {"ms": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum", "l2": "lts__t_bytes.sum", "l2s": "lts__t_sectors.sum",
     "lts": "lts__throughput.avg.pct_of_peak_sustained_elapsed", "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "warps": "sm__warps_active.avg.pct_of_peak_sustained_active", "lanes": "smsp__thread_inst_executed_per_inst_executed.ratio",
     "regs": "launch__registers_per_thread", "fp64": "sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active",
     "fp64b": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "fma": "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active", "alu": "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
     "lsu": "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "l1hit": "l1tex__t_sector_hit_rate.pct",
     "l2hit": "lts__t_sector_hit_rate.pct", "inst": "smsp__inst_executed.sum", "occ": "sm__maximum_warps_per_active_cycle_pct",
     "local": "sass__inst_executed_local_loads"}
M = {k: v for k, v in M.items() if v in h}
stall = [k for k in h if "issue_stalled" in k and "per_issue_active" in k]

def short(name):
    n = name.split("(")[0].split("::")[-1]
    if "<" in name.split("(")[0]:
        n = name.split("(")[0].split("::")[-1]
    n = n.replace("void ", "").replace("_kernel", "")
    if "wf_exact" in name:
        t = name.split("wf_exact_kernel<")[1].split(">")[0].replace(" ", "").replace("(bool)", "")
        # one launch for tubes and joint spheres since round 2; template arguments: geometry rays, packed records
        n = "wf_exact" + {"0,0": "", "1,0": "<geom>", "0,1": "<packed>"}.get(t, "<%s>" % t)
    return n[:26]

agg = collections.OrderedDict()
for i, r in enumerate(rows[2:]):
    d = dict(zip(h, r))
    key = short(d["Kernel Name"]) + (f"#{i}" if a.by_launch else "")
    e = agg.setdefault(key, collections.defaultdict(float))
    t = float(d[M["ms"]]) * scale(M["ms"])
    e["n"] += 1; e["ms"] += t
    for k in ("rd", "wr", "l2"):
        if k in M and d[M[k]] not in ("", "n/a"):
            e[k] += float(d[M[k]]) * scale(M[k])
    # (--set full carries the L2 traffic as sectors, not bytes: 32 bytes each)
    if "l2" not in M and "l2s" in M and d[M["l2s"]] not in ("", "n/a"):
        e["l2"] += float(d[M["l2s"]].replace(",", "")) * 32.0
    for k in ("lts", "issue", "warps", "lanes", "fp64", "fp64b", "fma", "alu", "lsu", "l1hit", "l2hit"):
        if k in M and d[M[k]] not in ("", "n/a"):
            e[k] += float(d[M[k]]) * t
    e["regs"] = float(d[M["regs"]]); e["grid"] = d.get("Grid Size", ""); e["block"] = d.get("Block Size", "")
    if "inst" in M: e["inst"] += float(d[M["inst"]])
    for k in stall:
        if d[k] not in ("", "n/a"):
            e["st_" + k.split("issue_stalled_")[1].split("_per")[0]] += float(d[k]) * t
tot = sum(e["ms"] for e in agg.values())
out = []
if a.title: out.append("# " + a.title)
out.append(f"# source: {os.path.basename(a.csv)}; ncu --set full, --clock-control none; per-launch times under ncu are cold-cache and serialised: compare SHARES; HBM peak {PEAK} GB/s (MEASURED_PEAKS.json)")
out.append(f"{'kernel':26s} {'n':>3s} {'ms':>8s} {'share':>6s} {'dramGB':>7s} {'GB/s':>6s} {'%hbm':>5s} {'L2 GB':>6s} {'lts%':>5s} {'L1hit':>5s} {'L2hit':>5s} {'issue%':>6s} {'warps%':>6s} {'lanes':>5s} {'fp64%':>5s} {'fma%':>5s} {'alu%':>5s} {'lsu%':>5s} {'regs':>4s}  top stalls (warps per issue slot)")
js = {}
for name, e in agg.items():
    t = e["ms"] or 1e-9
    st = sorted(((v / t, k[3:]) for k, v in e.items() if k.startswith("st_")), reverse=True)[:3]
    dram = e["rd"] + e["wr"]
    gbs = dram / t / 1e6
    out.append(f"{name:26s} {int(e['n']):3d} {e['ms']:8.3f} {100*e['ms']/tot:5.1f}% {dram/1e9:7.3f} {gbs:6.0f} {100*gbs/PEAK:5.1f} {e['l2']/1e9:6.2f} "
               f"{e['lts']/t:5.1f} {e['l1hit']/t:5.1f} {e['l2hit']/t:5.1f} {e['issue']/t:6.1f} {e['warps']/t:6.1f} {e['lanes']/t:5.1f} {max(e['fp64'], e['fp64b'])/t:5.1f} {e['fma']/t:5.1f} "
               f"{e['alu']/t:5.1f} {e['lsu']/t:5.1f} {int(e['regs']):4d}  " + " ".join(f"{n}={v:.2f}" for v, n in st))
    js[name] = {"launches": int(e["n"]), "ms": e["ms"], "dram_bytes": dram, "dram_read": e["rd"], "dram_write": e["wr"], "l2_bytes": e["l2"]}
dr = sum(e["rd"] + e["wr"] for e in agg.values()); l2 = sum(e["l2"] for e in agg.values())
out.append(f"{'total':26s} {int(sum(e['n'] for e in agg.values())):3d} {tot:8.3f} 100.0% {dr/1e9:7.3f} {dr/tot/1e6:6.0f} {100*dr/tot/1e6/PEAK:5.1f} {l2/1e9:6.2f}")
txt = "\n".join(out) + "\n"
print(txt)
if a.out: open(a.out, "w").write(txt)
if a.json:
    json.dump({"total_ms": tot, "dram_bytes": dr, "l2_bytes": l2, "kernels": js}, open(a.json, "w"), indent=1)
