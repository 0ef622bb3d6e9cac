"""Summarise an `ncu --set full` capture of one wavefront frame (all wf_* kernels) into
profiles/<tag>_wavefront_kernels.txt and profiles/traffic.json (developer tool).

    python tools/profile_wf.py <tag> [--workload c3]
reads gpurun_out/prof_wf_<tag>.ncu-rep
"""
import argparse, collections, csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser(); ap.add_argument("tag"); ap.add_argument("--workload", default="c3")
a = ap.parse_args()
rep = os.path.join(ROOT, "gpurun_out", f"prof_wf_{a.tag}.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
def col(name): return h.index(name)
def unit_scale(name):
    u = units[col(name)].lower()
    return {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
            "msecond": 1.0, "nsecond": 1e-6, "second": 1e3}.get(u, 1)
M = {"ms": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
     "lts": "lts__throughput.avg.pct_of_peak_sustained_elapsed", "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "warps": "sm__warps_active.avg.pct_of_peak_sustained_active", "lanes": "smsp__thread_inst_executed_per_inst_executed.ratio",
     "regs": "launch__registers_per_thread", "inst": "smsp__inst_executed.sum",
     "fp64": "sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active", "l2sec": "lts__t_sectors.sum",
     "l1hit": "l1tex__t_sector_hit_rate.pct", "l2hit": "lts__t_sector_hit_rate.pct"}
stall = [k for k in h if "issue_stalled" in k and "per_issue_active" in k]
agg = collections.OrderedDict()
n_begin = 0
for r in rows[2:]:
    d = dict(zip(h, r))
    if "wf_begin_kernel" in d["Kernel Name"]:
        n_begin += 1
    if n_begin != 1:
        continue  # exactly one frame: from the first wf_begin to the next
    name = d["Kernel Name"].split("(")[0].split("::")[-1]
    if "wf_exact_kernel" in d["Kernel Name"]:
        name = "wf_exact<%s>" % ("tube" if "<0" in d["Kernel Name"].split("wf_exact_kernel")[1][:4] else "sphere")
    e = agg.setdefault(name, collections.defaultdict(float))
    e["n"] += 1
    t = float(d[M["ms"]]) * unit_scale(M["ms"])
    e["ms"] += t
    if M["rd"] in d:
        e["rd"] += float(d[M["rd"]]) * unit_scale(M["rd"])
        e["wr"] += float(d[M["wr"]]) * unit_scale(M["wr"])
    else:  # section-limited capture: only the total rate is there (reported in the read column)
        k = "dram__bytes.sum.per_second"
        rate = float(d[k]) * {"gbyte/s": 1e9, "mbyte/s": 1e6, "kbyte/s": 1e3, "tbyte/s": 1e12, "byte/s": 1}.get(units[col(k)].lower(), 1)
        e["rd"] += rate * t * 1e-3
    e["inst"] += float(d[M["inst"]])
    e["l2sec"] += float(d.get(M["l2sec"]) or 0)
    for k in ("lts", "issue", "warps", "lanes", "fp64", "l1hit", "l2hit"):
        e[k] += float(d.get(M[k]) or 0) * t          # time-weighted
    e["regs"] = float(d[M["regs"]])
    for k in stall:
        e["st_" + k.split("issue_stalled_")[1].split("_per")[0]] += float(d[k] or 0) * t
out = [f"# ncu (SpeedOfLight, MemoryWorkloadAnalysis, WarpStateStats, SchedulerStats, LaunchStats, Occupancy, InstructionStats; --clock-control none; caches flushed before every kernel), every wf_* kernel of one wavefront frame, workload {a.workload}, capture tag {a.tag}",
       "# (times under ncu are cold-cache and serialised; bench.py's CUDA-event time is the number of record)", ""]
tot_ms = sum(e["ms"] for e in agg.values()); tot_rd = sum(e["rd"] for e in agg.values()); tot_wr = sum(e["wr"] for e in agg.values())
out.append(f"{'kernel':20s} {'n':>3s} {'ms':>7s} {'share':>6s} {'dram MB':>9s} {'':>9s} {'L2 GB':>6s} {'lts%':>5s} {'issue%':>6s} {'warps%':>6s} {'lanes':>5s} {'fp64%':>5s} {'regs':>4s}  top stalls (warps per issue slot)")
for name, e in agg.items():
    t = e["ms"] or 1
    st = sorted(((v / t, k[3:]) for k, v in e.items() if k.startswith("st_")), reverse=True)[:3]
    out.append(f"{name:20s} {int(e['n']):3d} {e['ms']:7.3f} {100*e['ms']/tot_ms:5.1f}% {e['rd']/1e6:9.1f} {e['wr']/1e6:9.1f} {e['l2sec']*32/1e9:6.2f} "
               f"{e['lts']/t:5.1f} {e['issue']/t:6.1f} {e['warps']/t:6.1f} {e['lanes']/t:5.1f} {e['fp64']/t:5.1f} {int(e['regs']):4d}  "
               + " ".join(f"{n}={v:.2f}" for v, n in st))
out.append(f"{'frame total':20s} {int(sum(e['n'] for e in agg.values())):3d} {tot_ms:7.3f} 100.0% {tot_rd/1e6:9.1f} {tot_wr/1e6:9.1f}")
txt = "\n".join(out) + "\n"
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
open(os.path.join(ROOT, "profiles", f"{a.tag}_wavefront_kernels.txt"), "w").write(txt)
print(txt)
tp = os.path.join(ROOT, "profiles", "traffic.json")
tj = json.load(open(tp)) if os.path.exists(tp) else {}
w = tj.setdefault(a.workload, {})
w["wavefront_frame"] = int(tot_rd + tot_wr)
w["wavefront_frame_detail"] = {"dram_read_bytes": int(tot_rd), "dram_write_bytes": int(tot_wr), "capture": a.tag,
                               "kernels": int(sum(e['n'] for e in agg.values()))}
json.dump(tj, open(tp, "w"), indent=1)
