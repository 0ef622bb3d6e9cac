"""Turn one GPU-box visit's ncu output into the tracked summaries under profiles/.

    python tools/profile_summary.py <tag> [--workload c3]

reads   gpurun_out/launches_<tag>.csv        (ncu --metrics gpu__time_duration.sum launch list)
        gpurun_out/prof_render_<tag>.ncu-rep (ncu --set full capture of the frame kernel)
writes  profiles/<tag>_launches.csv          per-kernel launch count / total / mean device time
        profiles/<tag>_render_kernel.txt     raw-page metrics + per-stage sample shares
        profiles/traffic.json                dram bytes per launch (bench.py's roofline.traffic)
"""
import argparse
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")

RAW_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__waves_per_multiprocessor", "launch__shared_mem_per_block_static",
    "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
    "sm__cycles_elapsed.max", "smsp__cycles_active.avg",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
    "smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio",
    "smsp__average_warp_latency_issue_stalled_wait.ratio",
    "smsp__average_warp_latency_issue_stalled_barrier.ratio",
    "smsp__average_warp_latency_issue_stalled_branch_resolving.ratio",
    "smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio",
    "smsp__average_warp_latency_issue_stalled_lg_throttle.ratio",
    "smsp__average_warp_latency_issue_stalled_no_instruction.ratio",
    "smsp__average_warp_latency_issue_stalled_not_selected.ratio",
    "smsp__average_warp_latency_issue_stalled_dispatch_stall.ratio",
]


def launches(tag):
    path = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"]
        a = agg.setdefault(k, [0, 0.0, d["Grid Size"], d["Block Size"]])
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", "")) / 1e6
    total = sum(a[1] for a in agg.values())
    out = os.path.join(OUT, f"{tag}_launches.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_ms", "mean_ms", "share_of_all_launches", "grid", "block"])
        for k, (n, t, g, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            w.writerow([k, n, f"{t:.4f}", f"{t / n:.4f}", f"{t / total:.4f}", g, b])
    return out


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (r[i], units[i]) for i, h in enumerate(hdr)}
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--kernel", default="render_kernel")
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    try:
        print("wrote", launches(args.tag))
    except FileNotFoundError:
        print("no launch list for", args.tag)
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{'render' if args.kernel == 'render_kernel' else args.kernel}_{args.tag}.ncu-rep")
    if not os.path.exists(rep):
        print("no full capture", rep)
        return
    ms = raw_metrics(rep)
    path = os.path.join(OUT, f"{args.tag}_{args.kernel}.txt")
    with open(path, "w") as f:
        f.write(f"# ncu --set full --clock-control none, {args.kernel}, workload {args.workload}, capture tag {args.tag}\n")
        f.write("# (times under ncu are cold-cache and serialised; bench.py's CUDA-event time is the number of record)\n")
        for d in ms:
            f.write(f"\nkernel: {d['Kernel Name'][0]}\n")
            for k in RAW_KEYS:
                if k in d:
                    f.write(f"  {k:75s} {d[k][0]:>18s} {d[k][1]}\n")
        lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "25"],
                               capture_output=True, text=True).stdout
        f.write("\n# source-page aggregation (tools/ncu_lines.py): hottest CUDA lines by sampled stalls\n")
        f.write(lines)
    print("wrote", path)
    d = ms[0]

    def num(k):
        v, u = d[k]
        x = float(v.replace(",", ""))
        mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return x * mul

    tj = os.path.join(OUT, "traffic.json")
    cur = json.load(open(tj)) if os.path.exists(tj) else {}
    cur.setdefault(args.workload, {})[args.kernel] = int(num("dram__bytes_read.sum") + num("dram__bytes_write.sum"))
    cur[args.workload][args.kernel + "_detail"] = {
        "dram_read_bytes": int(num("dram__bytes_read.sum")), "dram_write_bytes": int(num("dram__bytes_write.sum")),
        "capture": args.tag}
    json.dump(cur, open(tj, "w"), indent=1)
    print("wrote", tj)


if __name__ == "__main__":
    main()
