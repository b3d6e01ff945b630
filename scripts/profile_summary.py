"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU).

  python scripts/profile_summary.py report gpurun_out/x.ncu-rep [name]  -> text summary on stdout
  python scripts/profile_summary.py launches gpurun_out/launches.csv     -> per-kernel share table
  python scripts/profile_summary.py traffic gpurun_out/a.ncu-rep:knn_search gpurun_out/b.ncu-rep:replay_kernel
"""
import collections
import csv
import io
import json
import subprocess
import sys


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    r = ncu_csv(rep, "raw")
    hdr, units, vals = r[0], r[1], r[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def report(rep, name=None):
    rows = ncu_csv(rep, "details")
    hdr = rows[0]
    keep = ("Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
            "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
            "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM",
            "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
            "Grid Size", "Block Size", "Dynamic Shared Memory Per Block")
    kname = None
    lines = []
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        kname = kname or d.get("Kernel Name")
        if d.get("Metric Name") in keep:
            lines.append(f"  {d['Metric Name']:<36} {d['Metric Value']:>14} {d['Metric Unit']}")
    m = raw_metrics(rep)
    stalls = []
    tot = 0.0
    for h, (v, _) in m.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                tot += float(v)
            except ValueError:
                pass
    print(f"kernel: {kname}")
    print(f"report: {rep}")
    print("\n".join(lines))
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"):
        if key in m:
            print(f"  {key:<60} {m[key][0]} {m[key][1]}")
    print("  warp stall samples (share):")
    for v, h in sorted(stalls, reverse=True)[:8]:
        print(f"    {100 * v / tot:5.1f}%  {h}")


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    per = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = name.replace("void ", "").split("(")[0].split("<")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        v = v / 1e3 if unit == "nsecond" else v * 1e3 if unit == "msecond" else v  # -> usecond
        per[name][0] += 1
        per[name][1] += v
    tot = sum(v[1] for v in per.values())
    print(f"{'kernel':<40} {'launches':>8} {'total_us':>12} {'share':>7}")
    for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1]):
        print(f"{k:<40} {n:>8} {t:>12.1f} {100 * t / tot:>6.1f}%")


def traffic(specs):
    out = {}
    for spec in specs:
        rep, name = spec.split(":")
        m = raw_metrics(rep)
        rd = float(m["dram__bytes_read.sum"][0]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m["dram__bytes_read.sum"][1]]
        wr = float(m["dram__bytes_write.sum"][0]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m["dram__bytes_write.sum"][1]]
        out[name] = rd + wr
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "report":
        report(*sys.argv[2:])
    elif cmd == "launches":
        launches(sys.argv[2])
    else:
        traffic(sys.argv[2:])
