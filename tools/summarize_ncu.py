"""Summarise ncu outputs into the text files kept under profiles/.

    python tools/summarize_ncu.py launches gpurun_out/launches.csv > profiles/rNN_launches.txt
    python tools/summarize_ncu.py report gpurun_out/prof.ncu-rep > profiles/rNN_kernels.txt

`launches` aggregates a `--metrics gpu__time_duration.sum --csv` launch list per kernel (per
frame: the list must cover whole frames); `report` prints the key speed-of-light, occupancy,
DRAM-traffic and stall numbers of every kernel in a `--set full` report, plus the hottest source
lines.
"""

import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy",
        "Achieved Active Warps Per SM", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]


def launches(path, frames=None):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = OrderedDict()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"]
        agg.setdefault(k, [0.0, 0])
        agg[k][0] += float(d["Metric Value"])
        agg[k][1] += 1
    total = sum(v[0] for v in agg.values())
    n = len(data)
    print(f"# {n} launches, total {total / 1e3:.1f} us (ncu --clock-control none, serialised,"
          " cold cache: compare shares)")
    print(f"{'share':>6} {'total_us':>10} {'launches':>8}  kernel")
    for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{100 * v / total:5.1f}% {v / 1e3:10.1f} {c:8d}  {k[:110]}")


def _csv(args):
    out = subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(path):
    rows = _csv([path, "--page", "details", "--csv"])
    hdr = rows[0]
    per = OrderedDict()
    raw = _csv([path, "--page", "raw", "--csv"])
    rhdr = raw[0] if raw else []
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        key = (d.get("ID"), d.get("Kernel Name"))
        if d.get("Metric Name") in KEYS:
            per.setdefault(key, []).append(f"{d['Metric Name']}: {d['Metric Value']} "
                                           f"{d['Metric Unit']}".rstrip())
    dram = {}
    extra = {}
    units = dict(zip(rhdr, raw[1])) if len(raw) > 1 else {}
    pipes = ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
             "smsp__issue_active.avg.pct_of_peak_sustained_active",
             "smsp__thread_inst_executed_per_inst_executed.ratio"]
    for r in raw[2:]:
        d = dict(zip(rhdr, r))
        key = (d.get("ID"), d.get("Kernel Name"))
        vals = []
        for m in pipes:
            if m in d:
                vals.append(f"{m.split('.')[0].replace('sm__', '').replace('smsp__', '')}="
                            f"{d[m]}")
        stalls = []
        for m, v in d.items():
            if m.startswith("smsp__average_warps_issue_stalled_") and \
                    m.endswith("_per_issue_active.ratio") and "selected" not in m:
                try:
                    stalls.append((float(v.replace(",", "")), m[len(
                        "smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        extra[key] = (vals, stalls[:4])
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for r in raw[2:]:
        d = dict(zip(rhdr, r))
        try:
            rd = float(d.get("dram__bytes_read.sum", "nan").replace(",", ""))
            wr = float(d.get("dram__bytes_write.sum", "nan").replace(",", ""))
        except ValueError:
            continue
        rd *= scale.get(units.get("dram__bytes_read.sum", "byte"), 1.0)
        wr *= scale.get(units.get("dram__bytes_write.sum", "byte"), 1.0)
        dram[(d.get("ID"), d.get("Kernel Name"))] = (rd, wr)
    for key, lines in per.items():
        print(f"== [{key[0]}] {key[1][:120]}")
        for ln in lines:
            print("   " + ln)
        if key in dram:
            rd, wr = dram[key]
            print(f"   dram__bytes_read.sum: {rd:.0f} B, dram__bytes_write.sum: {wr:.0f} B, "
                  f"traffic: {rd + wr:.0f} B")
        if key in extra:
            vals, stalls = extra[key]
            if vals:
                print("   pipes (% of peak, active): " + ", ".join(vals))
            if stalls:
                print("   top stalls (warps per issue): " +
                      ", ".join(f"{n} {v:.2f}" for v, n in stalls))
        print()


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        launches(path)
    else:
        report(path)
