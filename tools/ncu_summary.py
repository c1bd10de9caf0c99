"""Summaries of ncu output for profiles/ (development aid).

  python tools/ncu_summary.py launches <launches.csv> [header]   per-kernel share of a launch list
  python tools/ncu_summary.py details <report.ncu-rep> [regex]    key --set full metrics per kernel
"""
import collections
import csv
import subprocess
import sys


def launches(path, header=""):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    if header:
        print(header)
    print(f"{'kernel':80s} {'launches':>8s} {'total_ns':>14s} {'avg_us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:80]:80s} {v[0]:8d} {v[1]:14.0f} {v[1] / v[0] / 1e3:10.2f} {v[1] / tot:6.3f}")


KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Registers Per Thread", "Achieved Occupancy", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "SM Busy", "Executed Ipc Active")


def details(rep, regex=""):
    cmd = ["ncu", "-i", rep, "--page", "details", "--csv"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if not rows:
        print("no rows")
        return
    h = rows[0]
    ki, si, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit",
                                               "Metric Value"))
    cur = None
    for r in rows[1:]:
        if len(r) <= vi or (regex and regex not in r[ki]):
            continue
        if r[ki] != cur:
            cur = r[ki]
            print(f"== {cur[:120]}")
        if r[mi] in KEYS:
            print(f"  [{r[si]}] {r[mi]}: {r[vi]} {r[ui]}")


def traffic(rep, regex=""):
    """dram__bytes_read.sum + dram__bytes_write.sum and duration per launch of the kernels matching regex."""
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
           "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki = h.index("Kernel Name")
    cols = {m: h.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
    units = rows[1]
    res = []
    for r in rows[2:]:
        if regex and regex not in r[ki]:
            continue
        vals = {}
        for m, i in cols.items():
            v = float(r[i].replace(",", ""))
            u = units[i]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                     "msecond": 1e-3}.get(u, 1)
            vals[m] = v * scale
        res.append({"kernel": r[ki][:100], "dram_bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                    "dram_read": vals["dram__bytes_read.sum"], "dram_write": vals["dram__bytes_write.sum"],
                    "duration_s": vals["gpu__time_duration.sum"]})
    import json
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
        sys.exit(0)
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    else:
        details(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
