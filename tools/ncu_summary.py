"""Summarise ncu output for profiles/ (committed evidence).

    python tools/ncu_summary.py launches <launches.csv> <hulls> <out.json>
        per-kernel launches / time / DRAM bytes of the LAST hull of a launch
        list (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
        dram__bytes_write.sum --csv), plus the ordered launch sequence
    python tools/ncu_summary.py full <capture.ncu-rep> <out.txt>
        the key --set full metrics of one captured launch
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys


def launches(path: str, hulls: int, out: str) -> None:
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    per: dict = collections.OrderedDict()
    for r in rows:
        per.setdefault((r["ID"], r["Kernel Name"]), {})[r["Metric Name"]] = float(
            r["Metric Value"].replace(",", ""))
    items = list(per.items())
    # the last COMPLETE hull: between the last two presort starts when the
    # capture holds them (a launch window need not align with hulls)
    marks = [i for i, ((_, name), _m) in enumerate(items) if "k_scan_init" in name]
    if len(marks) >= 2:
        last = items[marks[-2]:marks[-1]]
    else:
        last = items[len(items) - len(items) // hulls:]
    agg: dict = collections.OrderedDict()
    seq = []
    for (_, name), m in last:
        k = name.split("(")[0].replace("void ", "")
        t_ms = m.get("gpu__time_duration.sum", 0.0) / 1e6
        dram = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a = agg.setdefault(k, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0, "warp_inst": 0.0})
        a["launches"] += 1
        a["ms"] += t_ms
        a["dram_bytes"] += dram
        a["warp_inst"] += m.get("smsp__inst_executed.sum", 0.0)
        seq.append({"kernel": k, "ms": round(t_ms, 4), "dram_bytes": int(dram)})
    total = sum(a["ms"] for a in agg.values())
    kernels = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        kernels.append({"kernel": k, "launches": a["launches"], "ms": round(a["ms"], 4),
                        "share": round(a["ms"] / total, 4) if total else None,
                        "dram_bytes": int(a["dram_bytes"]),
                        "dram_bytes_per_launch": int(a["dram_bytes"] / a["launches"]),
                        "dram_gbps": round(a["dram_bytes"] / a["ms"] / 1e6, 1) if a["ms"] else None,
                        "warp_inst": int(a["warp_inst"]),
                        "warp_inst_per_launch": int(a["warp_inst"] / a["launches"])})
    doc = {"source": path, "hulls_in_capture": hulls, "note":
           "ncu --clock-control none, serialised cold-cache launches: compare shares, not absolutes",
           "total_ms": round(total, 4), "kernels": kernels, "sequence": seq}
    json.dump(doc, open(out, "w"), indent=1)
    print(f"{out}: {len(seq)} launches, {total:.3f} ms")
    for k in kernels[:12]:
        print(f"  {k['kernel'][:50]:50s} {k['launches']:4d} {k['ms']:8.3f} ms {k['share']*100:5.1f}%"
              f" {k['dram_gbps']} GB/s")


WANT = [
    "Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
    "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
    "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
    "Executed Instructions", "Registers Per Thread", "Dynamic Shared Memory Per Block",
    "Block Size", "Grid Size", "Theoretical Active Warps per SM", "Achieved Active Warps Per SM",
    "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate", "Branch Efficiency",
]


def full(rep: str, out: str) -> None:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = csv.reader(io.StringIO(txt))
    h = next(r)
    lines = []
    kname = None
    for row in r:
        d = dict(zip(h, row))
        kname = kname or d.get("Kernel Name")
        if d.get("Metric Name") in WANT:
            lines.append(f"{d['Metric Name']:40s} {d['Metric Value']:>16s} {d.get('Metric Unit', '')}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        hdr, units, vals = rr[0], rr[1], rr[2]
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                    "smsp__inst_executed_pipe_fp64.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
            if key in hdr:
                i = hdr.index(key)
                lines.append(f"{key:40s} {vals[i]:>16s} {units[i]}")
    with open(out, "w") as f:
        f.write(f"# {rep}\n# kernel: {kname}\n")
        f.write("\n".join(lines) + "\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    else:
        full(sys.argv[2], sys.argv[3])
