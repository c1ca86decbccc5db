#!/usr/bin/env python
"""Turn a round's raw ncu outputs (gpurun_out/, scratch) into the committed
summaries under profiles/.  Inputs, all from one gpurun call of
profiles/profile_round.sh (same bench command, N=1, config 2):

  prof_launches.csv  ncu --metrics gpu__time_duration.sum (every launch of
                     `bench.py --steps 2 --warmup 3`, cold-cache, serialised)
  prof_dram.csv      ncu --metrics dram__bytes_{read,write}.sum for the
                     simulator, stream and row-statistics kernels
  prof_full.ncu-rep, prof_full_stats.ncu-rep
                     ncu --set full of the simulator and the row-statistics kernel

    python profiles/make_summaries.py r1 [gpurun_out]
"""

from __future__ import annotations

import collections
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def _rows(path):
    with open(path) as fh:  # ncu CSV rows only (the profiled program's stdout may be interleaved)
        lines = [ln for ln in fh if ln.startswith('"')]
    hdr = lines[:1]  # captures appended one after another repeat the header
    return list(csv.DictReader(hdr + [ln for ln in lines[1:] if not ln.startswith('"ID"')]))


def short(name: str) -> str:
    name = name.split("(")[0]
    return name.replace("void ", "").replace("cs::", "")


def launches(tag, src):
    rows = [r for r in _rows(os.path.join(src, "prof_launches.csv"))
            if r["Metric Name"] == "gpu__time_duration.sum"]
    per = collections.OrderedDict()
    for r in rows:
        per.setdefault(short(r["Kernel Name"]), []).append(float(r["Metric Value"]) / 1e3)  # ns -> us
    total = sum(sum(v) for v in per.values())
    out = [f"# {tag}: ncu launch list of `python bench.py --steps 2 --warmup 3 --e2e-steps 0 "
           "--no-cpu-baseline` (config 2, N=1)",
           "# gpu__time_duration.sum, --clock-control none; cold-cache and serialised, so the",
           "# kernel SHARES are the comparable quantity, not absolute times.",
           f"{'kernel':48s} {'launches':>8s} {'avg_us':>12s} {'total_us':>12s} {'share':>7s}"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:48s} {len(v):8d} {sum(v) / len(v):12.1f} {sum(v):12.1f} {sum(v) / total:7.1%}")
    with open(os.path.join(HERE, f"{tag}_launches_summary.txt"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    with open(os.path.join(src, "prof_launches.csv")) as fin, \
            open(os.path.join(HERE, f"{tag}_launches.csv"), "w") as fout:
        fout.writelines(ln for ln in fin if not ln.startswith("=="))
    print("\n".join(out))


def traffic(tag, src):
    rows = _rows(os.path.join(src, "prof_dram.csv"))
    k = collections.OrderedDict()
    for r in rows:
        name = short(r["Kernel Name"])
        base = name.split("<")[0]
        d = k.setdefault(base, {"kernel": name})
        key = {"dram__bytes_read.sum": "dram_read_bytes", "dram__bytes_write.sum": "dram_write_bytes",
               "gpu__time_duration.sum": "duration_ms"}[r["Metric Name"]]
        v = float(r["Metric Value"])
        unit = r["Metric Unit"]
        if key == "duration_ms":
            v = v / 1e6 if unit == "ns" else (v / 1e3 if unit == "us" else v)
        else:
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[key] = v
    doc = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     "--clock-control none; python bench.py --steps 1 --warmup 0 --e2e-steps 0 "
                     "--no-cpu-baseline (first launch of each kernel)",
           "workload": "config2: 16 lambdas x 1024 reps x 100000 jobs", "kernels": k}
    with open(os.path.join(HERE, f"{tag}_traffic.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc, indent=1))


METRICS = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
           "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
           "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
           "Executed Instructions", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block")


def full(tag, src):
    txt = ""
    for name in ("prof_full.ncu-rep", "prof_full_stats.ncu-rep"):
        rep = os.path.join(src, name)
        if os.path.exists(rep):
            txt += subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True,
                                  text=True).stdout
    out, kernel = [f"# {tag}: ncu --set full --clock-control none of the top kernels "
                   "(python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline)"], None
    for line in txt.splitlines():
        if "Context" in line and "Stream" in line and "(" in line:
            kernel = short(line.strip())
            out.append(f"\n== {kernel}")
        s = line.strip()
        for m in METRICS:
            if s.startswith(m + " ") or s.startswith(m + "  "):
                out.append("  " + " ".join(s.split()))
    with open(os.path.join(HERE, f"{tag}_ncu_full_summary.txt"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(HERE), "gpurun_out")
    launches(tag, src)
    traffic(tag, src)
    full(tag, src)
