#!/usr/bin/env python
"""Committed round-2 summaries from one gpurun call of profiles/profile_r2.sh
(raw outputs in gpurun_out/, scratch):

  r2_launches_summary.txt  per-kernel share of one bench sweep (device time,
                           cold-cache, serialised: compare SHARES)
  r2_ncu_summary.json      per-launch counters (instructions, DRAM bytes,
                           issue-slot %) of every kernel of the config-2 sweep;
                           bench.py reads it for the issue roofline
  r2_ncu_full_summary.txt  ncu --set full key metrics of the simulator, the
                           row-statistics pass, the stream kernel, GBP and GCA
  r2_ncu_compose.json      issue utilisation of gbp/gca (config 4, full fleet)

    python profiles/make_summaries_r2.py [gpurun_out]
"""

from __future__ import annotations

import collections
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SHAPE = (16, 1024, 100000)  # points, replications, jobs (bench.py defaults)


def _rows(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    hdr = lines[:1]
    return list(csv.DictReader(hdr + [ln for ln in lines[1:] if not ln.startswith('"ID"')]))


def short(name: str) -> str:
    name = name.split("(")[0]
    for p in ("void ", "cs::seg::", "cs::"):
        name = name.replace(p, "")
    return name


def scale(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
                "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1)


def launches(src):
    per = collections.OrderedDict()
    for r in _rows(os.path.join(src, "prof_launches.csv")):
        k = short(r["Kernel Name"])
        d = per.setdefault(k, collections.defaultdict(list))
        d[r["Metric Name"]].append(scale(r["Metric Value"], r["Metric Unit"]))
    tot = sum(sum(v["gpu__time_duration.sum"]) for v in per.values())
    out = ["# r2: ncu launch list of `python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline "
           "--no-config5 --no-compose` (config 2, N=1; 3 warm-up + 1 timed + 2 stage sweeps)",
           "# gpu__time_duration.sum, --clock-control none; cold-cache and serialised: compare SHARES.",
           f"{'kernel':44s} {'launches':>8s} {'avg_ms':>10s} {'share':>7s} {'inst/launch':>14s} "
           f"{'DRAM GB/launch':>15s} {'issue %':>8s}"]
    summ = {"shape": list(SHAPE), "source": "profiles/profile_r2.sh (ncu launch list, averages per launch)",
            "kernels": {}}
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        n = len(v["gpu__time_duration.sum"])
        avg = lambda m: sum(v[m]) / len(v[m]) if v.get(m) else None
        t = avg("gpu__time_duration.sum")
        inst = avg("smsp__inst_executed.sum")
        rd, wr = avg("dram__bytes_read.sum") or 0.0, avg("dram__bytes_write.sum") or 0.0
        iss = avg("smsp__issue_active.avg.pct_of_peak_sustained_active")
        out.append(f"{k:44s} {n:8d} {t:10.3f} {sum(v['gpu__time_duration.sum']) / tot:7.1%} "
                   f"{inst or 0:14.4g} {(rd + wr) / 1e9:15.3f} {iss or 0:8.1f}")
        base = k.split("<")[0]
        summ["kernels"][base] = {"kernel": k, "launches": n, "duration_ms": t, "inst_executed": inst,
                                 "dram_read": rd, "dram_write": wr, "issue_active_pct": iss}
    with open(os.path.join(HERE, "r2_launches_summary.txt"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    with open(os.path.join(HERE, "r2_ncu_summary.json"), "w") as fh:
        json.dump(summ, fh, indent=1)
    print("\n".join(out))


METRICS = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
           "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
           "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
           "Executed Instructions", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
           "Static Shared Memory Per Block")


def full(src):
    out = ["# r2: ncu --set full --clock-control none (profiles/profile_r2.sh): simulator, row statistics,",
           "# stream kernel (config 2 bench sweep) and GBP/GCA (config 4, 2000 instances per regime)"]
    comp = {}
    for name in ("prof_seg", "prof_stats", "prof_streams", "prof_compose_moderate", "prof_compose_full"):
        rep = os.path.join(src, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        regime = name.split("_")[-1] if name.startswith("prof_compose") else None
        txt = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
        kernel = None
        for line in txt.splitlines():
            if "Context" in line and "Stream" in line and "(" in line:
                kernel = short(line.strip())
                out.append(f"\n== {kernel}" + (f"  [config 4, {regime}]" if regime else ""))
            s = line.strip()
            for m in METRICS:
                if s.startswith(m + " ") or s.startswith(m + "  "):
                    out.append("  " + " ".join(s.split()))
                    if regime and kernel and m in ("Issue Slots Busy", "Duration",
                                                   "Executed Instructions", "Achieved Occupancy"):
                        comp.setdefault(regime, {}).setdefault(kernel.split("<")[0], {})[m] = \
                            " ".join(s.split()[len(m.split()):])
    with open(os.path.join(HERE, "r2_ncu_full_summary.txt"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    if comp:
        comp["source"] = ("profiles/profile_r2.sh: ncu --set full, bench_compose.py --regime "
                          "{moderate,full} --instances 2000")
        with open(os.path.join(HERE, "r2_ncu_compose.json"), "w") as fh:
            json.dump(comp, fh, indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(HERE), "gpurun_out")
    launches(src)
    full(src)
