#!/usr/bin/env python
"""Secondary benchmark lines for BASELINE configs 3 and 5 (the headline is
bench.py, config 2).  Device-timed with CUDA events, one JSON line each.

config 3: LLaMA-2-70B-like service (L=80) over a 100-server two-tier fleet
  (workload.fleet(100, 80, seed=7)).  The design parameter c is swept over
  [1, c_max] through GBP-CR + GCA in one batched launch each; a grid of
  composed points (every feasible c in `--c-grid`) is then simulated at load
  rho=0.7 (lambda = 0.7 * nu(c)) x `--reps` replications x 1e5 jobs.
config 5: the config-1 composition (PETALS J=10, c=7: K=1, C=7) at
  lambda = 0.7 nu, 1e6 jobs x `--reps5` replications (1 GPU here; bench.py
  --gpus N covers the multi-GPU sharding).

    python bench_configs.py [--config 3|5|both]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def run_sweep(rates_list, caps_list, lams, n, reps, steps):
    import torch

    from paper_2604_14993_b200.engine import SweepEngine

    eng = SweepEngine(rates_list, caps_list, lams, n, 0.1, 1, reps)
    eng.step()
    torch.cuda.synchronize()
    times = [eng.step(timed=True) for _ in range(steps)]
    st = {k: float(np.mean([getattr(t, k) for t in times])) for k in ("streams_ms", "sim_ms", "stats_ms")}
    total = sum(st.values())
    return eng, st, total


def config3(args):
    import paper_2604_14993_b200 as P
    from paper_2604_14993_b200 import _compose as CE

    service, servers = P.fleet(100, 80, seed=7)
    c_max = P.capacity_upper_bound(servers, service)
    fleet = CE.Fleet.of(servers)
    caps_grid = list(range(1, c_max + 1))
    t0 = time.perf_counter()
    gbp = CE.gbp_batch([fleet], [service] * len(caps_grid), caps_grid, [1e9] * len(caps_grid),
                       [0.7] * len(caps_grid), fleet_of_point=[0] * len(caps_grid))
    feas = [p for p in range(len(caps_grid)) if gbp.status[p] == 0]
    firsts = [gbp.first[gbp.server_base[p]:gbp.server_base[p] + 100] for p in feas]
    counts = [gbp.count[gbp.server_base[p]:gbp.server_base[p] + 100] for p in feas]
    gca = CE.gca_batch([fleet], [service] * len(feas), firsts, counts, fleet_of_point=[0] * len(feas))
    compose_s = time.perf_counter() - t0
    want = [int(x) for x in args.c_grid.split(",")]
    pts = []
    for idx, p in enumerate(feas):
        c = caps_grid[p]
        K = int(gca.n_chains[idx])
        if c in want and K > 0:
            caps = [int(x) for x in gca.caps[idx, :K]]
            rates = [1.0 / float(x) for x in gca.times[idx, :K]]
            pts.append((c, rates, caps))
    lams = [0.7 * sum(r * c for r, c in zip(rates, caps)) for _, rates, caps in pts]
    eng, st, total = run_sweep([p[1] for p in pts], [p[2] for p in pts], lams, args.jobs, args.reps,
                               args.steps)
    jobs = len(pts) * args.reps * args.jobs
    return {
        "metric": "simulated jobs/sec (JFFC over composed chains)", "config": "3",
        "value": jobs / (total / 1e3), "unit": "jobs/s", "n_gpus": 1, "ms_per_step": total,
        "stages_ms": st,
        "workload": {"fleet": "fleet(J=100, L=80, seed=7)", "c_max": c_max,
                     "compose_sweep": f"{len(caps_grid)} c values, GBP+GCA batched, {compose_s:.3f} s incl. host",
                     "points": [{"c": c, "K": len(r), "C": sum(cp)} for c, r, cp in pts],
                     "rho": 0.7, "reps": args.reps, "jobs": args.jobs,
                     "kernel": "generic" if max(len(p[1]) for p in pts) > 8 or max(sum(p[2]) for p in pts) > 16
                     else "register"},
    }


def config5(args):
    import paper_2604_14993_b200 as P

    service, servers, _ = P.petals_instance(10, 0.2, 101)
    system = P.greedy_cache_allocation(P.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
    lam = 0.7 * system.total_rate
    eng, st, total = run_sweep([system.rates], [system.capacities], [lam], args.jobs5, args.reps5, 1)
    jobs = args.reps5 * args.jobs5
    return {
        "metric": "simulated jobs/sec (JFFC over composed chains)", "config": "5 (1 GPU)",
        "value": jobs / (total / 1e3), "unit": "jobs/s", "n_gpus": 1, "ms_per_step": total,
        "stages_ms": st,
        "workload": {"composition": "PETALS J=10 c=7 (K=1, C=7)", "lambda": "0.7 nu", "reps": args.reps5,
                     "jobs": args.jobs5},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="both", choices=["3", "5", "both"])
    ap.add_argument("--reps", type=int, default=4096)
    ap.add_argument("--jobs", type=int, default=100_000)
    ap.add_argument("--c-grid", default="1,2,3,4,5,6,7,8,10,12,14,16,20,24,28,32")
    ap.add_argument("--reps5", type=int, default=1024)
    ap.add_argument("--jobs5", type=int, default=1_000_000)
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    if a.config in ("3", "both"):
        print(json.dumps(config3(a)), flush=True)
    if a.config in ("5", "both"):
        print(json.dumps(config5(a)), flush=True)


if __name__ == "__main__":
    main()
