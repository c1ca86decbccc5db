"""Stage timings of one sweep shape on the GPU (development probe).

    python tools/probe_sim.py [--jobs N --reps R --points P --sweeps K]

Prints per-stage device times of SweepEngine.step() for the default
(segmented) single-chain simulator and for CS_SIM_EXACT=1, and checks that
both give the same order statistics and per-replication means.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=1024)
    ap.add_argument("--points", type=int, default=16)
    ap.add_argument("--sweeps", type=int, default=4)
    ap.add_argument("--rho", type=float, default=None, help="single point at this load")
    ap.add_argument("--modes", default="seg,exact")
    a = ap.parse_args()
    import torch

    import paper_2604_14993_b200 as P
    from paper_2604_14993_b200.engine import SweepEngine

    service, servers, _ = P.petals_instance(10, 0.2, 101)
    system = P.greedy_cache_allocation(P.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
    nu = system.total_rate
    if a.rho is not None:
        lams = [a.rho * nu] * a.points
    else:
        lams = [nu * x for x in np.linspace(0.05, 0.95, a.points)]
    from paper_2604_14993_b200 import _native as N

    print("plan", N.seg_plan(a.points, a.reps, int(sum(system.capacities)), a.jobs))
    out = {}
    for mode in a.modes.split(","):
        os.environ["CS_SIM_EXACT"] = "1" if mode == "exact" else "0"
        e = SweepEngine([system.rates] * a.points, [system.capacities] * a.points, lams, a.jobs, 0.1, 1,
                        a.reps)
        e.step()
        torch.cuda.synchronize()
        times = [e.step(timed=True) for _ in range(a.sweeps)]
        summ = e.summaries(0).copy()
        out[mode] = {"streams_ms": [round(t.streams_ms, 3) for t in times],
                     "sim_ms": [round(t.sim_ms, 3) for t in times],
                     "stats_ms": [round(t.stats_ms, 3) for t in times],
                     "jobs_per_s_sim": a.points * a.reps * a.jobs / (np.median([t.sim_ms for t in times]) / 1e3),
                     "order_stats": e.order_stats(), "rep_means": summ["resp_mean"]}
        del e
        torch.cuda.empty_cache()
    modes = list(out)
    if len(modes) == 2:
        x, y = out[modes[0]], out[modes[1]]
        print("order stats equal:", x["order_stats"] == y["order_stats"])
        print("rep means equal:", np.array_equal(x["rep_means"].view(np.uint64), y["rep_means"].view(np.uint64)))
    for m in modes:
        d = {k: v for k, v in out[m].items() if k not in ("order_stats", "rep_means")}
        print(m, json.dumps(d))


if __name__ == "__main__":
    main()
