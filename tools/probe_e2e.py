import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2604_14993_b200 as P
from paper_2604_14993_b200 import sim as S
service, servers, _ = P.petals_instance(10, 0.2, 101)
s = P.greedy_cache_allocation(P.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
lams = [s.total_rate * x for x in np.linspace(0.05, 0.95, 16)]
cfgs = [P.SimConfig(rates=s.rates, capacities=s.capacities, workload=P.PoissonWorkload(l), horizon_jobs=100000, warmup_fraction=0.1, seed=1, replications=1024) for l in lams]
for i in range(4):
    t0 = time.perf_counter(); r = P.simulate_sweep([s.rates]*16, [s.capacities]*16, lams, 100000, 0.1, 1, 1024); t1 = time.perf_counter()
    st = S._stats_from_batch(cfgs, r.summaries, r.busy, r.order_stats, None); t2 = time.perf_counter()
    print(f"simulate_sweep {t1-t0:.4f} s, stats_from_batch {t2-t1:.4f} s", flush=True)
if len(sys.argv) > 1:
    import torch
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        r = P.simulate_sweep([s.rates]*16, [s.capacities]*16, lams, 100000, 0.1, 1, 1024)
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" or "cuda" in e.name.lower()]
    t0 = min(e.time_range.start for e in prof.events())
    for e in sorted(prof.events(), key=lambda e: e.time_range.start):
        d = e.time_range.end - e.time_range.start
        if d > 200 or e.device_type.name == "CUDA":
            print(f"{(e.time_range.start - t0)/1e3:9.3f} ms  {d/1e3:8.3f} ms  {e.device_type.name:5s} {e.name[:80]}")
