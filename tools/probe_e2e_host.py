"""Host-side profile of one config-2 run_sim_batch call (development probe)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2604_14993_b200 as P

service, servers, _ = P.petals_instance(10, 0.2, 101)
s = P.greedy_cache_allocation(P.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
lams = [s.total_rate * x for x in np.linspace(0.05, 0.95, 16)]
cfgs = [P.SimConfig(rates=s.rates, capacities=s.capacities, workload=P.PoissonWorkload(l), horizon_jobs=100000,
                    warmup_fraction=0.1, seed=1, replications=1024) for l in lams]
for _ in range(3):
    P.run_sim_batch(cfgs)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    P.run_sim_batch(cfgs)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
