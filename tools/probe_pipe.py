"""Kernel timeline of SweepEngine.run_pipelined on config 2 (development probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2604_14993_b200 as P
    from paper_2604_14993_b200.engine import SweepEngine

    service, servers, _ = P.petals_instance(10, 0.2, 101)
    s = P.greedy_cache_allocation(P.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
    lams = [s.total_rate * x for x in np.linspace(0.05, 0.95, 16)]
    e = SweepEngine([s.rates] * 16, [s.capacities] * 16, lams, 100000, 0.1, 1, 1024)
    e.run_pipelined(3)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    e.run_pipelined(6)
    b.record()
    b.synchronize()
    print("pipelined ms/step", a.elapsed_time(b) / 6)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e.run_pipelined(4)
        torch.cuda.synchronize()
    evs = [x for x in prof.events() if x.device_type.name == "CUDA"]
    t0 = min(x.time_range.start for x in evs)
    for x in sorted(evs, key=lambda x: x.time_range.start):
        d = x.time_range.end - x.time_range.start
        if d > 20:
            print(f"{(x.time_range.start - t0) / 1e3:8.3f} -> {(x.time_range.end - t0) / 1e3:8.3f} ms "
                  f"{d / 1e3:7.3f}  {x.name[:60]}")


if __name__ == "__main__":
    main()
