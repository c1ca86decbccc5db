"""Kernel timeline of one config-5 simulate_sweep call (development probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2604_14993_b200 as P

    service, servers, _ = P.petals_instance(10, 0.2, 101)
    s = P.greedy_cache_allocation(P.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
    lam = 0.7 * s.total_rate
    P.simulate_sweep([s.rates], [s.capacities], [lam], 1_000_000, 0.1, 1, 8192, max_stream_bytes=64 << 30)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        P.simulate_sweep([s.rates], [s.capacities], [lam], 1_000_000, 0.1, 1, 8192, max_stream_bytes=64 << 30)
        torch.cuda.synchronize()
    evs = [x for x in prof.events() if x.device_type.name == "CUDA"]
    t0 = min(x.time_range.start for x in evs)
    for x in sorted(evs, key=lambda x: x.time_range.start):
        d = x.time_range.end - x.time_range.start
        if d > 50:
            print(f"{(x.time_range.start - t0) / 1e3:9.3f} -> {(x.time_range.end - t0) / 1e3:9.3f} ms "
                  f"{d / 1e3:8.3f}  {x.name[:70]}")


if __name__ == "__main__":
    main()
