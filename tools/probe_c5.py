"""Wall time of BASELINE config 5 through the public API (development probe).

    python tools/probe_c5.py [--reps 8192] [--calls 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=8192)
    ap.add_argument("--calls", type=int, default=3)
    ap.add_argument("--stream-gib", type=int, default=34)
    a = ap.parse_args()
    import paper_2604_14993_b200 as P

    service, servers, _ = P.petals_instance(10, 0.2, 101)
    s = P.greedy_cache_allocation(P.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
    lam = 0.7 * s.total_rate
    for c in range(a.calls):
        t0 = time.perf_counter()
        r = P.simulate_sweep([s.rates], [s.capacities], [lam], 1_000_000, 0.1, 1, a.reps,
                             max_stream_bytes=a.stream_gib << 30)
        dt = time.perf_counter() - t0
        print(f"call {c}: {dt:.3f} s  {a.reps * 1e6 / dt:.3e} jobs/s  p99={r.order_stats[0]}", flush=True)


if __name__ == "__main__":
    main()
