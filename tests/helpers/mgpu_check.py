"""torchrun helper for tests/test_multigpu.py: sharded run_sim over all ranks
must equal the single-GPU run_sim_batch on rank 0, field for field; and the
sharded SweepEngine's pipelined sweeps (the benchmark loop) must equal its
unpipelined step() (summaries, busy times, global order statistics)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2604_14993_b200 as P
    from paper_2604_14993_b200 import distributed as D

    D.init()
    service, servers, _ = P.petals_instance(10, 0.2, 101)
    system = P.greedy_cache_allocation(P.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
    nu = system.total_rate
    world = dist.get_world_size()
    cfgs = [P.SimConfig(rates=system.rates, capacities=system.capacities,
                        workload=P.PoissonWorkload(f * nu), horizon_jobs=12000, warmup_fraction=0.1,
                        seed=1, replications=48 * world) for f in (0.3, 0.92)]
    sharded = D.run_sim_sharded(cfgs)
    import numpy as np

    from paper_2604_14993_b200.engine import SweepEngine

    rank, R = dist.get_rank(), 32
    eng = SweepEngine([system.rates] * 2, [system.capacities] * 2, [0.4 * nu, 0.9 * nu], 10_000, 0.1, 1, R,
                      rep_begin=rank * R, distributed=True, total_reps=world * R)
    eng.step()
    torch.cuda.synchronize()
    ref = (eng.summaries(0).copy(), eng.busy(0).copy(), eng.order_stats())
    last = eng.run_pipelined(3)
    torch.cuda.synchronize()
    pipe_ok = (np.array_equal(eng.summaries(last).view(np.uint8), ref[0].view(np.uint8))
               and np.array_equal(eng.busy(last), ref[1]) and eng.order_stats() == ref[2])
    if dist.get_rank() == 0:
        single = P.run_sim_batch(cfgs)
        bad = []
        for a, b in zip(sharded, single):
            da, db = a.to_dict(), b.to_dict()
            for k in da:
                if da[k] != db[k] and not (k == "little_law_gap" and abs(da[k] - db[k]) < 1e-12):
                    bad.append((k, da[k] if not isinstance(da[k], list) else "list",
                                db[k] if not isinstance(db[k], list) else "list"))
        print(json.dumps({"world": world, "mismatches": bad[:10], "pipelined_ok": bool(pipe_ok)}), flush=True)
        code = 1 if bad or not pipe_ok else 0
    else:
        code = 0
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(code)


if __name__ == "__main__":
    main()
