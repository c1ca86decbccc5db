"""Multi-rank paths.

* CPU (gloo, world size 2): replication sharding keeps every replication's
  reference spawn key, and the sharded sweep's own host side
  (distributed.merge_sharded: the all-gather of the per-rank summary and busy
  buffers along the replication axis + the aggregation) gives the same
  statistics as one process (per-rank inputs from the CPU oracle).
* GPU (>= 2 devices): the sharded engine (NCCL all-gather + all-reduced
  radix-select histograms) equals the single-GPU engine field for field.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, same_float


def _gloo_worker(rank, world, port, q):
    """Each rank holds the summaries of its replication shard in the engine's
    device layout ([P, R/world] cs_rep_summary records, [P, R/world, ldb]
    busy times, point-major) -- produced here by the CPU oracle -- and runs
    the sharded sweep's own host side, distributed.merge_sharded (the
    all-gather along the replication axis + the reference's aggregation)."""
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2604_14993_b200 import _native as N
    from paper_2604_14993_b200 import distributed as D
    from paper_2604_14993_b200 import sim as S

    rates, caps, n, wf, seed, R = (1.5, 0.6), (2, 3), 4000, 0.1, 7, 8
    lams = (2.0, 3.1)
    ldb = len(rates)
    begin, count = D.shard(R, rank, world)
    summ = np.zeros((len(lams), count), N.SUMMARY_DTYPE)
    busy = np.zeros((len(lams), count, ldb))
    order = []
    for p, lam in enumerate(lams):
        resp, b, sm = O.simulate_reps(rates, caps, lam, n, wf, seed, begin, begin + count, threads=1)
        for r, (x, row) in enumerate(zip(sm, resp)):
            for f in ("wait_sum", "service_sum", "counted", "window_s", "mean_occupancy", "occ_first_half",
                      "occ_second_half", "lambda_effective", "end_queue_len"):
                summ[p, r][f] = getattr(x, f)
            summ[p, r]["resp_sum"] = float(np.add.reduce(row))
            summ[p, r]["resp_mean"] = float(row.mean())
        busy[p] = b
        # global order statistics (cs_rep_stats_dist's result): from the full run
        full, _, _ = O.simulate_reps(rates, caps, lam, n, wf, seed, 0, R, threads=1)
        merged = np.sort(full.ravel())
        order.append({k: float(merged[k]) for q in S.QUANTILES for k in S._quantile_ranks(merged.size, q)[:2]})
    cfgs = [S.SimConfig(rates=rates, capacities=caps, workload=S.PoissonWorkload(lam), horizon_jobs=n,
                        warmup_fraction=wf, seed=seed, replications=R) for lam in lams]
    t_summ = torch.from_numpy(summ.view(np.uint8).ravel().copy())
    t_busy = torch.from_numpy(busy.ravel().copy())
    got = [s.to_dict() for s in D.merge_sharded(cfgs, t_summ, t_busy, order, ldb)]
    if rank == 0:
        ref = [O.run_sim_stats(rates, caps, lam, n, wf, seed, R, threads=2) for lam in lams]
        q.put((got, ref))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_merge_matches_single_process_gloo():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got_all, ref_all = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got_all) == len(ref_all) == 2
    for got, ref in zip(got_all, ref_all):
        for k, v in ref.items():
            g = got[k]
            if k in ("mean_response_s", "little_law_gap"):
                assert abs(g - v) <= 1e-12 * max(abs(v), 1e-300), (k, g, v)
            elif isinstance(v, (list, tuple)):
                assert all(same_float(a, b) for a, b in zip(g, v)), k
            elif isinstance(v, float):
                assert same_float(g, v), (k, g, v)
            else:
                assert g == v, (k, g, v)


def test_shard_requires_equal_blocks():
    from paper_2604_14993_b200 import distributed as D

    assert D.shard(1024, 3, 8) == (384, 128)
    with pytest.raises(ValueError):
        D.shard(10, 0, 4)


@pytest.mark.gpu
def test_sharded_engine_matches_single_gpu():
    import torch

    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 4)}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + os.getpid() % 300),
           os.path.join(ROOT, "tests", "helpers", "mgpu_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
