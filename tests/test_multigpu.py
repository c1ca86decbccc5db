"""Multi-rank paths.

* CPU (gloo, world size 2): replication sharding keeps every replication's
  reference spawn key, and the host-side merge of per-rank summaries gives the
  same statistics as one process (checked with the CPU oracle).
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
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2604_14993_b200 import distributed as D
    from paper_2604_14993_b200 import sim as S

    rates, caps, lam, n, wf, seed, R = (1.5, 0.6), (2, 3), 2.0, 4000, 0.1, 7, 8
    begin, count = D.shard(R, rank, world)
    resp, busy, summ = O.simulate_reps(rates, caps, lam, n, wf, seed, begin, begin + count, threads=1)
    local = [dict(wait_sum=s.wait_sum, service_sum=s.service_sum, counted=s.counted,
                  window_s=s.window_s, mean_occupancy=s.mean_occupancy,
                  occ_first_half=s.occ_first_half, occ_second_half=s.occ_second_half,
                  lambda_effective=s.lambda_effective, end_queue_len=s.end_queue_len,
                  resp_sum=float(np.add.reduce(row)), resp_mean=float(row.mean()))
             for s, row in zip(summ, resp)]
    gathered = [None] * world
    dist.all_gather_object(gathered, (local, busy.tolist(), resp.ravel().tolist()))
    if rank == 0:
        rows = [r for part in gathered for r in part[0]]
        summ_all = np.zeros(len(rows), dtype=[(k, np.float64 if k not in ("counted", "end_queue_len")
                                               else np.int64) for k in rows[0]])
        for i, r in enumerate(rows):
            for k, v in r.items():
                summ_all[i][k] = v
        busy_all = np.array([b for part in gathered for b in part[1]])
        merged = np.sort(np.array([x for part in gathered for x in part[2]]))
        order = {k: float(merged[k]) for q in S.QUANTILES for k in S._quantile_ranks(merged.size, q)[:2]}
        cfg = S.SimConfig(rates=rates, capacities=caps, workload=S.PoissonWorkload(lam),
                          horizon_jobs=n, warmup_fraction=wf, seed=seed, replications=R)
        got = S._stats_from(cfg, summ_all, busy_all, order, None).to_dict()
        ref = O.run_sim_stats(rates, caps, lam, n, wf, seed, R, threads=2)
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
    got, ref = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
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
