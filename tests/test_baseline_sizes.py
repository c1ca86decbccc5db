"""Parity at the BASELINE.json configs' real sizes (GPU vs the pinned CPU
oracle on the same seeded inputs):

* config 2: the full headline sweep, 16 arrival rates x 1024 replications x
  1e5 jobs on the PETALS composition -- every response row, order statistic
  and rep mean bit-exact, summaries as in test_seg_sim;
* config 3: the c-grid compositions of fleet(J=100, L=80, seed=7) (K up to
  ~50 chains, the warp-per-replication kernel) at rho 0.7, 1e5 jobs x 64
  replications -- bit-exact in every field;
* config 4: 1000-server fleets through GBP-CR + GCA, 16 instances in each
  lambda regime (moderate and full fleet) -- placements, chains, capacities,
  service times and edge counts bit-exact;
* config 5: the config-1 composition at rho 0.7, 1e6 jobs x 32 replications.

These run the oracle on every host thread; about a minute on the B200 box.
"""

import concurrent.futures as cf
import os

import numpy as np
import pytest

from conftest import SUM_FIELDS, bits, close_rel, same_float

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

EXACT_FIELDS = ("counted", "window_s", "lambda_effective", "end_queue_len")
ALL_FIELDS = EXACT_FIELDS + SUM_FIELDS


@pytest.fixture(scope="module")
def eng():
    import paper_2604_14993_b200 as P
    from paper_2604_14993_b200 import _native as N

    assert N.load().cs_device_count() >= 1
    return P


def _petals(eng):
    service, servers, _ = eng.petals_instance(10, 0.2, 101)
    return eng.greedy_cache_allocation(
        eng.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)


def _check_summary(s, ref, busy_got, busy_ref, seg):
    for f in ALL_FIELDS:
        g, r = s[f], getattr(ref, f)
        ok = close_rel(g, r) if (seg and f in SUM_FIELDS) else same_float(g, r)
        assert ok, (f, g, r)
    for x, y in zip(busy_got, busy_ref):
        assert close_rel(x, y) if seg else same_float(x, y), (x, y)


def test_config2_full_sweep(eng, oracle):
    """16 x 1024 x 1e5 = 1.64e9 jobs, device-resident (SweepEngine, the
    benchmark's path), every row compared."""
    import torch

    from paper_2604_14993_b200.engine import SweepEngine

    system = _petals(eng)
    nu = system.total_rate
    lams = [nu * x for x in np.linspace(0.05, 0.95, 16)]
    n, wf, seed, R = 100_000, 0.1, 1, 1024
    e = SweepEngine([system.rates] * 16, [system.capacities] * 16, lams, n, wf, seed, R)
    e.step()
    torch.cuda.synchronize()
    summ, busy, ostats = e.summaries(0), e.busy(0), e.order_stats()
    rows = e.sets[0]["resp"].view(16, R, e.ldr)
    for p in range(16):
        resp, rbusy, rsumm = oracle.simulate_reps(system.rates, system.capacities, lams[p], n, wf, seed, 0, R)
        got = rows[p, :, :e.m].cpu().numpy()
        assert np.array_equal(bits(got), bits(resp)), p
        for r in range(R):
            _check_summary(summ[p, r], rsumm[r], busy[p, r, :1], rbusy[r], seg=True)
            assert same_float(summ[p, r]["resp_mean"], resp[r].mean()), (p, r)
        merged = np.sort(resp.ravel())
        for rank, v in ostats[p].items():
            assert same_float(v, merged[rank]), (p, rank)
        del resp, got, merged


def test_config3_c_grid(eng, oracle):
    """fleet(J=100, L=80, seed=7): c swept through GBP+GCA (batched), the
    composed points of a 16-value c grid simulated at rho 0.7."""
    service, servers = eng.fleet(100, 80, seed=7)
    grid = [1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 14, 16, 20, 24, 28, 32]
    placed = eng.greedy_block_placement_batch([servers] * len(grid), [service] * len(grid), grid,
                                              [1e9] * len(grid), [0.7] * len(grid))
    systems = eng.greedy_cache_allocation_batch([p.placement for p in placed])
    pts = [(s.rates, s.capacities) for s in systems if s.chains]
    assert len(pts) >= 12 and max(len(r) for r, _ in pts) > 8
    lams = [0.7 * sum(r * c for r, c in zip(*pt)) for pt in pts]
    n, R = 100_000, 64
    res = eng.simulate_sweep([p[0] for p in pts], [p[1] for p in pts], lams, n, 0.1, 1, R,
                             return_responses=True)
    for p, (rates, caps) in enumerate(pts):
        resp, rbusy, rsumm = oracle.simulate_reps(rates, caps, lams[p], n, 0.1, 1, 0, R)
        assert np.array_equal(bits(res.responses[p]), bits(resp)), p
        K = len(rates)
        assert np.array_equal(bits(res.busy[p][:, :K]), bits(rbusy)), p
        for r in range(R):
            _check_summary(res.summaries[p, r], rsumm[r], [], [], seg=False)
        merged = np.sort(resp.ravel())
        for rank, v in res.order_stats[p].items():
            assert same_float(v, merged[rank]), (p, rank)


def _oracle_compose(args):
    from oracle import oracle as O
    from paper_2604_14993_b200.compose_engine import fleet_soa

    seed, lam = args
    mem, tc, tp = fleet_soa(1000, 80, seed)
    ids = [f"n{i:04d}" for i in range(1000)]
    st, g = O.gbp(mem, tc, tp, ids, 80, int(1.32e9), int(0.11e9), 7, lam, 0.7)
    st2, a = O.gca(mem, tc, tp, ids, 80, int(1.32e9), int(0.11e9), g["first"], g["count"])
    return st, g, st2, a


@pytest.mark.parametrize("lam", [5.0, 1e9], ids=["moderate", "full_fleet"])
def test_config4_thousand_server_fleets(eng, oracle, lam):
    from paper_2604_14993_b200.compose_engine import ComposeEngine, fleet_soa

    n_inst = 16
    parts = [fleet_soa(1000, 80, s) for s in range(n_inst)]
    ce = ComposeEngine(np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]),
                       np.concatenate([p[2] for p in parts]), 1000, 80, int(1.32e9), int(0.11e9), 7, lam,
                       0.7, max_chains=64 if lam < 1e6 else 512)
    ce.run()
    res = ce.results()
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:  # the oracle releases the GIL
        refs = list(ex.map(_oracle_compose, [(s, lam) for s in range(n_inst)]))
    for seed, (st, g, st2, a) in enumerate(refs):
        assert st == 0 and st2 == 0
        assert int(res["gbp_status"][seed]) == 0 and int(res["gca_status"][seed]) == 0
        k = int(res["n_chains"][seed])
        assert k == len(a["caps"]), seed
        assert list(res["caps"][seed, :k]) == list(a["caps"]), seed
        assert np.array_equal(bits(res["times"][seed, :k]), bits(a["times"])), seed
        assert int(res["n_edges"][seed]) == int(a["n_edges"]), seed
        assert list(res["first"][seed]) == list(g["first"]), seed
        assert list(res["count"][seed]) == list(g["count"]), seed
        got = [list(res["chain_srv"][seed, q, :res["chain_len"][seed, q]]) for q in range(k)]
        assert got == [list(c) for c in a["chains"]], seed


def test_config5_long_replications(eng, oracle):
    system = _petals(eng)
    lam = 0.7 * system.total_rate
    n, R = 1_000_000, 32
    res = eng.simulate_sweep([system.rates], [system.capacities], [lam], n, 0.1, 1, R, return_responses=True)
    resp, rbusy, rsumm = oracle.simulate_reps(system.rates, system.capacities, lam, n, 0.1, 1, 0, R)
    assert np.array_equal(bits(res.responses[0]), bits(resp))
    for r in range(R):
        _check_summary(res.summaries[0, r], rsumm[r], res.busy[0, r, :1], rbusy[r], seg=True)
        assert same_float(res.summaries[0, r]["resp_mean"], resp[r].mean()), r
    merged = np.sort(resp.ravel())
    for rank, v in res.order_stats[0].items():
        assert same_float(v, merged[rank]), rank
