"""The rest of run_sim's signature on the GPU
(csrc/sim_ext.cu) against golden outputs of the reference's own
_simulate_once / run_sim (tests/golden/make_golden_ext.py): dedicated-queue
policies jsq / sa-jsq / jiq / sed, the time-horizon Poisson mode, sampled and
trace workloads.  Everything bit-exact except the merged mean (<= 1e-12 rel,
as for the jffc path)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, bits, same_float

FIELDS = ("wait_sum", "service_sum", "counted", "window_s", "mean_occupancy", "occ_first_half",
          "occ_second_half", "lambda_effective", "end_queue_len")


@pytest.fixture(scope="module")
def gx():
    with open(os.path.join(GOLDEN, "golden_ext.json")) as fh:
        meta = json.load(fh)
    return meta, dict(np.load(os.path.join(GOLDEN, "golden_ext.npz")))


_TRACE = {}


def _trace_system(P, comp):
    """The trace cases' chains: the PETALS fixture composed on the GPU (the
    composition itself is pinned bit-exact by test_gpu_parity)."""
    if "sys" not in _TRACE:
        service, servers, model = P.petals_instance(10, 0.2, 101)
        placed = P.greedy_block_placement(servers, service, comp["capacity"], comp["arrival_rate"],
                                          comp["load_target"])
        _TRACE["sys"] = (P.greedy_cache_allocation(placed.placement), model)
    return _TRACE["sys"]


def _config(P, meta, arrs, c, reps, collect):
    wd = c["workload"]
    kw = dict(rates=tuple(c["rates"]), capacities=tuple(c["caps"]), policy=c["policy"],
              horizon_jobs=c["n"], warmup_fraction=c["wf"], seed=c["seed"], replications=reps,
              horizon_time_s=c["horizon"], collect_jobs=collect)
    if wd["kind"] == "poisson":
        kw["workload"] = P.PoissonWorkload(wd["lam"])
    elif wd["kind"] == "sampled":
        kw["workload"] = P.SampledWorkload(tuple(arrs["sampled_arrivals"].tolist()),
                                           tuple(arrs["sampled_sizes"].tolist()))
    else:
        system, model = _trace_system(P, meta["trace_composition"])
        assert list(system.rates) == meta["trace_composition"]["rates"]
        recs = tuple(P.TraceRecord(float(a), int(i), int(o)) for a, i, o in
                     zip(arrs["trace_arrivals"], arrs["trace_tin"], arrs["trace_tout"]))
        kw.update(workload=P.TraceWorkload(recs), chains=system.chains, service_model=model)
    return P.SimConfig(**kw)


def test_golden_ext_is_loadable(gx):
    meta, arrs = gx
    assert len(meta["cases"]) >= 70 and len(meta["runsim"]) == 4
    for c in meta["cases"]:
        for r in c["reps"]:
            assert r["responses"] in arrs and r["busy"] in arrs


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(75))
def test_simulate_ext_matches_reference(gx, idx):
    import paper_2604_14993_b200 as P
    from paper_2604_14993_b200.sim_ext import simulate_ext

    meta, arrs = gx
    c = meta["cases"][idx]
    collect = "jobs" in c["reps"][0]
    R = max(r["rep"] for r in c["reps"]) + 1
    cfg = _config(P, meta, arrs, c, R, collect)
    summ, busy, _, jobs, resp = simulate_ext(cfg, return_responses=True)
    for rr in c["reps"]:
        r = rr["rep"]
        assert np.array_equal(bits(resp[r]), bits(arrs[rr["responses"]])), (c["tag"], r)
        assert np.array_equal(bits(busy[r]), bits(arrs[rr["busy"]])), (c["tag"], r)
        for f in FIELDS:
            assert same_float(summ[r][f], rr["fields"][f]), (c["tag"], r, f)
        if collect:
            assert np.array_equal(bits(jobs[r]), bits(arrs[rr["jobs"]])), (c["tag"], r)


@pytest.mark.gpu
def test_horizon_errors_match_reference(gx):
    import paper_2604_14993_b200 as P

    meta, _ = gx
    for e in meta["errors"]:
        cfg = P.SimConfig(rates=(1.0,), capacities=(1,), workload=P.PoissonWorkload(e["lam"]),
                          horizon_jobs=e["n"], warmup_fraction=e["wf"], horizon_time_s=e["horizon"],
                          seed=1)
        with pytest.raises(ValueError) as ei:
            P.run_sim(cfg)
        assert str(ei.value) == e["message"]


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(4))
def test_run_sim_ext_matches_reference(gx, i):
    import paper_2604_14993_b200 as P

    meta, arrs = gx
    c = meta["runsim"][i]
    st = P.run_sim(_config(P, meta, arrs, c, c["reps"], False)).to_dict()
    for k, v in c["stats"].items():
        g = st[k]
        if k == "mean_response_s":
            assert abs(g - v) <= 1e-12 * abs(v), (g, v)
        elif k == "little_law_gap":
            assert abs(g - v) <= 1e-9 * max(abs(v), 1e-12), (g, v)
        elif isinstance(v, list):
            assert len(g) == len(v) and all(same_float(a, b) for a, b in zip(g, v)), (k, g, v)
        elif isinstance(v, float):
            assert same_float(g, v), (k, g, v)
        else:
            assert g == v, (k, g, v)


def _random_system(rng, K, C):
    rates = tuple(sorted((float(x) for x in rng.uniform(0.2, 2.0, K)), reverse=True))
    caps = [1] * K
    for _ in range(C - K):
        caps[int(rng.integers(K))] += 1
    return rates, tuple(caps)


EXT_RANDOM = [(K, C, pol, rho, hz) for (K, C) in ((1, 3), (3, 9), (12, 40), (40, 100))
              for pol in ("jffc", "jsq", "jiq", "sed") for rho, hz in ((0.6, None), (0.97, None),
                                                                       (1.2, 2500.0))]


@pytest.mark.gpu
@pytest.mark.parametrize("K,C,pol,rho,hz", EXT_RANDOM)
def test_simulate_ext_matches_oracle(oracle, K, C, pol, rho, hz):
    """Fresh seeded configurations beyond the golden ones (K up to 40 chains,
    overloaded systems with long dedicated queues, time horizon): GPU vs the
    pinned oracle, bit-exact."""
    import paper_2604_14993_b200 as P
    from conftest import ext_inputs
    from paper_2604_14993_b200.sim_ext import simulate_ext

    rng = np.random.default_rng(K * 7919 + C)
    rates, caps = _random_system(rng, K, C)
    nu = sum(r * c for r, c in zip(rates, caps))
    lam = rho * nu
    n, wf, seed, R = 4000, 0.1, 17, 3
    t_end = None if hz is None else hz / lam
    cfg = P.SimConfig(rates=rates, capacities=caps, workload=P.PoissonWorkload(lam), policy=pol,
                      horizon_jobs=n, horizon_time_s=t_end, warmup_fraction=wf, seed=seed,
                      replications=R, collect_jobs=True)
    summ, busy, _, jobs, resp = simulate_ext(cfg, return_responses=True, queue_capacity=64)
    c = {"workload": {"kind": "poisson", "lam": lam}, "n": n, "wf": wf, "horizon": t_end,
         "seed": seed}
    for r in range(R):
        arr, warm, sizes, _ = ext_inputs(oracle, c, {}, r)
        o = oracle.simulate_ext(rates, caps, pol, arr, warm, sizes, None, collect_jobs=True)
        assert np.array_equal(bits(resp[r]), bits(o["responses"])), r
        assert np.array_equal(bits(busy[r]), bits(o["busy_time_s"])), r
        assert np.array_equal(bits(jobs[r]), bits(o["jobs"])), r
        for f in FIELDS:
            assert same_float(summ[r][f], o[f]), (r, f)
