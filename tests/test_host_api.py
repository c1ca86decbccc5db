"""Host-side behaviour of the drop-in API that needs no GPU: validation and
exceptions mirror the reference (tests/test_model.py, test_sim.py
TestValidation/TestPolicyStep of chainserve), numpy-exact host arithmetic, the
instance generators, and the unsupported-mode contract."""

import math

import numpy as np
import pytest

import paper_2604_14993_b200 as P
from paper_2604_14993_b200 import sim as S
from conftest import servers_from_rows


def test_service_and_server_validation():
    with pytest.raises(ValueError):
        P.ServiceSpec(0, 1, 1)
    with pytest.raises(ValueError):
        P.ServiceSpec(3, 1.5, 1)
    with pytest.raises(ValueError):
        P.ServerSpec("a", -1, 0.0, 0.0)
    with pytest.raises(ValueError):
        P.ServerSpec(P.HEAD_ID, 10, 0.0, 0.0)
    with pytest.raises(ValueError):
        P.ServerSpec("a", True, 0.0, 0.0)


def test_placement_validation_and_frontiers():
    svc = P.ServiceSpec(10, 10, 1)
    srv = tuple(P.ServerSpec(f"s{i}", 44, 1.0, 0.1) for i in range(3))
    pl = P.BlockPlacement(svc, srv, (1, 5, 7), (4, 4, 4))
    assert pl.frontier("s0") == 5 and pl.range_of("s2") == (7, 10)
    assert pl.frontier(P.TAIL_ID) == 12 and pl.range_of(P.HEAD_ID) == (0, 0)
    chain = P.build_chain(pl, ("s0", "s1", "s2"))
    assert chain.edges[-2].blocks_at_dst == 2
    with pytest.raises(ValueError):
        P.BlockPlacement(svc, srv, (1, 5, 8), (4, 4, 4))  # range beyond L
    with pytest.raises(ValueError):
        P.BlockPlacement(svc, (srv[0], srv[0]), (1, 1), (4, 4))  # duplicate id


def test_feasible_edges_match_golden_counts(golden):
    meta, _ = golden
    checked = 0
    for c in meta["compose_cases"]:
        if "first" not in c:
            continue
        servers = servers_from_rows(c["servers"], P)
        pl = P.BlockPlacement(P.ServiceSpec(*c["service"]), servers, tuple(c["first"]),
                              tuple(c["count"]))
        assert len(P.feasible_edges(pl)) == c["gca"]["n_edges"]
        for ids, t in zip(c["gca"]["chains"], c["gca"]["times"]):
            assert P.build_chain(pl, ids).service_time_s == t  # Neumaier sum, bit-exact
        checked += 1
    assert checked > 200


def test_policy_step_matches_reference_semantics():
    rates, caps = (2.0, 1.0, 0.5), (1, 2, 2)
    assert P.policy_step("jffc", rates, caps, [0, 0, 0], [0], ("arrival",)) == 0
    assert P.policy_step("jffc", rates, caps, [1, 2, 0], [0], ("arrival",)) == 2
    assert P.policy_step("jffc", rates, caps, [1, 2, 2], [0], ("arrival",)) is None
    assert P.policy_step("jffc", rates, caps, [1, 2, 1], [3], ("completion", 2)) == 2
    assert P.policy_step("sed", (2.0, 1.0), (5, 5), [3, 1], [0, 0], ("arrival",)) == 0
    assert P.policy_step("jsq", (2.0, 1.0), (1, 1), [1, 1], [2, 0], ("arrival",)) == 1
    assert P.policy_step("jiq", (2.0, 1.0, 0.5), (1, 1, 1), [1, 1, 1], [4, 0, 1], ("arrival",)) == 1
    with pytest.raises(ValueError):
        P.policy_step("jffc", rates, caps, [0, 0, 0], [0], ("bogus",))


def test_simconfig_validation():
    base = dict(rates=(1.0,), capacities=(1,), workload=P.PoissonWorkload(0.5))
    with pytest.raises(ValueError):
        P.SimConfig(**{**base, "policy": "round-robin"})
    with pytest.raises(ValueError):
        P.SimConfig(**{**base, "warmup_fraction": 0.6})
    with pytest.raises(ValueError):
        P.SimConfig(**{**base, "rates": (1.0, 2.0), "capacities": (1, 1)})
    with pytest.raises(ValueError):
        P.SimConfig(rates=(1.0,), capacities=(1,),
                    workload=P.TraceWorkload((P.TraceRecord(0.0, 10, 5),)))


@pytest.mark.parametrize("kw", [
    dict(policy="jsq"),
    dict(workload=P.SampledWorkload((0.0,), (1.0,))),
    dict(horizon_time_s=10.0),
])
def test_extended_modes_have_no_cpu_path(kw):
    """Policies / sampled / horizon run on the GPU (sim_ext.cu) or not at all:
    without a device the call fails loudly, and the batched jffc sweep API
    rejects them."""
    import torch

    cfg = P.SimConfig(**{**dict(rates=(1.0,), capacities=(1,), workload=P.PoissonWorkload(0.5)), **kw})
    if not torch.cuda.is_available():
        with pytest.raises(P.NativeUnavailable):
            P.run_sim(cfg)
    with pytest.raises(ValueError, match="run_sim_batch"):
        P.run_sim_batch([cfg])


@pytest.mark.parametrize("n", [1, 2, 7, 100, 1001, 90000, 123457])
def test_quantile_from_order_statistics_is_numpy_exact(n):
    rng = np.random.default_rng(n)
    x = np.sort(rng.exponential(3.0, n))
    for q in S.QUANTILES:
        prev, nxt, gamma = S._quantile_ranks(n, q)
        assert S._lerp(float(x[prev]), float(x[nxt]), gamma) == float(np.quantile(x, q))


def test_petals_instance_matches_reference_fixture(golden):
    meta, _ = golden
    svc, servers, _ = P.petals_instance(10, 0.2, 101)
    wan = next(c for c in meta["compose_cases"] if c["name"] == "wan10")
    assert [[s.id, s.memory_bytes, s.comm_time_s, s.per_block_compute_s] for s in servers] == wan["servers"]
    assert [svc.block_count, svc.block_bytes, svc.cache_slot_bytes] == wan["service"]


def test_chainrates():
    cr = P.ChainRates.from_unsorted([1.0, 3.0, 2.0], [1, 2, 3])
    assert cr.rates == (3.0, 2.0, 1.0) and cr.capacities == (2, 3, 1)
    assert cr.total_capacity == 6 and cr.total_rate == 13.0
    with pytest.raises(ValueError):
        P.ChainRates((1.0, 2.0), (1, 1))


def test_batched_aggregation_matches_per_point_numpy():
    """_stats_from_batch reduces each point's row exactly as numpy reduces that
    point's 1-D arrays (sim.py:406-456): compare against direct 1-D numpy on
    random summaries with NaNs, several replication counts and chain counts."""
    from paper_2604_14993_b200 import _native as N

    rng = np.random.default_rng(5)

    def bits_equal(a, b):
        return (math.isnan(a) and math.isnan(b)) or np.float64(a).tobytes() == np.float64(b).tobytes()

    class Order(dict):
        def __missing__(self, k):
            return 1.0 + k * 1e-9

    for R in (1, 2, 7, 129, 1024):
        Pn, K = 3, 2
        summ = np.zeros((Pn, R), N.SUMMARY_DTYPE)
        for f in summ.dtype.names:
            summ[f] = (rng.uniform(0.1, 50, (Pn, R)) if summ.dtype[f].kind == "f"
                       else rng.integers(1, 90000, (Pn, R)))
        summ["mean_occupancy"][rng.random((Pn, R)) < 0.05] = np.nan
        busy = rng.uniform(0, 5, (Pn, R, K))
        cfgs = [P.SimConfig(rates=(0.5, 0.25), capacities=(2, 3), workload=P.PoissonWorkload(0.2),
                            horizon_jobs=1000, warmup_fraction=0.1, seed=1, replications=R)
                for _ in range(Pn)]
        out = S._stats_from_batch(cfgs, summ, busy, [Order() for _ in range(Pn)], None)
        for p in range(Pn):
            occ = np.array(summ["mean_occupancy"][p])
            fin = occ[~np.isnan(occ)]
            assert bits_equal(out[p].mean_occupancy, float(fin.mean()) if fin.size else math.nan)
            rm = np.array(summ["resp_mean"][p])
            ci = (math.nan if R < 2 else float(S._t975(R - 1) * rm.std(ddof=1) / math.sqrt(R)))
            assert bits_equal(out[p].response_ci_half_width_s, ci)
            w = np.array(summ["window_s"][p])
            for k in range(K):
                u = np.where(w > 0, np.array(busy[p, :, k]) / (cfgs[p].capacities[k] * w), math.nan)
                fu = u[~np.isnan(u)]
                assert bits_equal(out[p].per_chain_utilization[k], float(fu.mean()) if fu.size else math.nan)
            ws = 0.0
            for x in summ["wait_sum"][p]:
                ws += x
            assert bits_equal(out[p].mean_waiting_s, float(ws) / int(summ["counted"][p].sum()))
            assert out[p].rep_mean_response_s == tuple(summ["resp_mean"][p].tolist())
