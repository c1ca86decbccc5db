"""GPU parity: the CUDA engine (through the C-ABI / drop-in API) vs the
reference's golden outputs and vs the pinned CPU oracle on the same seeded
inputs.  Bit-exact for everything except the merged-mean response time, whose
stated tolerance (north_star) is 1e-6 relative -- we assert 1e-12 -- and, on
the segmented single-chain path, the per-job sums of conftest.SUM_FIELDS and
busy time (reassociated, asserted <= 1e-12 relative).
"""

import math

import numpy as np
import pytest

from conftest import bits, close_rel, same_float, same_rep_field, seg_path, servers_from_rows

pytestmark = pytest.mark.gpu

REP_FIELDS = ("wait_sum", "service_sum", "counted", "window_s", "mean_occupancy",
              "occ_first_half", "occ_second_half", "lambda_effective", "end_queue_len")


@pytest.fixture(scope="module")
def eng():
    import paper_2604_14993_b200 as P
    from paper_2604_14993_b200 import _native as N

    lib = N.load()  # raises NativeUnavailable without a GPU: no silent fallback
    assert lib.cs_device_count() >= 1
    return P


def _exp_streams(keys: np.ndarray, n: int, variant: int):
    import torch
    from paper_2604_14993_b200 import _native as N

    lib = N.load()
    d_keys = torch.from_numpy(np.ascontiguousarray(keys, np.uint64).view(np.int64)).cuda()
    out = torch.empty((len(keys), n), dtype=torch.float64, device="cuda")
    st = lib.cs_exp_streams(d_keys.data_ptr(), len(keys), n, out.data_ptr(), n, variant,
                            torch.cuda.current_stream().cuda_stream)
    N.check(st, "cs_exp_streams")
    return out.cpu().numpy()


def test_exp_streams_match_numpy_golden(eng, golden, oracle):
    meta, arr = golden
    keys = np.array([oracle.philox_key(s, r) for s, r in meta["rng_exp_cases"]])
    got = _exp_streams(keys, arr["rng_exp"].shape[1], variant=1)  # golden host had FMA+AVX2
    assert np.array_equal(bits(got), bits(arr["rng_exp"]))


def test_exp_streams_match_oracle_many_keys(eng, oracle):
    from paper_2604_14993_b200 import _native as N

    variant = N.load().cs_host_log1p_variant()  # the oracle calls this host's libm
    keys = np.array([oracle.philox_key(1, r) for r in range(48)])
    n = 150_000  # ~7e6 draws: ~3.2e3 log1p tail draws, ~1.6e5 wedge tests
    got = _exp_streams(keys, n, variant)
    for i in range(len(keys)):
        ref, _ = oracle.standard_exponential(keys[i], n)
        assert np.array_equal(bits(got[i]), bits(ref)), i


def _sweep(eng, c, collect=True):
    return eng.simulate_sweep([c["rates"]], [c["caps"]], [c["lam"]], c["n"], c["wf"], c["seed"], 1,
                              rep_begin=c["rep"], collect_jobs=collect and c["jobs"],
                              return_responses=True, total_replications=1)


@pytest.mark.parametrize("i", range(9))
def test_simulate_once_matches_reference(eng, golden, i):
    meta, arr = golden
    c = meta["sim_cases"][i]
    res = _sweep(eng, c)
    s = res.summaries[0, 0]
    K = len(c["rates"])
    seg = seg_path(K, c["jobs"])
    for f in REP_FIELDS:
        assert same_rep_field(f, s[f], c["fields"][f], seg), (f, s[f], c["fields"][f])
    assert np.array_equal(bits(res.responses[0, 0]), bits(arr[c["responses"]]))
    if seg:
        assert all(close_rel(x, y) for x, y in zip(res.busy[0, 0, :K], arr[c["busy"]]))
    else:
        assert np.array_equal(bits(res.busy[0, 0, :K]), bits(arr[c["busy"]]))
    if c["rep_mean"] is not None:
        assert same_float(s["resp_mean"], c["rep_mean"])  # numpy pairwise mean, bit-exact
    if c["jobs"]:
        assert np.array_equal(bits(res.jobs[0, 0]), bits(arr[c["job_records"]]))


@pytest.mark.parametrize("i", range(3))
def test_run_sim_matches_reference(eng, golden, i):
    meta, _ = golden
    c = meta["runsim_cases"][i]
    st = eng.run_sim(eng.SimConfig(rates=tuple(c["rates"]), capacities=tuple(c["caps"]),
                                   workload=eng.PoissonWorkload(c["lam"]), horizon_jobs=c["n"],
                                   warmup_fraction=c["wf"], seed=c["seed"],
                                   replications=c["reps"])).to_dict()
    # statistics derived from the per-job sums (SUM_FIELDS, busy) on the
    # segmented single-chain path: 1e-12 relative
    seg = seg_path(len(c["rates"]))
    summed = {"mean_waiting_s", "mean_service_s", "mean_occupancy", "occupancy_ci_half_width",
              "per_chain_utilization", "rep_mean_occupancy", "occ_first_half", "occ_second_half"}
    for k, v in c["stats"].items():
        g = st[k]
        eq = close_rel if seg and k in summed else same_float
        if k == "mean_response_s":
            assert abs(g - v) <= 1e-12 * abs(v), (g, v)
        elif k == "little_law_gap":
            assert abs(g - v) <= 1e-9 * max(abs(v), 1e-12) + (1e-11 if seg else 0.0), (g, v)
        elif isinstance(v, list):
            assert len(g) == len(v) and all(eq(a, b) for a, b in zip(g, v)), (k, g, v)
        elif isinstance(v, float):
            assert eq(g, v), (k, g, v)
        else:
            assert g == v, (k, g, v)


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "segmented"])
def test_sweep_matches_oracle_bit_exact(eng, oracle, exact, monkeypatch):
    """16 arrival rates x 24 reps on the PETALS composition (config-2 shape,
    small n), through the serial bit-exact kernel (CS_SIM_EXACT=1) and the
    default segmented one."""
    monkeypatch.setenv("CS_SIM_EXACT", "1" if exact else "0")
    service, servers, _ = eng.petals_instance(10, 0.2, 101)
    system = eng.greedy_cache_allocation(
        eng.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
    nu = system.total_rate
    lams = [nu * x for x in np.linspace(0.05, 0.95, 16)]
    n, wf, seed, R = 12_000, 0.1, 1, 24
    res = eng.simulate_sweep([system.rates] * 16, [system.capacities] * 16, lams, n, wf, seed, R,
                             return_responses=True)
    for p in (0, 7, 15):
        resp, busy, summ = oracle.simulate_reps(system.rates, system.capacities, lams[p], n, wf,
                                                seed, 0, R, threads=4)
        assert np.array_equal(bits(res.responses[p]), bits(resp)), p
        K = len(system.rates)
        if exact:
            assert np.array_equal(bits(res.busy[p][:, :K]), bits(busy)), p
        else:
            assert all(close_rel(x, y) for x, y in zip(res.busy[p][:, 0], busy[:, 0])), p
        for r in range(R):
            for f in REP_FIELDS:
                assert same_rep_field(f, res.summaries[p, r][f], getattr(summ[r], f), not exact), (p, r, f)
        # exact order statistics of the merged responses
        merged = np.sort(resp.ravel())
        for rank, v in res.order_stats[p].items():
            assert same_float(v, merged[rank]), (p, rank)


def _chain_set(K, C, seed):
    rng = np.random.default_rng(seed)
    rates = tuple(sorted((float(x) for x in rng.uniform(0.2, 2.0, K)), reverse=True))
    caps = [1] * K
    for _ in range(C - K):
        caps[int(rng.integers(K))] += 1
    return rates, tuple(caps)


# (K, C) per kernel path: warp kernel SPL x KPL variants (up to K = 512,
# C = 1024: the J=1000 full-fleet compositions), then the generic
# (workspace heap) kernel beyond
LARGE_CASES = [(3, 20), (12, 40), (40, 100), (70, 200), (20, 400), (2, 600), (300, 700),
               (2, 1100), (600, 1200)]


@pytest.mark.parametrize("K,C", LARGE_CASES)
def test_large_composition_kernels(eng, oracle, K, C):
    """Compositions beyond the register kernel (K > 8 or C > 16): warp-per-
    replication kernel, and the generic kernel for K > 512 or C > 1024."""
    rates, caps = _chain_set(K, C, K * 1000 + C)
    lam = 0.9 * sum(r * c for r, c in zip(rates, caps))
    n, R = 6000, 5
    res = eng.simulate_sweep([rates], [caps], [lam], n, 0.1, 3, R, return_responses=True,
                             collect_jobs=True)
    for r in range(R):
        o = oracle.simulate_once(rates, caps, lam, n, 0.1, 3, r, collect_jobs=True)
        assert np.array_equal(bits(res.responses[0, r]), bits(o["responses"])), r
        assert np.array_equal(bits(res.jobs[0, r]), bits(o["jobs"])), r
        assert np.array_equal(bits(res.busy[0][r, :K]), bits(o["busy_time_s"])), r
        for f in REP_FIELDS:
            assert same_float(res.summaries[0, r][f], o[f]), (r, f)


def test_warp_kernel_mixed_points(eng, oracle):
    """Several compositions of different K/C (and one register-sized one) in
    one launch: the kernel is sized by the largest, smaller points pad."""
    sets = [_chain_set(5, 30, 1), _chain_set(1, 7, 2), _chain_set(34, 87, 3)]
    lams = [0.7 * sum(r * c for r, c in zip(*s)) for s in sets]
    n, R = 4000, 4
    res = eng.simulate_sweep([s[0] for s in sets], [s[1] for s in sets], lams, n, 0.1, 11, R,
                             return_responses=True)
    for p, (rates, caps) in enumerate(sets):
        for r in range(R):
            o = oracle.simulate_once(rates, caps, lams[p], n, 0.1, 11, r)
            assert np.array_equal(bits(res.responses[p, r]), bits(o["responses"])), (p, r)
            assert np.array_equal(bits(res.busy[p][r, :len(rates)]), bits(o["busy_time_s"])), (p, r)


def _compose_inputs(c):
    rows = c["servers"]
    ids = [r[0] for r in rows]
    return ids, [int(r[1]) for r in rows], [float(r[2]) for r in rows], [float(r[3]) for r in rows]


def test_compose_matches_reference(eng, golden):
    meta, _ = golden
    n = 0
    for c in meta["compose_cases"]:
        servers = servers_from_rows(c["servers"], eng)
        service = eng.ServiceSpec(*c["service"])
        if "gbp" in c:
            if "infeasible" in c["gbp"]:
                with pytest.raises(eng.InfeasibleError, match=f"capacity {c['capacity']}"):
                    eng.greedy_block_placement(servers, service, c["capacity"], c["arrival_rate"],
                                               c["load_target"])
                continue
            res = eng.greedy_block_placement(servers, service, c["capacity"], c["arrival_rate"],
                                             c["load_target"])
            ref = c["gbp"]
            assert list(res.placement.first_block) == ref["first"], c["name"]
            assert list(res.placement.block_count) == ref["count"], c["name"]
            assert [list(ch) for ch in res.chains] == ref["chains"], c["name"]
            assert same_float(res.scaled_rate, ref["scaled_rate"])
            assert res.rate_satisfied == ref["rate_satisfied"]
            assert list(res.profile.max_blocks) == ref["max_blocks"]
            assert np.array_equal(bits(res.profile.bound_time_s), bits(ref["bound_time"]))
            placement = res.placement
        else:
            placement = eng.BlockPlacement(service, servers, tuple(c["first"]), tuple(c["count"]))
        system = eng.greedy_cache_allocation(placement, c.get("residual"))
        ref = c["gca"]
        assert [list(ch.server_ids) for ch in system.chains] == ref["chains"], c["name"]
        assert list(system.capacities) == ref["caps"], c["name"]
        assert np.array_equal(bits([ch.service_time_s for ch in system.chains]),
                              bits(ref["times"])), c["name"]
        n += 1
    assert n > 400


def test_compose_batch_random_fleets_match_oracle(eng, oracle):
    """J=100, L=80 fleets through GBP+GCA in ONE batched launch each, vs the oracle."""
    fleets = [eng.fleet(100, 80, seed=s) for s in range(6)]
    svc = fleets[0][0]
    pts = [(f[1], c, lam) for f in fleets for c, lam in ((7, 5.0), (3, 1e9), (20, 2.0))]
    res = eng.greedy_block_placement_batch([p[0] for p in pts], [svc] * len(pts),
                                           [p[1] for p in pts], [p[2] for p in pts],
                                           [0.7] * len(pts))
    systems = eng.greedy_cache_allocation_batch([r.placement for r in res])
    for (servers, c, lam), r, sysm in zip(pts, res, systems):
        ids = [s.id for s in servers]
        mem = [s.memory_bytes for s in servers]
        tc = [s.comm_time_s for s in servers]
        tp = [s.per_block_compute_s for s in servers]
        st, g = oracle.gbp(mem, tc, tp, ids, 80, svc.block_bytes, svc.cache_slot_bytes, c, lam, 0.7)
        assert list(r.placement.first_block) == list(g["first"])
        assert list(r.placement.block_count) == list(g["count"])
        st, a = oracle.gca(mem, tc, tp, ids, 80, svc.block_bytes, svc.cache_slot_bytes,
                           g["first"], g["count"])
        assert [list(ch.server_ids) for ch in sysm.chains] == [[ids[j] for j in ch] for ch in a["chains"]]
        assert list(sysm.capacities) == list(a["caps"])
        assert np.array_equal(bits([ch.service_time_s for ch in sysm.chains]), bits(a["times"]))


def _surrogate_cases():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "golden_surrogate.json")) as fh:
        return json.load(fh)["cases"]


@pytest.mark.parametrize("case", _surrogate_cases(), ids=lambda c: c["name"])
def test_tune_capacity_surrogate_matches_reference(eng, case):
    """c in [1, c_max] evaluated in one GBP launch: c_star and every
    TuningRow (placement.py:161-200) bit-exact vs the reference, or the same
    InfeasibleError message and best_rate."""
    servers = tuple(eng.ServerSpec(r[0], int(r[1]), float.fromhex(r[2]), float.fromhex(r[3]))
                    for r in case["servers"])
    service = eng.ServiceSpec(*case["service"])
    lam, rho = float.fromhex(case["lam"]), float.fromhex(case["rho"])
    if "infeasible" in case:
        with pytest.raises(eng.InfeasibleError) as exc:
            eng.tune_capacity_surrogate(servers, service, lam, rho)
        assert str(exc.value) == case["infeasible"]
        assert same_float(exc.value.best_rate, float.fromhex(case["best_rate"]))
        return
    t = eng.tune_capacity_surrogate(servers, service, lam, rho)
    assert t.c_star == case["c_star"]
    assert len(t.rows) == len(case["rows"])
    for row, ref in zip(t.rows, case["rows"]):
        assert [row.capacity, row.chain_count, row.scaled_cost, row.rate_satisfied] == ref[:4], ref
        assert same_float(row.achieved_rate, float.fromhex(ref[4])), ref


def test_no_silent_fallback_loaded_native(eng):
    import paper_2604_14993_b200._native as N

    assert N._lib is not None and N.LIB_PATH.endswith("libchainserve_b200.so")


def test_sample_select_and_pairwise_means(eng, oracle):
    """Groups above 2^20 responses take the sample-select path; per-rep means
    are the statistics pass's numpy pairwise sums (bit-exact)."""
    service, servers, _ = eng.petals_instance(10, 0.2, 101)
    system = eng.greedy_cache_allocation(
        eng.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
    nu = system.total_rate
    lams = [0.3 * nu, 0.93 * nu]
    n, wf, seed, R = 10_000, 0.1, 3, 128
    res = eng.simulate_sweep([system.rates] * 2, [system.capacities] * 2, lams, n, wf, seed, R)
    for p in range(2):
        resp, busy, summ = oracle.simulate_reps(system.rates, system.capacities, lams[p], n, wf,
                                                seed, 0, R, threads=8)
        assert resp.size > (1 << 20)
        merged = np.sort(resp.ravel())
        for rank, v in res.order_stats[p].items():
            assert same_float(v, merged[rank]), (p, rank, v, merged[rank])
        means = np.array([row.mean() for row in resp])
        assert np.array_equal(bits(res.summaries[p]["resp_mean"]), bits(means))


def test_sweep_engine_pipelined_equals_unpipelined(eng):
    """SweepEngine.run_pipelined (two buffer sets, two CUDA streams; the
    benchmark's timed loop) computes every sweep exactly like step()."""
    import torch

    from paper_2604_14993_b200.engine import SweepEngine

    service, servers, _ = eng.petals_instance(10, 0.2, 101)
    system = eng.greedy_cache_allocation(
        eng.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)
    lams = [system.total_rate * x for x in (0.3, 0.9)]
    e = SweepEngine([system.rates] * 2, [system.capacities] * 2, lams, 20_000, 0.1, 1, 64)
    e.step()
    torch.cuda.synchronize()
    ref_s, ref_b, ref_o = e.summaries(0).copy(), e.busy(0).copy(), e.order_stats()
    last = e.run_pipelined(3)
    torch.cuda.synchronize()
    for b in (0, 1):  # both buffer sets hold a complete, identical sweep
        assert np.array_equal(e.summaries(b).view(np.uint8), ref_s.view(np.uint8)), b
        assert np.array_equal(bits(e.busy(b)), bits(ref_b)), b
    assert e.order_stats() == ref_o and last == 0


def test_long_rows_statistics(eng, oracle):
    """Rows of 225k responses (the split-tree leaf values spill from shared
    memory to a global scratch, as for config 5's 9e5-response rows): exact
    pairwise rep means and order statistics vs the oracle."""
    rates, caps = (0.9,), (3,)
    lam = 0.8 * 0.9 * 3
    n, R = 250_000, 3
    res = eng.simulate_sweep([rates], [caps], [lam], n, 0.1, 5, R, return_responses=True)
    allr = []
    for r in range(R):
        o = oracle.simulate_once(rates, caps, lam, n, 0.1, 5, r)
        assert np.array_equal(bits(res.responses[0, r]), bits(o["responses"])), r
        assert same_float(res.summaries[0, r]["resp_mean"], o["responses"].mean()), r
        allr.append(o["responses"])
    merged = np.sort(np.concatenate(allr))
    for rank, v in res.order_stats[0].items():
        assert same_float(v, merged[rank]), rank


@pytest.mark.parametrize("C", [1, 3, 4, 7, 8, 12, 16])
def test_single_chain_kernel_stress(eng, oracle, C):
    """The single-chain recursion + merge kernel (jffc_sim_k1_kernel) across
    capacities and loads from light to overloaded (long FCFS queues, lagging
    merges), plus heavy warm-up: every RepResult field, responses, busy time
    and job records bit-exact vs the oracle."""
    rate = 0.7 + 0.05 * C
    lams = [rho * rate * C for rho in (0.2, 0.95, 1.3)]
    n, R = 20_000, 4
    for wf in (0.0, 0.5):
        res = eng.simulate_sweep([(rate,)] * 3, [(C,)] * 3, lams, n, wf, 23, R, return_responses=True,
                                 collect_jobs=True)
        for p, lam in enumerate(lams):
            for r in range(R):
                o = oracle.simulate_once((rate,), (C,), lam, n, wf, 23, r, collect_jobs=True)
                assert np.array_equal(bits(res.responses[p, r]), bits(o["responses"])), (p, r)
                assert np.array_equal(bits(res.jobs[p, r]), bits(o["jobs"])), (p, r)
                assert same_float(res.busy[p][r, 0], o["busy_time_s"][0]), (p, r)
                for f in REP_FIELDS:
                    assert same_float(res.summaries[p, r][f], o[f]), (p, r, f)


def test_event_loop_fallback_equals_recursion(eng, oracle, monkeypatch):
    """CS_SIM_FORCE_EVENT_LOOP (the per-event register kernel the host path
    falls back to when the serial recursion kernel reports a backed-up merge)
    gives the same bits as the recursion kernel and the oracle."""
    import ctypes as C

    import torch

    from paper_2604_14993_b200 import _native as N

    monkeypatch.setenv("CS_SIM_EXACT", "1")
    lib = N.load()
    rates, caps = (0.8,), (5,)
    lams = [0.5 * 4.0, 0.97 * 4.0]
    n, warm, R, P = 8000, 800, 6, 2
    keys = np.concatenate([oracle.philox_key(3, r) for r in range(R)]).astype(np.uint64)
    d_keys = torch.from_numpy(keys.view(np.int64)).cuda()
    pts = (N.SimPoint * P)(*[N.SimPoint(1, 0, l) for l in lams])
    d_pts = torch.frombuffer(bytearray(bytes(pts)), dtype=torch.uint8).cuda()
    d_rates = torch.tensor(rates, dtype=torch.float64, device="cuda")
    d_caps = torch.tensor(caps, dtype=torch.int32, device="cuda")
    lds, ldr = 2 * n, (n - warm + 15) & ~15
    S = torch.empty(R * lds + 512, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    N.check(lib.cs_exp_streams(d_keys.data_ptr(), R, lds, S.data_ptr(), lds, -1, st), "streams")
    outs = []
    for flags in (0, N.CS_SIM_FORCE_EVENT_LOOP):
        resp = torch.zeros(P * R * ldr, dtype=torch.float64, device="cuda")
        busy = torch.zeros(P * R, dtype=torch.float64, device="cuda")
        summ = torch.zeros(P * R * C.sizeof(N.RepSummary), dtype=torch.uint8, device="cuda")
        N.check(lib.cs_jffc_sim_ex(d_pts.data_ptr(), P, d_rates.data_ptr(), d_caps.data_ptr(), 1, 5,
                                   S.data_ptr(), lds, 0, R, R, n, warm, resp.data_ptr(), ldr,
                                   busy.data_ptr(), 1, summ.data_ptr(), None, None, 0, flags, st), "sim")
        outs.append((resp.cpu().numpy().reshape(P, R, ldr)[:, :, :n - warm], busy.cpu().numpy(),
                     summ.cpu().numpy().view(N.SUMMARY_DTYPE).reshape(P, R)))
    assert np.array_equal(bits(outs[0][0]), bits(outs[1][0]))
    assert np.array_equal(bits(outs[0][1]), bits(outs[1][1]))
    for f in REP_FIELDS:
        assert np.array_equal(bits(outs[0][2][f].astype(np.float64)), bits(outs[1][2][f].astype(np.float64))), f
    for p in range(P):
        resp, _, _ = oracle.simulate_reps(rates, caps, lams[p], n, 0.1, 3, 0, R)
        assert np.array_equal(bits(outs[1][0][p]), bits(resp)), p
