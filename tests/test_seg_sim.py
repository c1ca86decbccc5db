"""GPU parity of the segmented (time-parallel) single-chain simulator
(csrc/jffc_seg.cu) against the pinned CPU oracle: responses in completion
order, counted, window, lambda_eff, end_queue, order statistics and rep means
bit-exact; the per-job sums (conftest.SUM_FIELDS, busy time) within 1e-12
relative.  Results must not depend on the number of segments (CS_SEG_S).
"""

import numpy as np
import pytest

from conftest import SUM_FIELDS, bits, close_rel, same_float

pytestmark = pytest.mark.gpu

EXACT_FIELDS = ("counted", "window_s", "lambda_effective", "end_queue_len")


@pytest.fixture(scope="module")
def eng():
    import paper_2604_14993_b200 as P
    from paper_2604_14993_b200 import _native as N

    assert N.load().cs_device_count() >= 1
    return P


def _check_rows(res, p, oracle, rates, caps, lam, n, wf, seed, R, rep0=0):
    resp, busy, summ = oracle.simulate_reps(rates, caps, lam, n, wf, seed, rep0, rep0 + R, threads=8)
    assert np.array_equal(bits(res.responses[p]), bits(resp)), p
    for r in range(R):
        s = res.summaries[p, r]
        for f in EXACT_FIELDS:
            assert same_float(s[f], getattr(summ[r], f)), (p, r, f, s[f], getattr(summ[r], f))
        for f in SUM_FIELDS:
            assert close_rel(s[f], getattr(summ[r], f)), (p, r, f, s[f], getattr(summ[r], f))
        assert close_rel(res.busy[p][r, 0], busy[r, 0]), (p, r)
        assert same_float(s["resp_mean"], resp[r].mean()), (p, r)
    merged = np.sort(resp.ravel())
    for rank, v in res.order_stats[p].items():
        assert same_float(v, merged[rank]), (p, rank)


def _petals(eng):
    service, servers, _ = eng.petals_instance(10, 0.2, 101)
    return eng.greedy_cache_allocation(
        eng.greedy_block_placement(servers, service, 7, 0.2, 0.7).placement)


def test_config2_shape_vs_oracle(eng, oracle):
    """16 arrival rates nu*linspace(0.05, 0.95) x 32 reps on the PETALS
    composition (K=1, C=7), n = 30k: several segments per row."""
    from paper_2604_14993_b200 import _native as N

    system = _petals(eng)
    nu = system.total_rate
    lams = [nu * x for x in np.linspace(0.05, 0.95, 16)]
    n, wf, seed, R = 30_000, 0.1, 1, 32
    assert N.seg_plan(16, R, 7, n)["segments"] > 1
    res = eng.simulate_sweep([system.rates] * 16, [system.capacities] * 16, lams, n, wf, seed, R,
                             return_responses=True)
    for p in range(16):
        _check_rows(res, p, oracle, system.rates, system.capacities, lams[p], n, wf, seed, R)


@pytest.mark.parametrize("C", [1, 3, 4, 7, 8, 12, 16])
def test_capacities_and_loads(eng, oracle, C):
    """Capacities 1..16 (every CMAX instance), loads from light to overloaded
    (rho 1.3: no coupling, the exact segment runs through every later one),
    no and heavy warm-up."""
    rate = 0.7 + 0.05 * C
    lams = [rho * rate * C for rho in (0.2, 0.8, 0.97, 1.3)]
    n, R = 24_000, 4
    for wf in (0.0, 0.5):
        res = eng.simulate_sweep([(rate,)] * 4, [(C,)] * 4, lams, n, wf, 23, R, return_responses=True)
        for p, lam in enumerate(lams):
            _check_rows(res, p, oracle, (rate,), (C,), lam, n, wf, 23, R)


def test_independent_of_segment_count(eng, monkeypatch):
    """The same sweep with 1, 2, 3 and the default number of segments: every
    output bit-identical (block sums fix the association of the per-job sums)."""
    system = _petals(eng)
    nu = system.total_rate
    lams = [nu * x for x in (0.3, 0.7, 0.95, 1.1)]
    n, R = 40_000, 16
    from paper_2604_14993_b200 import _native as N

    outs = []
    for S in ("1", "2", "3", "64"):
        monkeypatch.setenv("CS_SEG_S", S)
        plan = N.seg_plan(4, R, 7, n)
        assert plan["segments"] == min(int(S), 19), plan  # n / (8 blocks of 256 jobs) = 19
        res = eng.simulate_sweep([system.rates] * 4, [system.capacities] * 4, lams, n, 0.1, 9, R,
                                 return_responses=True)
        outs.append(res)
    for res in outs[1:]:
        assert np.array_equal(bits(res.responses), bits(outs[0].responses))
        assert np.array_equal(res.summaries.view(np.uint8), outs[0].summaries.view(np.uint8))
        assert np.array_equal(bits(res.busy), bits(outs[0].busy))
        assert res.order_stats == outs[0].order_stats


def test_rep_offset_and_odd_sizes(eng, oracle):
    """Replications not starting at 0, a row count not a multiple of 32 and
    n not a multiple of the job block."""
    rates, caps = (0.61,), (5,)
    lam = 0.85 * 0.61 * 5
    n, R = 17_777, 37
    res = eng.simulate_sweep([rates], [caps], [lam], n, 0.13, 4, R, rep_begin=100,
                             return_responses=True, total_replications=R)
    _check_rows(res, 0, oracle, rates, caps, lam, n, 0.13, 4, R, rep0=100)


def test_long_rows_vs_oracle(eng, oracle):
    """n = 1e6 (config 5's row length) on the PETALS composition at rho 0.7:
    many segments per row, 9e5 responses per row."""
    system = _petals(eng)
    lam = 0.7 * system.total_rate
    n, R = 1_000_000, 4
    res = eng.simulate_sweep([system.rates], [system.capacities], [lam], n, 0.1, 1, R,
                             return_responses=True)
    _check_rows(res, 0, oracle, system.rates, system.capacities, lam, n, 0.1, 1, R)


def test_many_points_standalone_prefix(eng, oracle):
    """40 points share each stream (> 32: the stream kernel does not fuse the
    arrival-time prefix, the simulator's own pre-pass computes it)."""
    rates, caps = (0.8,), (4,)
    lams = [x * 0.8 * 4 for x in np.linspace(0.1, 0.98, 40)]
    n, R = 9_000, 3
    res = eng.simulate_sweep([rates] * 40, [caps] * 40, lams, n, 0.1, 5, R, return_responses=True)
    for p in (0, 21, 39):
        _check_rows(res, p, oracle, rates, caps, lams[p], n, 0.1, 5, R)


def test_engine_fused_prefix_equals_host_path(eng):
    """SweepEngine (streams stage writes the simulator's prefix into its
    buffer set's workspace) equals the host-buffer path bit for bit."""
    import torch

    from paper_2604_14993_b200.engine import SweepEngine

    system = _petals(eng)
    lams = [system.total_rate * x for x in (0.2, 0.6, 0.9)]
    n, R = 30_000, 40
    e = SweepEngine([system.rates] * 3, [system.capacities] * 3, lams, n, 0.1, 2, R)
    e.step()
    torch.cuda.synchronize()
    assert e.sets[0]["flags"].value & 1  # CS_SIM_PREFIX_READY
    res = eng.simulate_sweep([system.rates] * 3, [system.capacities] * 3, lams, n, 0.1, 2, R)
    got = e.summaries(0)
    for f in ("wait_sum", "service_sum", "mean_occupancy", "end_queue_len", "window_s", "resp_mean"):
        assert np.array_equal(np.asarray(got[f]).view(np.uint64), np.asarray(res.summaries[f]).view(np.uint64)), f
    assert e.order_stats() == res.order_stats


@pytest.mark.parametrize("R", [64, 40], ids=["interleaved", "row_major"])
def test_stream_layouts_vs_oracle(eng, oracle, R):
    """Few points per stream: the streams are written in the simulator's
    32-row interleaved layout when the replication count is a multiple of 32
    (CS_SIM_STREAMS_IL4), row-major otherwise; both exact against the oracle."""
    import torch

    from paper_2604_14993_b200 import _native as N
    from paper_2604_14993_b200.engine import SweepEngine

    system = _petals(eng)
    lams = [system.total_rate * x for x in (0.5, 0.93)]
    n = 20_000
    e = SweepEngine([system.rates] * 2, [system.capacities] * 2, lams, n, 0.1, 4, R)
    e.step()
    torch.cuda.synchronize()
    il4 = bool(e.sets[0]["flags"].value & N.CS_SIM_STREAMS_IL4)
    assert il4 == (R % 32 == 0)
    res = eng.simulate_sweep([system.rates] * 2, [system.capacities] * 2, lams, n, 0.1, 4, R,
                             return_responses=True)
    for p in range(2):
        _check_rows(res, p, oracle, system.rates, system.capacities, lams[p], n, 0.1, 4, R)
    got = e.summaries(0)
    for f in ("wait_sum", "mean_occupancy", "end_queue_len", "resp_mean"):
        assert np.array_equal(np.asarray(got[f]).view(np.uint64), np.asarray(res.summaries[f]).view(np.uint64)), f


def test_instrumentation_switches_keep_results(eng, monkeypatch, capfd):
    """The development switches (CS_SEG_TRACE: the simulator's per-segment
    timeline; CS_TRACE_STATS: the statistics' phase times; CS_DEBUG_STATS)
    only print to stderr: every output is unchanged."""
    system = _petals(eng)
    lams = [system.total_rate * x for x in (0.3, 0.9)]
    args = ([system.rates] * 2, [system.capacities] * 2, lams, 30_000, 0.1, 9, 64)
    ref = eng.simulate_sweep(*args)
    for var in ("CS_SEG_TRACE", "CS_TRACE_STATS", "CS_DEBUG_STATS"):
        monkeypatch.setenv(var, "1")
    got = eng.simulate_sweep(*args)
    err = capfd.readouterr().err
    assert "jffc_seg_kernel" in err and "[stats]" in err
    assert np.array_equal(got.summaries.view(np.uint8), ref.summaries.view(np.uint8))
    assert np.array_equal(bits(got.busy), bits(ref.busy))
    assert got.order_stats == ref.order_stats


def test_random_shapes_vs_oracle(eng, oracle):
    """Seeded random shapes (points, replications, jobs, capacity, rate, load,
    warm-up) through the segmented path, every field against the oracle --
    the hand-over between segments under every mix of coupling lengths."""
    rng = np.random.default_rng(20260419)
    for _ in range(40):
        P = int(rng.integers(1, 20))
        R = int(rng.choice([1, 3, 31, 32, 33, 64]))
        n = int(rng.integers(3_000, 60_000))
        C = int(rng.integers(1, 17))
        rate = float(rng.uniform(0.3, 2.0))
        wf = float(rng.choice([0.0, 0.1, 0.37]))
        seed = int(rng.integers(0, 2**31))
        lams = [float(rng.uniform(0.05, 1.15)) * rate * C for _ in range(P)]
        res = eng.simulate_sweep([(rate,)] * P, [(C,)] * P, lams, n, wf, seed, R, return_responses=True)
        for p in {0, P - 1, P // 2}:
            _check_rows(res, p, oracle, (rate,), (C,), lams[p], n, wf, seed, R)
