"""Occupancy bounds and the capacity-bound sweep (SURVEY.md §8(f) row 1,
chainserve analysis.py:67-147,270-336) against golden outputs of the
reference (tests/golden/make_golden_bounds.py).

Tolerances: death rates, chain counts, capacities and total rates are
bit-exact; occupancy / response bounds go through log/exp/log1p and a
reduction order different from numpy's, so they are checked to 1e-9 relative
(north_star: <= 1e-6).  The numpy oracle restatement is checked to 1e-13.
"""

import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN

RTOL_GPU = 1e-9
RTOL_ORACLE = 1e-13


def fx(h):
    return None if h is None else float.fromhex(h)


@pytest.fixture(scope="module")
def gb():
    with open(os.path.join(GOLDEN, "golden_bounds.json")) as fh:
        return json.load(fh)


def close(a, b, rtol):
    return abs(a - b) <= rtol * abs(b)


# ---------------------------------------------------------------- CPU


def test_death_rate_bounds_bit_exact(gb):
    import paper_2604_14993_b200 as P

    for case in gb["death"]:
        cr = P.ChainRates(tuple(fx(r) for r in case["rates"]), tuple(case["caps"]))
        for n, (u, lo) in enumerate(case["rows"]):
            assert P.death_rate_bounds(cr, n) == (fx(u), fx(lo)), n
    with pytest.raises(ValueError, match="n must be >= 0"):
        P.death_rate_bounds(cr, -1)


def test_oracle_bounds_match_reference(gb, oracle):
    n = 0
    for case in gb["bounds"]:
        rates = [fx(r) for r in case["rates"]]
        out = oracle.occupancy_bounds(rates, case["caps"], fx(case["lam"]))
        if "unstable" in case:
            assert out is None
            continue
        for got, want in zip(out, case["out"]):
            assert close(got, fx(want), RTOL_ORACLE), (case["caps"], got, fx(want))
        n += 1
    assert n > 50
    for case in gb["bd"]:
        got = oracle.birth_death_mean_occupancy(fx(case["lam"]), [fx(x) for x in case["death"]],
                                                fx(case["nu"]))
        assert close(got, fx(case["out"]), RTOL_ORACLE)


def test_oracle_death_rates_match_reference(gb, oracle):
    for case in gb["death"]:
        fast, slow = oracle.death_rates([fx(r) for r in case["rates"]], case["caps"])
        for n in range(1, len(fast) + 1):
            assert (fast[n - 1], slow[n - 1]) == (fx(case["rows"][n][0]), fx(case["rows"][n][1]))


def test_bounds_validation_without_device():
    import paper_2604_14993_b200 as P

    cr = P.ChainRates((1.0,), (2,))
    with pytest.raises(ValueError, match="arrival_rate must be positive"):
        P.occupancy_bounds(cr, 0.0)
    with pytest.raises(P.UnstableError, match="arrival rate 2 >= total service rate 2"):
        P.occupancy_bounds(cr, 2.0)
    with pytest.raises(ValueError, match="death rates must be positive"):
        P.birth_death_mean_occupancy(0.5, [1.0, 0.0], 2.0)
    with pytest.raises(ValueError, match="which must be"):
        P.tune_capacity_bound([], None, 1.0, 0.5, which="middle")


# ---------------------------------------------------------------- GPU


@pytest.mark.gpu
def test_occupancy_bounds_match_reference(gb):
    import paper_2604_14993_b200 as P

    systems, lams, cases = [], [], []
    for case in gb["bounds"]:
        cr = P.ChainRates(tuple(fx(r) for r in case["rates"]), tuple(case["caps"]))
        lam = fx(case["lam"])
        if "unstable" in case:
            with pytest.raises(P.UnstableError) as ei:
                P.occupancy_bounds(cr, lam)
            assert str(ei.value) == case["unstable"]
            continue
        b = P.occupancy_bounds(cr, lam)  # single-system drop-in call
        got = (b.lower_mean_occupancy, b.upper_mean_occupancy, b.lower_mean_response_s,
               b.upper_mean_response_s)
        for g, w in zip(got, case["out"]):
            assert close(g, fx(w), RTOL_GPU), (case["caps"], g, fx(w))
        systems.append(cr)
        lams.append(lam)
        cases.append(case)
    # all systems in one batched launch give the same numbers
    out = P.occupancy_bounds_batch(systems, lams)
    for r, case in zip(out, cases):
        assert int(r["status"]) == 0
        assert close(float(r["lower_occupancy"]), fx(case["out"][0]), RTOL_GPU)
        assert close(float(r["upper_response_s"]), fx(case["out"][3]), RTOL_GPU)


@pytest.mark.gpu
def test_birth_death_matches_reference(gb):
    import paper_2604_14993_b200 as P

    for case in gb["bd"]:
        got = P.birth_death_mean_occupancy(fx(case["lam"]), [fx(x) for x in case["death"]],
                                           fx(case["nu"]))
        assert close(got, fx(case["out"]), RTOL_GPU)


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(4))
def test_bound_curve_matches_reference(gb, idx):
    import paper_2604_14993_b200 as P

    case = gb["curves"][idx]
    servers = tuple(P.ServerSpec(r[0], int(r[1]), fx(r[2]), fx(r[3])) for r in case["servers"])
    service = P.ServiceSpec(*case["service"])
    lam, rho = fx(case["lam"]), case["rho"]
    rows = P.bound_curve(servers, service, lam, rho)
    assert len(rows) == len(case["rows"]), case["name"]
    for r, w in zip(rows, case["rows"]):
        assert (r.capacity, r.chain_count, r.total_capacity, r.stable) == (w[0], w[1], w[2], w[6])
        assert r.total_rate == fx(w[3])
        if w[6]:
            assert close(r.lower_response_s, fx(w[4]), RTOL_GPU), (case["name"], r.capacity)
            assert close(r.upper_response_s, fx(w[5]), RTOL_GPU), (case["name"], r.capacity)
        else:
            assert r.lower_response_s is None and r.upper_response_s is None
    for which in ("lower", "upper"):
        want = case[f"c_star_{which}"]
        if isinstance(want, str):
            with pytest.raises(P.UnstableError) as ei:
                P.tune_capacity_bound(servers, service, lam, rho, which)
            assert str(ei.value) == want
        else:
            assert P.tune_capacity_bound(servers, service, lam, rho, which).c_star == want
