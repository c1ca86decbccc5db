"""Pin the oracle's extended simulator (oracle/cs_oracle.c orc_simulate_ext
plus the numpy input restatements in oracle/oracle.py) against the
reference's own outputs (tests/golden/make_golden_ext.py): every policy,
time-horizon, sampled and trace case, bit-exact.  CPU only."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, bits, ext_inputs, same_float, trace_tables_cpu

FIELDS = ("wait_sum", "service_sum", "counted", "window_s", "mean_occupancy", "occ_first_half",
          "occ_second_half", "lambda_effective", "end_queue_len")


@pytest.fixture(scope="module")
def gx():
    with open(os.path.join(GOLDEN, "golden_ext.json")) as fh:
        meta = json.load(fh)
    return meta, dict(np.load(os.path.join(GOLDEN, "golden_ext.npz")))


@pytest.fixture(scope="module")
def trace_tables(oracle, gx):
    meta, _ = gx
    tables, rates, caps = trace_tables_cpu(oracle, meta["trace_composition"])
    assert rates == meta["trace_composition"]["rates"]
    assert caps == meta["trace_composition"]["caps"]
    return tables


def test_oracle_ext_matches_reference(oracle, gx, trace_tables):
    meta, arrs = gx
    n_cases = 0
    for c in meta["cases"]:
        for rr in c["reps"]:
            arr, warm, sizes, dur = ext_inputs(oracle, c, arrs, rr["rep"], trace_tables)
            o = oracle.simulate_ext(c["rates"], c["caps"], c["policy"], arr, warm, sizes, dur,
                                    collect_jobs="jobs" in rr)
            assert np.array_equal(bits(o["responses"]), bits(arrs[rr["responses"]])), c["tag"]
            assert np.array_equal(bits(o["busy_time_s"]), bits(arrs[rr["busy"]])), c["tag"]
            for f in FIELDS:
                assert same_float(o[f], rr["fields"][f]), (c["tag"], f)
            if "jobs" in rr:
                assert np.array_equal(bits(o["jobs"]), bits(arrs[rr["jobs"]])), c["tag"]
            n_cases += 1
    assert n_cases >= 150


def test_oracle_ext_errors_match_reference(oracle, gx):
    meta, arrs = gx
    for e in meta["errors"]:
        c = {"workload": {"kind": "poisson", "lam": e["lam"]}, "n": e["n"], "wf": e["wf"],
             "horizon": e["horizon"], "seed": 1}
        with pytest.raises(ValueError) as ei:
            ext_inputs(oracle, c, arrs, 0)
        assert str(ei.value) == e["message"]
