"""Shared test setup.

* ``-m gpu`` tests need a B200 (the CUDA engine); everything else runs on CPU.
* The CPU oracle (oracle/, test infrastructure) is built on first use.
* Golden fixtures come from tests/golden/make_golden.py (the reference run in
  the build container); /root/reference is never read here.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")
    config.addinivalue_line("markers", "slow: longer-running test")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN, "golden.npz")))
    return meta, arrays


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def same_float(a: float, b: float) -> bool:
    """Bit-identical doubles (NaN == NaN)."""
    return np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64) or (
        np.isnan(a) and np.isnan(b))


# RepResult fields the single-chain SEGMENTED simulator (csrc/jffc_seg.cu)
# accumulates per job in fixed job blocks instead of per event: the same
# quantities as the reference's sequential sums, reassociated.  Stated
# tolerance 1e-12 relative (north_star allows 1e-6 for derived statistics);
# everything else (responses, their order, counted, window, lambda_eff,
# end_queue, order statistics, rep means) stays bit-exact.
SUM_FIELDS = ("wait_sum", "service_sum", "mean_occupancy", "occ_first_half", "occ_second_half")
SUM_RTOL = 1e-12


def close_rel(a: float, b: float, rtol: float = SUM_RTOL) -> bool:
    """|a - b| <= rtol * max(|a|, |b|) (NaN == NaN)."""
    if np.isnan(a) or np.isnan(b):
        return bool(np.isnan(a) and np.isnan(b))
    return abs(a - b) <= rtol * max(abs(a), abs(b))


def seg_path(K: int, collect_jobs: bool = False) -> bool:
    """True when cs_jffc_sim takes the segmented single-chain kernel."""
    return K == 1 and not collect_jobs and os.environ.get("CS_SIM_EXACT", "0") != "1"


def same_rep_field(f: str, got: float, ref: float, seg: bool) -> bool:
    if seg and f in SUM_FIELDS:
        return close_rel(got, ref)
    return same_float(got, ref)


def servers_from_rows(rows, mod):
    return tuple(mod.ServerSpec(r[0], int(r[1]), float(r[2]), float(r[3])) for r in rows)


def ext_inputs(oracle, c, arrs, rep, trace_tables=None):
    """Oracle-side inputs of a golden_ext case (tests/golden/make_golden_ext.py):
    (arrivals, warm, sizes, durations) restating _materialize (sim.py:136-178)
    and the warm-up rule (sim.py:184-190).  Raises ValueError as the reference."""
    import math

    wd, n, wf, hz = c["workload"], c["n"], c["wf"], c["horizon"]
    sizes = durations = None
    if wd["kind"] == "poisson":
        arr, sizes = oracle.poisson_inputs(wd["lam"], n, c["seed"], rep, hz)
        if arr.size == 0:
            raise ValueError("no arrivals fall inside the time horizon")
    elif wd["kind"] == "sampled":
        arr, sizes = arrs["sampled_arrivals"], arrs["sampled_sizes"]
        if hz is not None:
            keep = arr <= hz
            arr, sizes = arr[keep], sizes[keep]
        arr, sizes = arr[:n], sizes[:n]
    else:
        arr = arrs["trace_arrivals"]
        tin, tout = arrs["trace_tin"], arrs["trace_tout"]
        if hz is not None:
            keep = arr <= hz
            arr, tin, tout = arr[keep], tin[keep], tout[keep]
        arr, tin, tout = arr[:n], tin[:n], tout[:n]
        hops, params = trace_tables
        durations = oracle.trace_durations(tin, tout, hops, params)
    if hz is None:
        warm = int(wf * arr.size)
    else:
        warm = int(np.searchsorted(arr, wf * hz, side="left"))
        if warm >= arr.size:
            raise ValueError("warmup consumed every arrival in the time horizon")
    return arr, warm, sizes, durations


def trace_tables_cpu(oracle, comp):
    """Chains of the golden trace cases composed by the ORACLE (GBP + GCA on
    the PETALS fixture), as (hops per chain, per-server timing constants)
    restating workload.py:39-60,108-120 -- no GPU involved."""
    import paper_2604_14993_b200 as P

    service, servers, model = P.petals_instance(10, 0.2, 101)
    ids = [s.id for s in servers]
    mem = [s.memory_bytes for s in servers]
    tc = [s.comm_time_s for s in servers]
    tp = [s.per_block_compute_s for s in servers]
    st, g = oracle.gbp(mem, tc, tp, ids, service.block_count, service.block_bytes,
                       service.cache_slot_bytes, comp["capacity"], comp["arrival_rate"],
                       comp["load_target"])
    assert st == 0
    st, a = oracle.gca(mem, tc, tp, ids, service.block_count, service.block_bytes,
                       service.cache_slot_bytes, g["first"], g["count"])
    assert st == 0
    placement = P.BlockPlacement(service, tuple(servers), tuple(int(x) for x in g["first"]),
                                 tuple(int(x) for x in g["count"]))
    params, hops = [], []
    for k, members in enumerate(a["chains"]):
        chain = P.build_chain(placement, [ids[i] for i in members])
        h = []
        for e in chain.edges:
            if e.dst == P.TAIL_ID:
                continue
            prof = model.profiles[e.dst]
            h.append((len(params), e.blocks_at_dst))
            params.append((model.rtt.rtt_ms(model.orchestrator, e.dst) + model.rtt.overhead_ms,
                           prof.per_block_overhead_ms,
                           prof.per_block_flops_gflop / prof.flops_tflops,
                           (service.block_bytes / P.GB) / prof.mem_bandwidth_gb_per_ms))
        hops.append(h)
    rates = [1.0 / t for t in a["times"]]
    return (hops, params), rates, [int(x) for x in a["caps"]]
