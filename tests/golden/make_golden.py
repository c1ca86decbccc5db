"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports chainserve from /root/reference/pkg/src (and its test fixtures
from pkg/tests/conftest.py) and numpy 2.3.5, and writes
tests/golden/golden.npz + tests/golden/golden.json.  The GPU box never reads
/root/reference: tests compare the oracle and the CUDA engine against these
committed files.  Contents:

* rng: SeedSequence->Philox keys, Philox random_raw words and
  Generator.exponential streams (sim.py:141-145,159 semantics).
* sim: _simulate_once RepResult fields, responses, busy times and job
  records (sim.py:181-324) for small configurations.
* runsim: run_sim(...).to_dict() for small multi-replication configurations.
* compose: greedy_block_placement + greedy_cache_allocation outputs for the
  reference's named fixtures and seeded random / tie-heavy instances.
"""

from __future__ import annotations

import json
import os
import platform
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import chainserve as cs  # noqa: E402
from chainserve.sim import _simulate_once  # noqa: E402
from conftest import (  # noqa: E402
    philox,
    random_placement,
    random_servers,
    random_service,
    tiered_instance,
    uniform_tradeoff_instance,
    wan_gpu_fixture,
)

HERE = os.path.dirname(os.path.abspath(__file__))
arrays: dict[str, np.ndarray] = {}
meta: dict = {
    "generator": "tests/golden/make_golden.py",
    "numpy": np.__version__,
    "python": platform.python_version(),
    "glibc": " ".join(platform.libc_ver()),
    "machine": platform.machine(),
}


def put(name, a):
    arrays[name] = np.asarray(a)
    return name


# ---------------------------------------------------------------- rng
KEY_CASES = [(1, 0), (1, 1), (1, 1023), (0, 0), (5, 3), (29, 0), (2**40 + 3, 77),
             (123456789, 2**33 + 1), (7, 4095)]
keys = []
for seed, rep in KEY_CASES:
    keys.append(np.random.SeedSequence(entropy=seed, spawn_key=(rep,)).generate_state(2, np.uint64))
meta["rng_key_cases"] = [[int(s), int(r)] for s, r in KEY_CASES]
put("rng_keys", np.array(keys))
raw = [np.random.Philox(np.random.SeedSequence(entropy=s, spawn_key=(r,))).random_raw(256)
       for s, r in KEY_CASES[:4]]
put("rng_raw", np.array(raw))
EXP_CASES = [(1, 0), (1, 1), (5, 3), (29, 0)]
EXP_N = 60000
exp = []
for s, r in EXP_CASES:
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy=s, spawn_key=(r,))))
    exp.append(g.exponential(1.0, EXP_N))
meta["rng_exp_cases"] = [[s, r] for s, r in EXP_CASES]
put("rng_exp", np.array(exp))

# ---------------------------------------------------------------- sim (_simulate_once)
service1, servers1, _ = wan_gpu_fixture(J=10, eta=0.2, seed=101)
petals = cs.greedy_cache_allocation(cs.greedy_block_placement(servers1, service1, 7, 0.2, 0.7).placement)
nu = petals.total_rate
SIM_CASES = [
    dict(rates=(1.0,), caps=(1,), lam=0.5, n=20000, wf=0.1, seed=5, rep=0, jobs=False),
    dict(rates=(1.5, 0.6), caps=(1, 2), lam=1.3, n=8000, wf=0.0, seed=29, rep=0, jobs=True),
    dict(rates=(2.0, 0.7, 0.3), caps=(2, 3, 2), lam=2.4, n=20000, wf=0.1, seed=13, rep=3, jobs=False),
    dict(rates=(1.0, 0.5), caps=(1, 1), lam=1.575, n=20000, wf=0.1, seed=3, rep=1, jobs=False),
    dict(rates=tuple(petals.rates), caps=tuple(petals.capacities), lam=0.2, n=10000, wf=0.1,
         seed=1, rep=0, jobs=True),
    dict(rates=tuple(petals.rates), caps=tuple(petals.capacities), lam=0.95 * nu, n=20000,
         wf=0.1, seed=1, rep=7, jobs=False),
    dict(rates=(3.0, 2.0, 2.0, 1.0, 0.5), caps=(2, 3, 1, 4, 5), lam=9.0, n=6000, wf=0.5,
         seed=11, rep=2, jobs=True),
    dict(rates=(1.0,), caps=(1,), lam=0.3, n=1, wf=0.0, seed=9, rep=0, jobs=True),
    dict(rates=(1.0,), caps=(7,), lam=6.0, n=3001, wf=0.25, seed=2, rep=5, jobs=False),
]
meta["sim_cases"] = []
for i, c in enumerate(SIM_CASES):
    cfg = cs.SimConfig(rates=c["rates"], capacities=c["caps"], workload=cs.PoissonWorkload(c["lam"]),
                       horizon_jobs=c["n"], warmup_fraction=c["wf"], seed=c["seed"], replications=1,
                       collect_jobs=c["jobs"])
    r = _simulate_once(cfg, c["rep"])
    entry = dict(c)
    entry["rates"] = list(c["rates"])
    entry["caps"] = list(c["caps"])
    entry["fields"] = {f: getattr(r, f) for f in (
        "wait_sum", "service_sum", "counted", "window_s", "mean_occupancy", "occ_first_half",
        "occ_second_half", "lambda_effective", "end_queue_len")}
    entry["responses"] = put(f"sim{i}_responses", r.responses)
    entry["busy"] = put(f"sim{i}_busy", np.array(r.busy_time_s))
    entry["rep_mean"] = float(r.responses.mean()) if r.responses.size else None
    if c["jobs"]:
        entry["job_records"] = put(f"sim{i}_jobs", np.array(r.jobs, dtype=np.float64))
    meta["sim_cases"].append(entry)

# ---------------------------------------------------------------- run_sim
RUN_CASES = [
    dict(rates=(1.0,), caps=(2,), lam=1.0, n=5000, wf=0.1, seed=11, reps=4),
    dict(rates=tuple(petals.rates), caps=tuple(petals.capacities), lam=0.7 * nu, n=4000, wf=0.1,
         seed=1, reps=3),
    dict(rates=(2.0, 0.7, 0.3), caps=(2, 3, 2), lam=1.0, n=3000, wf=0.2, seed=13, reps=5),
]
meta["runsim_cases"] = []
for c in RUN_CASES:
    st = cs.run_sim(cs.SimConfig(rates=c["rates"], capacities=c["caps"],
                                 workload=cs.PoissonWorkload(c["lam"]), horizon_jobs=c["n"],
                                 warmup_fraction=c["wf"], seed=c["seed"], replications=c["reps"]))
    e = dict(c)
    e["rates"] = list(c["rates"])
    e["caps"] = list(c["caps"])
    e["stats"] = st.to_dict()
    meta["runsim_cases"].append(e)


# ---------------------------------------------------------------- compose
def server_rows(servers):
    return [[s.id, s.memory_bytes, s.comm_time_s, s.per_block_compute_s] for s in servers]


def compose_case(name, servers, service, c, lam, rho):
    e = dict(name=name, servers=server_rows(servers),
             service=[service.block_count, service.block_bytes, service.cache_slot_bytes],
             capacity=c, arrival_rate=lam, load_target=rho)
    try:
        res = cs.greedy_block_placement(servers, service, c, lam, rho)
    except cs.InfeasibleError as exc:
        e["gbp"] = {"infeasible": str(exc)}
        return e
    e["gbp"] = dict(first=list(res.placement.first_block), count=list(res.placement.block_count),
                    chains=[list(ch) for ch in res.chains], scaled_rate=res.scaled_rate,
                    rate_satisfied=res.rate_satisfied, max_blocks=list(res.profile.max_blocks),
                    bound_time=list(res.profile.bound_time_s))
    system = cs.greedy_cache_allocation(res.placement)
    e["gca"] = dict(chains=[list(ch.server_ids) for ch in system.chains],
                    caps=list(system.capacities), times=[ch.service_time_s for ch in system.chains],
                    n_edges=len(cs.feasible_edges(res.placement)))
    return e


def placement_case(name, placement, residual=None):
    e = dict(name=name, servers=server_rows(placement.servers),
             service=[placement.service.block_count, placement.service.block_bytes,
                      placement.service.cache_slot_bytes],
             first=list(placement.first_block), count=list(placement.block_count),
             residual=residual)
    system = cs.greedy_cache_allocation(placement, residual)
    e["gca"] = dict(chains=[list(ch.server_ids) for ch in system.chains],
                    caps=list(system.capacities), times=[ch.service_time_s for ch in system.chains],
                    n_edges=len(cs.feasible_edges(placement)))
    return e


comp = []
five = (cs.ServiceSpec(3, 10, 1), tuple(cs.ServerSpec(f"j{l}", 30 if l == 2 else 20,
                                                      2.0 if l == 2 else 1.0, l * 0.01)
                                        for l in range(1, 6)))
for c, lam in [(1, 1.0), (1, 0.7 / (3 + 5 * 0.01)), (100, 1.0), (2, 1.0)]:
    comp.append(compose_case("five_server", five[1], five[0], c, lam, 0.7))
for name, (svc, srv) in [("uniform_tradeoff", uniform_tradeoff_instance()), ("tiered", tiered_instance())]:
    for c in (1, 2, 5, 10, 100):
        for lam in (0.5, 5.0, 100.0, 1e9):
            comp.append(compose_case(name, srv, svc, c, lam, 0.7))
for J in (10, 20):
    svc, srv, _ = wan_gpu_fixture(J=J, eta=0.2, seed=101)
    for c in (1, 3, 7, 20, 100, 351):
        for lam in (0.05, 0.2, 1.0, 1e9):
            comp.append(compose_case(f"wan{J}", srv, svc, c, lam, 0.7))
rng = philox(1234)
for i in range(120):
    svc = random_service(rng, max_blocks=8)
    srv = random_servers(rng, int(rng.integers(1, 7)), svc)
    comp.append(placement_case(f"random_placement{i}", random_placement(rng, svc, srv)))
    c = int(rng.integers(1, 5))
    comp.append(compose_case(f"random_gbp{i}", srv, svc, c, float(rng.uniform(0, 5)), 0.7))
rng = philox(55)
for i in range(120):
    svc = cs.ServiceSpec(int(rng.integers(1, 9)), 10, 1)
    J = int(rng.integers(1, 8))
    srv = tuple(cs.ServerSpec(f"t{int(rng.integers(0, 100)):02d}_{k}", int(rng.integers(10, 120)),
                              float(rng.integers(0, 3)), float(rng.integers(0, 2)) * 0.5)
                for k in range(J))
    comp.append(placement_case(f"tie_heavy{i}", random_placement(rng, svc, srv)))
# residual override and depleted-hop cases from the reference tests
pl = cs.greedy_block_placement(five[1], five[0], 1, 1.0, 0.7).placement
resid = {sid: cs.cache_slots(pl, sid) for sid in pl.used_ids()}
resid["j2"] = 0
comp.append(placement_case("five_server_resid", pl, resid))
dep = cs.BlockPlacement(cs.ServiceSpec(3, 10, 1),
                        (cs.ServerSpec("x", 30, 0.1, 0.0), cs.ServerSpec("y", 20, 0.2, 0.0),
                         cs.ServerSpec("z", 23, 0.1, 0.01)), (1, 1, 2), (2, 1, 2))
comp.append(placement_case("depleted_hop", dep))
meta["compose_cases"] = comp

np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
with open(os.path.join(HERE, "golden.json"), "w") as fh:
    json.dump(meta, fh, indent=0, allow_nan=True)
print("wrote", len(arrays), "arrays,", len(comp), "compose cases")
