"""Command line for the compose -> simulate path (the reference's
``chainserve compose`` / ``chainserve simulate``, cli.py:43-92,179-243).

    python -m paper_2604_14993_b200 compose  --service sys.json --lambda 5 --out runs/a
    python -m paper_2604_14993_b200 simulate --chains runs/a/chains.json --lambda 5 --reps 32 --out runs/a

``compose`` picks the per-chain capacity c (``--c``, else the batched
surrogate tuner or a bound tuner), places blocks (GBP-CR) and allocates cache
slots (GCA) on the GPU, and writes placement.json and a self-contained
chains.json.  ``simulate`` reruns a chains.json through ``run_sim`` on the GPU
and writes stats.json (plus the per-job CSV with ``--jobs-csv``).  Same files,
same exit codes (0 ok, 2 infeasible composition, 3 unstable system, 1 other
errors).  The reference's token-level trace mode (``--trace``, request-trace
ingest and GPU profiles) and its tune / analyze / report commands are outside
this engine's scope and are refused explicitly.
"""

from __future__ import annotations

import argparse
import csv
import sys
from pathlib import Path

from . import analysis, placement as placement_mod, sim
from .cache_alloc import greedy_cache_allocation
from .config import (load_composed, load_servers, load_system, placement_to_dict, provenance, save_json,
                     system_to_dict)
from .errors import InfeasibleError, UnstableError
from .model import evaluate_composition
from .workload import PoissonWorkload


def _out(args) -> Path:
    d = Path(args.out)
    d.mkdir(parents=True, exist_ok=True)
    return d


def _choose_capacity(args, servers, service) -> int:
    if args.c is not None:
        return args.c
    if args.tune in (None, "surrogate"):
        return placement_mod.tune_capacity_surrogate(servers, service, args.lam, args.rho_bar).c_star
    return analysis.tune_capacity_bound(servers, service, args.lam, args.rho_bar, which=args.tune).c_star


def cmd_compose(args) -> int:
    out = _out(args)
    service, servers = load_system(args.service)
    if args.servers:
        servers = load_servers(args.servers)
    if not servers:
        raise InfeasibleError("server list is empty")
    c = _choose_capacity(args, servers, service)
    placed = placement_mod.greedy_block_placement(servers, service, c, args.lam, args.rho_bar)
    system = greedy_cache_allocation(placed.placement)
    report = evaluate_composition(placed.placement, system.chains, system.capacities, args.lam, args.rho_bar)
    inputs = {"service": args.service}
    if args.servers:
        inputs["servers"] = args.servers
    prov = provenance(inputs, command="compose", capacity=c, arrival_rate=args.lam, load_target=args.rho_bar)
    save_json(out / "placement.json", {"provenance": prov, "placement": placement_to_dict(placed.placement)})
    chains = {"provenance": prov, **system_to_dict(system, capacity_parameter=c)}
    chains["evaluation"] = {"objective_total_capacity": report.objective, "rate_ok": report.rate_ok,
                            "memory_ok": report.memory_ok, "total_rate_per_s": report.total_rate,
                            "required_rate_per_s": report.required_rate,
                            "violations": list(report.violations)}
    save_json(out / "chains.json", chains)
    print(f"composed {len(system.chains)} chains (c={c}), total rate {system.total_rate:.6g}/s, "
          f"rate_ok={report.rate_ok}, memory_ok={report.memory_ok}")
    return 0


def cmd_simulate(args) -> int:
    if args.trace or args.profiles or args.rtt:
        raise NotImplementedError("token-level trace simulation from the CLI is outside this engine's scope; "
                                  "use run_sim with a TraceWorkload")
    if args.lam is None:
        raise ValueError("either --trace or --lambda is required")
    out = _out(args)
    system, _ = load_composed(args.chains)
    rates = analysis.ChainRates.from_system(system)
    horizon = args.jobs
    if args.lam >= rates.total_rate:  # overloaded: the reference caps the horizon
        horizon = min(horizon, 100_000)
        print(f"warning: arrival rate {args.lam:.6g} >= total rate {rates.total_rate:.6g}; "
              f"capping horizon at {horizon} jobs", file=sys.stderr)
    cfg = sim.SimConfig(rates=rates.rates, capacities=rates.capacities, workload=PoissonWorkload(args.lam),
                        policy=args.policy, horizon_jobs=horizon, warmup_fraction=args.warmup, seed=args.seed,
                        replications=args.reps, collect_jobs=args.jobs_csv is not None, workers=args.workers)
    stats = sim.run_sim(cfg)
    prov = provenance({"chains": args.chains}, command="simulate", policy=args.policy, arrival_rate=args.lam,
                      horizon_jobs=horizon, seed=args.seed, replications=args.reps,
                      warmup_fraction=args.warmup)
    save_json(out / "stats.json", {"provenance": prov, **stats.to_dict()})
    if args.jobs_csv:
        with open(args.jobs_csv, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["replication", "arrival_s", "start_s", "finish_s", "chain_id"])
            w.writerows(stats.job_records)
    print(f"{args.policy}: mean response {stats.mean_response_s:.6g} s "
          f"(+/- {stats.response_ci_half_width_s:.2g}), occupancy {stats.mean_occupancy:.6g}")
    return 0


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2604_14993_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("compose", help="place blocks and allocate cache capacity (GPU)")
    p.add_argument("--out", required=True, help="output directory")
    p.add_argument("--service", required=True, help="system JSON (service + servers)")
    p.add_argument("--servers", help="optional separate server list JSON")
    p.add_argument("--lambda", dest="lam", type=float, required=True)
    p.add_argument("--rho-bar", dest="rho_bar", type=float, default=0.7)
    p.add_argument("--c", type=int, help="required per-chain capacity (skips tuning)")
    p.add_argument("--tune", choices=["surrogate", "lower", "upper"])
    p.set_defaults(func=cmd_compose)
    p = sub.add_parser("simulate", help="discrete-event simulation of a chains.json (GPU)")
    p.add_argument("--out", required=True, help="output directory")
    p.add_argument("--chains", required=True)
    p.add_argument("--lambda", dest="lam", type=float)
    p.add_argument("--trace")
    p.add_argument("--profiles")
    p.add_argument("--rtt")
    p.add_argument("--policy", default="jffc", choices=list(sim.POLICIES))
    p.add_argument("--jobs", type=int, default=100_000)
    p.add_argument("--warmup", type=float, default=0.1)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--reps", type=int, default=1)
    p.add_argument("--workers", type=int, default=1)
    p.add_argument("--jobs-csv", help="also write per-job records to this CSV")
    p.set_defaults(func=cmd_simulate)
    return ap


def main(argv=None) -> int:
    args = parser().parse_args(argv)
    try:
        return args.func(args)
    except InfeasibleError as exc:
        print(f"infeasible: {exc}", file=sys.stderr)
        return 2
    except UnstableError as exc:
        print(f"unstable: {exc}", file=sys.stderr)
        return 3
    except Exception as exc:  # as the reference: any other failure is exit code 1
        print(f"error: {exc}", file=sys.stderr)
        return 1
