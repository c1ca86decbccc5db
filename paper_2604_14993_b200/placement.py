"""GBP-CR block placement and capacity tuning -- CUDA-backed drop-in for
chainserve/placement.py.

``greedy_block_placement`` keeps the reference signature (placement.py:67-73)
and result type; the reservation profile, the (amortized time, id) sort and
the greedy chain scan run in compose.cu:gbp_kernel.  ``tune_capacity_surrogate``
(placement.py:161-200) evaluates every capacity c in [1, c_max] in ONE batched
launch instead of c_max sequential calls.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _compose as CE
from .errors import InfeasibleError
from .model import BlockPlacement, ServerSpec, ServiceSpec


@dataclass(frozen=True)
class ReservationProfile:
    """m_j(c) and t_j(c) per server (placement.py:20-32)."""

    capacity: int
    max_blocks: tuple[int, ...]
    bound_time_s: tuple[float, ...]

    def amortized_time_s(self, index: int) -> float:
        m = self.max_blocks[index]
        if m == 0:
            raise ValueError("amortized time undefined for a server hosting no blocks")
        return self.bound_time_s[index] / m


@dataclass(frozen=True)
class PlacementResult:
    placement: BlockPlacement
    chains: tuple[tuple[str, ...], ...]
    scaled_rate: float
    rate_satisfied: bool
    capacity: int
    profile: ReservationProfile

    @property
    def chain_count(self) -> int:
        return len(self.chains)


def _validate(arrival_rate: float, load_target: float, capacity: int) -> None:
    if arrival_rate < 0:
        raise ValueError("arrival_rate must be >= 0")
    if not 0 < load_target < 1:
        raise ValueError("load_target must lie in (0, 1)")
    if capacity < 1:
        raise ValueError("capacity must be >= 1")


def _results(out: CE.GbpOut, p: int, fleet: CE.Fleet, service: ServiceSpec, capacity: int,
             raise_infeasible: bool = True):
    b, n = int(out.server_base[p]), int(out.n_servers[p])
    servers = fleet.servers
    profile = ReservationProfile(
        int(capacity), tuple(int(x) for x in out.max_blocks[b:b + n]),
        tuple(float(x) for x in out.bound_time[b:b + n]))
    st = int(out.status[p])
    if st == 1:
        if raise_infeasible:
            raise InfeasibleError(
                f"required capacity {capacity} infeasible: no server can host a single block")
        return None
    if st != 0:
        raise ValueError(f"greedy_block_placement: invalid input (status {st})")
    order = out.order[b:b + n]
    ends = out.chain_end[b:b + n]
    chains, cur = [], []
    for q in range(n):
        j = int(order[q])
        if j < 0:
            break
        cur.append(servers[j].id)
        if ends[q]:
            chains.append(tuple(cur))
            cur = []
    placement = BlockPlacement(service, servers, tuple(int(x) for x in out.first[b:b + n]),
                               tuple(int(x) for x in out.count[b:b + n]))
    return PlacementResult(placement, tuple(chains), float(out.scaled_rate[p]),
                           bool(out.rate_satisfied[p]), int(capacity), profile)


def greedy_block_placement(servers: Sequence[ServerSpec], service: ServiceSpec, capacity: int,
                           arrival_rate: float, load_target: float) -> PlacementResult:
    """Algorithm 1 (GBP-CR), placement.py:67-132, on the GPU."""
    _validate(arrival_rate, load_target, capacity)
    fleet = CE.Fleet.of(servers)
    out = CE.gbp_batch([fleet], [service], [capacity], [arrival_rate], [load_target])
    return _results(out, 0, fleet, service, capacity)


def greedy_block_placement_batch(servers_list: Sequence[Sequence[ServerSpec]],
                                 services: Sequence[ServiceSpec], capacities: Sequence[int],
                                 arrival_rates: Sequence[float], load_targets: Sequence[float]):
    """Batched GBP-CR: one GPU launch for all points.  Infeasible points give None."""
    fleets = [CE.Fleet.of(s) for s in servers_list]
    for a, r, c in zip(arrival_rates, load_targets, capacities):
        _validate(a, r, c)
    out = CE.gbp_batch(fleets, services, capacities, arrival_rates, load_targets)
    return [_results(out, p, fleets[p], services[p], capacities[p], raise_infeasible=False)
            for p in range(len(capacities))]


def reservation_profile(servers: Sequence[ServerSpec], service: ServiceSpec,
                        capacity: int) -> ReservationProfile:
    """m_j(c) = min(M_j // (s_m + s_c c), L), t_j = tau_c + tau_p m_j (placement.py:35-48)."""
    if capacity < 1:
        raise ValueError("capacity must be >= 1")
    fleet = CE.Fleet.of(servers)
    out = CE.gbp_batch([fleet], [service], [capacity], [0.0], [0.5])
    n = len(fleet.servers)
    return ReservationProfile(int(capacity), tuple(int(x) for x in out.max_blocks[:n]),
                              tuple(float(x) for x in out.bound_time[:n]))


def capacity_upper_bound(servers: Sequence[ServerSpec], service: ServiceSpec) -> int:
    """(max M - s_m) // s_c (placement.py:135-143)."""
    if not servers:
        raise InfeasibleError("no servers given")
    c_max = (max(s.memory_bytes for s in servers) - service.block_bytes) // service.cache_slot_bytes
    if c_max < 1:
        raise InfeasibleError("no server can host one block plus one cache slot")
    return c_max


@dataclass(frozen=True)
class TuningRow:
    capacity: int
    chain_count: int | None
    scaled_cost: int | None
    rate_satisfied: bool
    achieved_rate: float


@dataclass(frozen=True)
class CapacityTuning:
    c_star: int
    rows: tuple[TuningRow, ...]


def tune_capacity_surrogate(servers: Sequence[ServerSpec], service: ServiceSpec,
                            arrival_rate: float, load_target: float) -> CapacityTuning:
    """argmin_c c*K(c) over rate-feasible c (placement.py:161-200), all c in one launch."""
    c_max = capacity_upper_bound(servers, service)
    _validate(arrival_rate, load_target, 1)
    fleet = CE.Fleet.of(servers)
    caps = list(range(1, c_max + 1))
    out = CE.gbp_batch([fleet], [service] * len(caps), caps, [arrival_rate] * len(caps),
                       [load_target] * len(caps), fleet_of_point=[0] * len(caps))
    rows, best_c, best_cost, best_rate = [], None, None, 0.0
    for p, c in enumerate(caps):
        st = int(out.status[p])
        if st == 1:
            rows.append(TuningRow(c, None, None, False, 0.0))
            continue
        if st != 0:
            raise ValueError(f"tune_capacity_surrogate: invalid input (status {st})")
        k = int(out.n_chains[p])
        achieved = c * float(out.scaled_rate[p])
        best_rate = max(best_rate, achieved)
        if bool(out.rate_satisfied[p]):
            cost = c * k
            rows.append(TuningRow(c, k, cost, True, achieved))
            if best_cost is None or cost < best_cost:
                best_cost, best_c = cost, c
        else:
            rows.append(TuningRow(c, k, None, False, achieved))
    if best_c is None:
        raise InfeasibleError(
            f"no capacity in [1, {c_max}] meets the rate target "
            f"{arrival_rate / load_target:.6g}/s; best achievable total rate is {best_rate:.6g}/s",
            best_rate=best_rate)
    return CapacityTuning(best_c, tuple(rows))
