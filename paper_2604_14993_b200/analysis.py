"""Chain rates and steady-state occupancy bounds -- CUDA-backed drop-in for
chainserve/analysis.py.

``ChainRates`` is the compose -> simulate handoff type (analysis.py:27-64).
``occupancy_bounds`` / ``birth_death_mean_occupancy`` (analysis.py:84-147)
run in bounds.cu, one CTA per (system, bound); ``bound_curve`` and
``tune_capacity_bound`` (analysis.py:270-336) evaluate the whole capacity
sweep c = 1..c_max as three batched launches (GBP-CR, GCA, bounds) instead of
c_max sequential compose + bound calls.  The bounds use CUDA log/exp/log1p:
agreement with the reference is within 1e-9 relative; the
death rates themselves (analysis.py:67-81) are bit-exact.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as N
from .errors import InfeasibleError, UnstableError
from .model import ComposedSystem, ServerSpec, ServiceSpec, py_sum


@dataclass(frozen=True)
class ChainRates:
    """Chain service rates (descending) with aligned capacities."""

    rates: tuple[float, ...]
    capacities: tuple[int, ...]

    def __post_init__(self):
        if len(self.rates) != len(self.capacities):
            raise ValueError("one capacity per rate required")
        if any(r <= 0 for r in self.rates):
            raise ValueError("rates must be positive")
        if any(c < 1 or not isinstance(c, int) for c in self.capacities):
            raise ValueError("capacities must be positive integers")
        if any(a < b for a, b in zip(self.rates, self.rates[1:])):
            raise ValueError("rates must be sorted in descending order")

    @classmethod
    def from_system(cls, system: ComposedSystem) -> "ChainRates":
        return cls(system.rates, system.capacities)

    @classmethod
    def from_unsorted(cls, rates: Sequence[float], capacities: Sequence[int]) -> "ChainRates":
        order = sorted(range(len(rates)), key=lambda i: -rates[i])  # stable: ties keep order
        return cls(tuple(rates[i] for i in order), tuple(capacities[i] for i in order))

    @property
    def chain_count(self) -> int:
        return len(self.rates)

    @property
    def total_rate(self) -> float:
        return py_sum(r * c for r, c in zip(self.rates, self.capacities))

    @property
    def total_capacity(self) -> int:
        return sum(self.capacities)


def death_rate_bounds(rates: ChainRates, n: int) -> tuple[float, float]:
    """(upper, lower) aggregate departure rate with n jobs (analysis.py:67-81):
    jobs packed onto the fastest chains / onto the slowest.  Scalar helper;
    the batched bounds evaluate the same sums on the device."""
    if n < 0:
        raise ValueError("n must be >= 0")
    fast = slow = 0.0
    before = 0                      # capacity of the faster chains
    after = rates.total_capacity    # capacity of the slower chains
    for mu, c in zip(rates.rates, rates.capacities):
        after -= c
        fast += mu * min(c, max(n - before, 0))
        slow += mu * min(c, max(n - after, 0))
        before += c
    return fast, slow


@dataclass(frozen=True)
class OccupancyBounds:
    """Bracketing mean occupancy (jobs) and mean response time (seconds)."""

    lower_mean_occupancy: float
    upper_mean_occupancy: float
    lower_mean_response_s: float
    upper_mean_response_s: float


def _dev(torch, a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def occupancy_bounds_batch(systems: Sequence[ChainRates], arrival_rates: Sequence[float]) -> np.ndarray:
    """occupancy_bounds for many systems in one launch.  Returns the
    cs_bounds_out records (N.BOUNDS_DTYPE); status CS_UNSTABLE marks
    lam >= total_rate (no bounds computed)."""
    lib = N.load()
    import torch

    P = len(systems)
    if P != len(arrival_rates):
        raise ValueError("one arrival rate per system required")
    out = np.zeros(P, N.BOUNDS_DTYPE)
    if P == 0:
        return out
    pts = (N.BoundPoint * P)()
    rates, caps, base, max_cap = [], [], 0, 1
    for p, (cr, lam) in enumerate(zip(systems, arrival_rates)):
        pts[p].n_chains, pts[p].chain_base, pts[p].lam = cr.chain_count, base, float(lam)
        rates.extend(cr.rates)
        caps.extend(cr.capacities)
        base += cr.chain_count
        max_cap = max(max_cap, cr.total_capacity)
    d_pts = _dev(torch, np.frombuffer(pts, np.uint8), torch.uint8)
    d_rates = _dev(torch, np.asarray(rates or [0.0], np.float64), torch.float64)
    d_caps = _dev(torch, np.asarray(caps or [0], np.int32), torch.int32)
    d_ws = torch.empty(P * 2 * (max_cap + 1), dtype=torch.float64, device="cuda")
    d_out = torch.zeros(P * out.itemsize, dtype=torch.uint8, device="cuda")
    st = lib.cs_occupancy_bounds(d_pts.data_ptr(), P, d_rates.data_ptr(), d_caps.data_ptr(), max_cap,
                                 d_ws.data_ptr(), d_out.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream)
    N.check(st, "cs_occupancy_bounds")
    return d_out.cpu().numpy().view(N.BOUNDS_DTYPE).copy()


def _unstable(lam: float, nu: float) -> UnstableError:
    return UnstableError(f"arrival rate {lam:.6g} >= total service rate {nu:.6g}")


def occupancy_bounds(rates: ChainRates, arrival_rate: float) -> OccupancyBounds:
    """Theoretical bracket on steady-state mean occupancy and response time
    (analysis.py:121-147)."""
    lam = float(arrival_rate)
    if lam <= 0:
        raise ValueError("arrival_rate must be positive")
    nu = rates.total_rate
    if lam >= nu:
        raise _unstable(lam, nu)
    r = occupancy_bounds_batch([rates], [lam])[0]
    N.check(int(r["status"]), "occupancy_bounds")
    return OccupancyBounds(float(r["lower_occupancy"]), float(r["upper_occupancy"]),
                           float(r["lower_response_s"]), float(r["upper_response_s"]))


def birth_death_mean_occupancy(arrival_rate: float, death_rates: Sequence[float],
                               total_rate: float) -> float:
    """Mean occupancy of the birth-death process with death_rates[n-1] for
    n = 1..C jobs and total_rate beyond C (analysis.py:84-109)."""
    lam, nu = float(arrival_rate), float(total_rate)
    if lam <= 0:
        raise ValueError("arrival_rate must be positive")
    if lam >= nu:
        raise _unstable(lam, nu)
    d = np.asarray(death_rates, dtype=float)
    if d.size == 0 or np.any(d <= 0):
        raise ValueError("death rates must be positive")
    lib = N.load()
    import torch

    pt = N.BdPoint(int(d.size), 0, lam, nu)
    d_pt = _dev(torch, np.frombuffer(pt, np.uint8), torch.uint8)
    d_d = _dev(torch, d, torch.float64)
    d_ws = torch.empty(d.size + 1, dtype=torch.float64, device="cuda")
    d_out = torch.empty(1, dtype=torch.float64, device="cuda")
    st = lib.cs_birth_death_occupancy(d_pt.data_ptr(), 1, d_d.data_ptr(), int(d.size), d_ws.data_ptr(),
                                      d_out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    N.check(st, "cs_birth_death_occupancy")
    return float(d_out.cpu()[0])


@dataclass(frozen=True)
class BoundCurveRow:
    capacity: int
    chain_count: int
    total_capacity: int
    total_rate: float
    lower_response_s: float | None
    upper_response_s: float | None
    stable: bool


def bound_curve(servers: Sequence[ServerSpec], service: ServiceSpec, arrival_rate: float,
                load_target: float) -> list[BoundCurveRow]:
    """Response-time bounds for every workable capacity (analysis.py:270-297):
    GBP-CR for all c in [1, c_max], GCA for the feasible ones, bounds for the
    stable ones -- three batched launches."""
    from . import _compose as CE
    from .placement import _validate, capacity_upper_bound

    c_max = capacity_upper_bound(servers, service)
    _validate(arrival_rate, load_target, 1)
    fleet = CE.Fleet.of(servers)
    grid = list(range(1, c_max + 1))
    g = CE.gbp_batch([fleet], [service] * len(grid), grid, [arrival_rate] * len(grid),
                     [load_target] * len(grid), fleet_of_point=[0] * len(grid))
    feas = []
    for p in range(len(grid)):
        st = int(g.status[p])
        if st == N.CS_INFEASIBLE:
            continue
        N.check(st, "bound_curve: greedy_block_placement")
        feas.append(p)
    if not feas:
        return []
    J = len(fleet.servers)
    firsts = [g.first[g.server_base[p]:g.server_base[p] + J] for p in feas]
    counts = [g.count[g.server_base[p]:g.server_base[p] + J] for p in feas]
    a = CE.gca_batch([fleet], [service] * len(feas), firsts, counts, fleet_of_point=[0] * len(feas))
    systems, caps_of = [], []
    for i, p in enumerate(feas):
        st = int(a.status[i])
        if st == N.CS_INVALID:
            raise ValueError("bound_curve: greedy_cache_allocation: invalid placement")
        if st != N.CS_OK:
            raise AssertionError("bound_curve: greedy_cache_allocation failed")
        K = int(a.n_chains[i])
        if K == 0:
            continue
        rates = tuple(float(x) for x in 1.0 / a.times[i, :K])
        systems.append(ChainRates(rates, tuple(int(x) for x in a.caps[i, :K])))
        caps_of.append(grid[p])
    lam = float(arrival_rate)
    if systems and lam <= 0:  # occupancy_bounds on the first (stable) row raises
        raise ValueError("arrival_rate must be positive")
    b = occupancy_bounds_batch(systems, [lam] * len(systems))
    rows = []
    for c, cr, r in zip(caps_of, systems, b):
        nu = cr.total_rate
        if lam >= nu:
            rows.append(BoundCurveRow(c, cr.chain_count, cr.total_capacity, nu, None, None, False))
            continue
        N.check(int(r["status"]), "bound_curve: occupancy_bounds")
        rows.append(BoundCurveRow(c, cr.chain_count, cr.total_capacity, nu,
                                  float(r["lower_response_s"]), float(r["upper_response_s"]), True))
    return rows


@dataclass(frozen=True)
class BoundTuning:
    c_star: int
    which: str
    rows: tuple[BoundCurveRow, ...]


def tune_capacity_bound(servers: Sequence[ServerSpec], service: ServiceSpec, arrival_rate: float,
                        load_target: float, which: str = "lower") -> BoundTuning:
    """Capacity minimising the chosen response-time bound; ties to the
    smaller capacity, unstable rows excluded (analysis.py:307-336)."""
    if which not in ("lower", "upper"):
        raise ValueError("which must be 'lower' or 'upper'")
    rows = bound_curve(servers, service, arrival_rate, load_target)
    stable = [r for r in rows if r.stable]
    if not stable:
        raise UnstableError(f"no capacity yields a stable system at arrival rate {arrival_rate:.6g}")
    key = (lambda r: r.lower_response_s) if which == "lower" else (lambda r: r.upper_response_s)
    best = min(stable, key=key)  # first minimum = smallest capacity
    if not key(best) < math.inf:
        raise UnstableError(f"no capacity yields a stable system at arrival rate {arrival_rate:.6g}")
    return BoundTuning(best.capacity, which, tuple(rows))
