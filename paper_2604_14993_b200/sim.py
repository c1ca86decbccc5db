"""JFFC simulation -- CUDA-backed drop-in for chainserve/sim.py.

``run_sim(config) -> SimStats`` keeps the reference signature (sim.py:397) and
statistics; the replications (RNG streams, event loops, per-rep means and the
exact order statistics behind the percentiles) run on the GPU through
``cs_run_sim_host``.  ``run_sim_batch`` simulates many sweep points (e.g. 16
arrival rates) that share seed/replications in ONE call; each point's
SimStats is identical to a separate ``run_sim`` call.

The rest of the signature (dedicated-queue
policies jsq/sa-jsq/jiq/sed, sampled and trace workloads, the time-horizon
mode) runs through ``sim_ext.simulate_ext`` (csrc/sim_ext.cu), also on the
GPU and bit-exact.
"""

from __future__ import annotations

import ctypes as C
import functools
import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as N
from .model import ServerChain, py_sum
from .workload import PoissonWorkload, SampledWorkload, ServiceTimeModel, TraceWorkload

POLICIES = ("jffc", "jsq", "jiq", "sed", "sa-jsq")
CENTRAL_QUEUE = None


@dataclass(frozen=True)
class SimConfig:
    """Simulation knobs; same fields and validation as sim.py:31-72."""

    rates: tuple[float, ...]
    capacities: tuple[int, ...]
    workload: PoissonWorkload | SampledWorkload | TraceWorkload
    policy: str = "jffc"
    horizon_jobs: int = 100_000
    horizon_time_s: float | None = None
    warmup_fraction: float = 0.1
    seed: int = 1
    replications: int = 1
    chains: tuple[ServerChain, ...] | None = None
    service_model: ServiceTimeModel | None = None
    collect_jobs: bool = False
    workers: int = 1

    def __post_init__(self):
        if self.policy not in POLICIES:
            raise ValueError(f"unknown policy {self.policy!r}; choose from {POLICIES}")
        if not self.rates or len(self.rates) != len(self.capacities):
            raise ValueError("rates and capacities must align and be nonempty")
        if any(b > a for a, b in zip(self.rates, self.rates[1:])):
            raise ValueError("rates must be sorted in descending order")
        if any(c < 1 for c in self.capacities):
            raise ValueError("capacities must be >= 1")
        if self.horizon_jobs < 1:
            raise ValueError("horizon_jobs must be >= 1")
        if self.horizon_time_s is not None and self.horizon_time_s <= 0:
            raise ValueError("horizon_time_s must be positive")
        if not 0.0 <= self.warmup_fraction <= 0.5:
            raise ValueError("warmup_fraction must lie in [0, 0.5]")
        if self.replications < 1:
            raise ValueError("replications must be >= 1")
        if isinstance(self.workload, TraceWorkload):
            if self.chains is None or self.service_model is None:
                raise ValueError("trace workloads need chains and a service-time model")
            if len(self.chains) != len(self.rates):
                raise ValueError("one chain object per rate required")

    @property
    def total_rate(self) -> float:
        return py_sum(r * c for r, c in zip(self.rates, self.capacities))


def policy_step(policy: str, rates: Sequence[float], capacities: Sequence[int],
                in_service: Sequence[int], queue_lengths: Sequence[int], event: tuple):
    """Dispatch decision on a snapshot (sim.py:75-117); the GPU event loop
    inlines the "jffc" branch (first chain with a free slot)."""
    K = len(rates)
    kind = event[0]
    if kind == "completion":
        k = event[1]
        backlog = queue_lengths[0] if policy == "jffc" else queue_lengths[k]
        return k if backlog > 0 else CENTRAL_QUEUE
    if kind != "arrival":
        raise ValueError(f"unknown event {event!r}")
    if policy == "jffc":
        return next((k for k in range(K) if in_service[k] < capacities[k]), CENTRAL_QUEUE)
    load = [in_service[k] + queue_lengths[k] for k in range(K)]
    if policy in ("jsq", "sa-jsq"):
        return min(range(K), key=lambda k: (load[k], k))
    if policy == "jiq":
        for k in range(K):
            if load[k] < capacities[k]:
                return k
        return min(range(K), key=lambda k: (load[k], k))
    if policy == "sed":
        return min(range(K), key=lambda k: ((load[k] + 1) / rates[k], k))
    raise ValueError(f"unknown policy {policy!r}")


@dataclass(frozen=True)
class SimStats:
    """Aggregated steady-state statistics (sim.py:327-380)."""

    policy: str
    jobs_counted: int
    mean_response_s: float
    median_response_s: float
    p95_response_s: float
    p99_response_s: float
    mean_waiting_s: float
    mean_service_s: float
    mean_occupancy: float
    response_ci_half_width_s: float
    occupancy_ci_half_width: float
    per_chain_utilization: tuple[float, ...]
    lambda_effective: float
    little_law_gap: float
    unstable: bool
    seed: int
    replications: int
    rep_mean_response_s: tuple[float, ...]
    rep_mean_occupancy: tuple[float, ...]
    occ_first_half: float
    occ_second_half: float
    end_queue_len: int
    job_records: tuple | None = None

    _KEYS = ("policy", "jobs_counted", "mean_response_s", "median_response_s", "p95_response_s",
             "p99_response_s", "mean_waiting_s", "mean_service_s", "mean_occupancy",
             "response_ci_half_width_s", "occupancy_ci_half_width", "per_chain_utilization",
             "lambda_effective", "little_law_gap", "unstable", "seed", "replications",
             "rep_mean_response_s", "rep_mean_occupancy", "occ_first_half", "occ_second_half",
             "end_queue_len")

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k in self._KEYS}
        for k in ("per_chain_utilization", "rep_mean_response_s", "rep_mean_occupancy"):
            d[k] = list(d[k])
        return d


# ---------------------------------------------------------------------------
# numpy-exact host arithmetic on the few values the GPU returns
# ---------------------------------------------------------------------------
QUANTILES = (0.5, 0.95, 0.99)


def _quantile_ranks(n: int, q: float) -> tuple[int, int, float]:
    """np.quantile(method='linear') neighbours and gamma (numpy _quantile)."""
    vi = (n - 1) * np.float64(q)
    prev = math.floor(vi)
    nxt = prev + 1
    if vi >= n - 1:
        prev = nxt = n - 1
        gamma = float(vi - (-1))  # numpy uses index -1 here; a == b so gamma is irrelevant
    elif vi < 0:
        prev = nxt = 0
        gamma = float(vi - 0)
    else:
        gamma = float(vi - prev)
    return prev, nxt, gamma


def _lerp(a: float, b: float, t: float) -> float:
    """numpy _lerp: a + (b-a)*t, or b - (b-a)*(1-t) when t >= 0.5."""
    d = b - a
    return b - d * (1 - t) if t >= 0.5 else a + d * t


def _naive_sum(values) -> float:
    """Left-to-right float sum from 0.0 (builtin sum() over np.float64s);
    np.add.accumulate is sequential, so its last element is that sum."""
    x = np.asarray(values, dtype=np.float64)
    return float(np.add.accumulate(x)[-1]) if x.size else 0.0


def _nanmean(values) -> float:
    x = np.asarray(values, dtype=float)
    finite = x[~np.isnan(x)]
    return float(finite.mean()) if finite.size else math.nan


@functools.lru_cache(maxsize=64)
def _t975(df: int) -> float:
    from scipy import stats as _st

    return _st.t.ppf(0.975, df)


def _ci_half_width(values) -> float:
    """sim.py:383-388 (the t quantile per degrees of freedom is cached)."""
    x = np.asarray(values, dtype=float)
    if x.size < 2 or np.any(np.isnan(x)):
        return math.nan
    return float(_t975(x.size - 1) * x.std(ddof=1) / math.sqrt(x.size))


def _require_supported(cfg: SimConfig) -> None:
    """The fast batched path: JFFC over a Poisson stream without time horizon."""
    from .sim_ext import needs_ext

    if needs_ext(cfg):
        raise ValueError("run_sim_batch: batched sweeps cover jffc/Poisson configs; "
                         "use run_sim for other policies and workloads")


def _rows_nanmean(x: np.ndarray) -> np.ndarray:
    """_nanmean of every row of a [P, R] array (row means are numpy's pairwise
    sums of the contiguous rows, as for the 1-D finite copy)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    nan = np.isnan(x)
    out = x.mean(axis=1) if x.shape[1] else np.full(x.shape[0], math.nan)
    for p in np.flatnonzero(nan.any(axis=1)):
        out[p] = _nanmean(x[p])
    return out


def _rows_ci_half_width(x: np.ndarray) -> np.ndarray:
    """_ci_half_width of every row (x.std(ddof=1) reduces each contiguous row
    exactly as the 1-D call does)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    P, R = x.shape
    if R < 2:
        return np.full(P, math.nan)
    out = _t975(R - 1) * x.std(axis=1, ddof=1) / math.sqrt(R)
    out[np.isnan(x).any(axis=1)] = math.nan
    return out


def _stats_from(cfg: SimConfig, summ: np.ndarray, busy: np.ndarray, order_stats: dict,
                jobs: np.ndarray | None) -> SimStats:
    """sim.py:406-456 on one point's per-replication summaries."""
    return _stats_from_batch([cfg], summ[None], busy[None], [order_stats],
                             None if jobs is None else jobs[None])[0]


def _stats_from_batch(configs: Sequence[SimConfig], summ: np.ndarray, busy: np.ndarray,
                      order_stats: Sequence[dict], jobs: np.ndarray | None) -> list[SimStats]:
    """sim.py:406-456 for P points at once ([P, R] summaries, [P, R, ldb] busy
    times): the per-point reductions run row-wise over contiguous copies of
    the summary fields, each row reduced exactly as the reference reduces
    that point's list (no response re-reads on host)."""
    R = configs[0].replications
    summ = summ[:, :R]
    # every field is 8 bytes: one transposing copy gives each field as a
    # contiguous [P, R] array
    # (blocked: a plain strided transpose of the 128-byte records is ~3x slower)
    names = summ.dtype.names
    rec = np.ascontiguousarray(summ).view(np.float64).reshape(-1, len(names))
    planes = np.empty((len(names), rec.shape[0]), np.float64)
    for i in range(0, rec.shape[0], 1024):
        planes[:, i:i + 1024] = rec[i:i + 1024].T
    planes = planes.reshape((len(names),) + summ.shape)
    col = {f: planes[i].view(summ.dtype[f]) for i, f in enumerate(names)}
    if np.any(col["counted"] < 0):  # jffc_sim_k1_kernel merge-feed overflow (never seen)
        raise AssertionError("simulation merge feed overflowed (exact finish-time ties)")
    counted = col["counted"].sum(axis=1)
    rep_means = col["resp_mean"].tolist()
    rep_occ = col["mean_occupancy"].tolist()
    resp_sums = col["resp_sum"].tolist()
    # sim.py:410-411 sums np.float64 values, so builtin sum() is the naive
    # left-to-right sum there (CPython compensates exact floats only);
    # np.add.accumulate runs left to right along each row
    total_wait = np.add.accumulate(col["wait_sum"], axis=1)[:, -1] if R else np.zeros(len(configs))
    total_service = np.add.accumulate(col["service_sum"], axis=1)[:, -1] if R else np.zeros(len(configs))
    mean_occ = _rows_nanmean(col["mean_occupancy"])
    lam_eff = _rows_nanmean(col["lambda_effective"])
    occ_h1 = _rows_nanmean(col["occ_first_half"])
    occ_h2 = _rows_nanmean(col["occ_second_half"])
    resp_ci = _rows_ci_half_width(col["resp_mean"])
    occ_ci = _rows_ci_half_width(col["mean_occupancy"])
    # per-chain utilisation: busy / (c_k * window) where window > 0, row nanmeans
    windows = col["window_s"]
    K = max(len(c.capacities) for c in configs)
    caps_pk = np.ones((len(configs), K), np.float64)
    for p, c in enumerate(configs):
        caps_pk[p, :len(c.capacities)] = c.capacities
    with np.errstate(divide="ignore", invalid="ignore"):  # same IEEE ops, element-wise
        ratio = np.where(windows[:, None, :] > 0,
                         np.asarray(busy[:, :R, :K], np.float64).transpose(0, 2, 1)
                         / (caps_pk[:, :, None] * windows[:, None, :]), math.nan)
    util_all = _rows_nanmean(ratio.reshape(-1, R)).reshape(len(configs), K)
    end_q = col["end_queue_len"].max(axis=1) if R else np.zeros(len(configs), np.int64)
    out = []
    for p, cfg in enumerate(configs):
        n_counted = int(counted[p])
        # merged.mean(): correctly rounded sum of the per-rep pairwise sums
        mean_resp = math.fsum(resp_sums[p]) / n_counted
        util = tuple(float(v) for v in util_all[p, :len(cfg.capacities)])
        mo, le = float(mean_occ[p]), float(lam_eff[p])
        little = (abs(mo - le * mean_resp) / mo if mo and not math.isnan(mo) else math.nan)
        qv = {}
        for q in QUANTILES:
            prev, nxt, gamma = _quantile_ranks(n_counted, q)
            qv[q] = _lerp(order_stats[p][prev], order_stats[p][nxt], gamma)
        records = None
        if cfg.collect_jobs and jobs is not None:
            records = tuple((r, float(a), float(s), float(f), int(k))
                            for r in range(R) for a, s, f, k in jobs[p][r])
        # sim.py:442,452: offered load is the Poisson rate, else the measured one
        offered = cfg.workload.rate if isinstance(cfg.workload, PoissonWorkload) or (
            hasattr(cfg.workload, "rate") and not hasattr(cfg.workload, "sizes")) else le
        unstable = bool(offered >= cfg.total_rate) if not math.isnan(offered) else False
        out.append(SimStats(
            policy=cfg.policy, jobs_counted=n_counted, mean_response_s=mean_resp,
            median_response_s=qv[0.5], p95_response_s=qv[0.95], p99_response_s=qv[0.99],
            mean_waiting_s=float(total_wait[p]) / n_counted,
            mean_service_s=float(total_service[p]) / n_counted,
            mean_occupancy=mo, response_ci_half_width_s=float(resp_ci[p]),
            occupancy_ci_half_width=float(occ_ci[p]), per_chain_utilization=util,
            lambda_effective=le, little_law_gap=little,
            unstable=unstable, seed=cfg.seed, replications=R,
            rep_mean_response_s=tuple(rep_means[p]), rep_mean_occupancy=tuple(rep_occ[p]),
            occ_first_half=float(occ_h1[p]), occ_second_half=float(occ_h2[p]),
            end_queue_len=int(end_q[p]), job_records=records))
    return out


@dataclass
class SweepResult:
    """Raw device outputs of one batched sweep (point-major rows)."""

    summaries: np.ndarray      # [P, R] SUMMARY_DTYPE
    busy: np.ndarray           # [P, R, ldb]
    order_stats: list[dict]    # per point: rank -> value
    jobs: np.ndarray | None    # [P, R, n, 4]
    responses: np.ndarray | None = None  # [P, R, n - warm] (completion order)


def simulate_sweep(rates_list: Sequence[Sequence[float]], caps_list: Sequence[Sequence[int]],
                   lams: Sequence[float], n_jobs: int, warmup_fraction: float, seed: int,
                   replications: int, rep_begin: int = 0, collect_jobs: bool = False,
                   order_stats: bool = True, max_stream_bytes: int = 8 << 30,
                   log1p_variant: int = -1, total_replications: int | None = None,
                   return_responses: bool = False) -> SweepResult:
    """One GPU call for P points x R replications (all points share the streams
    of replications rep_begin..rep_begin+R-1 of `seed`)."""
    lib = N.load()
    P = len(lams)
    R = replications
    warm = int(warmup_fraction * n_jobs)
    m = n_jobs - warm
    pts = (N.SimPoint * P)()
    rates, caps = [], []
    for p in range(P):
        pts[p] = N.SimPoint(len(rates_list[p]), len(rates), float(lams[p]))
        rates.extend(float(x) for x in rates_list[p])
        caps.extend(int(x) for x in caps_list[p])
    rates_a = np.asarray(rates, np.float64)
    caps_a = np.asarray(caps, np.int32)
    ldb = max(len(r) for r in rates_list)
    # order statistics needed by np.quantile over the merged responses of each point
    N_total = (total_replications or R) * m
    rank_list = sorted({r for q in QUANTILES for r in _quantile_ranks(N_total, q)[:2]})
    n_ranks = len(rank_list) if order_stats else 0
    ranks = np.asarray([rank_list] * P, np.int64).ravel() if order_stats else np.zeros(1, np.int64)
    out_vals = np.zeros(max(P * n_ranks, 1), np.float64)
    summ = np.zeros(P * R, N.SUMMARY_DTYPE)
    busy = np.zeros(P * R * ldb, np.float64)
    jobs = np.zeros(P * R * n_jobs * 4, np.float64) if collect_jobs else None
    resp = np.zeros(P * R * m, np.float64) if return_responses else None
    ent = N.seed_words(seed)
    st = lib.cs_run_sim_host(
        pts, P, N.ptr(rates_a, C.c_double), N.ptr(caps_a, C.c_int32), len(rates), N.ptr(ent, C.c_uint32),
        len(ent), rep_begin, R, n_jobs, warm, N.ptr(ranks, C.c_int64) if order_stats else None,
        n_ranks, log1p_variant, max_stream_bytes, summ.ctypes.data, N.ptr(busy, C.c_double), ldb,
        N.ptr(out_vals, C.c_double), N.ptr(resp, C.c_double) if resp is not None else None,
        N.ptr(jobs, C.c_double) if jobs is not None else None, None)
    N.check(st, "cs_run_sim_host")
    os_list = [{rank_list[i]: float(out_vals[p * n_ranks + i]) for i in range(n_ranks)}
               for p in range(P)]
    return SweepResult(summ.reshape(P, R), busy.reshape(P, R, ldb), os_list,
                       jobs.reshape(P, R, n_jobs, 4) if jobs is not None else None,
                       resp.reshape(P, R, m) if resp is not None else None)


def release_memory() -> None:
    """Return the engine's reserved device scratch (kept across calls: the
    host-buffer path re-uses it instead of re-mapping tens of GB per call)."""
    N.check(N.load().cs_release_memory(), "cs_release_memory")


def run_sim_batch(configs: Sequence[SimConfig]) -> list[SimStats]:
    """Batched run_sim: configs that differ only in rates/capacities/arrival
    rate share one GPU call (and their common random number streams)."""
    if not configs:
        return []
    c0 = configs[0]
    for c in configs:
        _require_supported(c)
        if (c.horizon_jobs, c.warmup_fraction, c.seed, c.replications, c.collect_jobs) != \
                (c0.horizon_jobs, c0.warmup_fraction, c0.seed, c0.replications, c0.collect_jobs):
            raise ValueError("run_sim_batch: configs must share horizon, warmup, seed, "
                             "replications and collect_jobs")
    res = simulate_sweep([c.rates for c in configs], [c.capacities for c in configs],
                         [c.workload.rate for c in configs], c0.horizon_jobs, c0.warmup_fraction,
                         c0.seed, c0.replications, collect_jobs=c0.collect_jobs)
    return _stats_from_batch(configs, res.summaries, res.busy, res.order_stats, res.jobs)


def run_sim(config: SimConfig) -> SimStats:
    """All replications on the GPU, aggregated exactly as sim.py:397-456.

    ``workers`` is accepted for signature parity; parallelism is the GPU's.
    """
    from .sim_ext import needs_ext, simulate_ext

    if needs_ext(config):
        summ, busy, os_, jobs, _ = simulate_ext(config)
        return _stats_from(config, summ, busy, os_, jobs)
    return run_sim_batch([config])[0]
