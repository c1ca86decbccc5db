"""ctypes front-end of the CPU oracle.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this module, and only as the checker or the
timed CPU baseline.  The product package never imports it.

Each wrapper names the reference code it restates (paths relative to
/root/reference/pkg/src/chainserve).  ``run_sim_stats`` restates the
aggregation of sim.py:397-456 in numpy on top of ``orc_simulate_reps``.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle_cs.so")

OK, INFEASIBLE, INVALID, INTERNAL = 0, 1, 2, 3


class RepSummary(C.Structure):
    _fields_ = [
        ("wait_sum", C.c_double), ("service_sum", C.c_double), ("counted", C.c_int64),
        ("window_s", C.c_double), ("mean_occupancy", C.c_double),
        ("occ_first_half", C.c_double), ("occ_second_half", C.c_double),
        ("lambda_effective", C.c_double), ("end_queue_len", C.c_int64),
        ("w_start", C.c_double), ("t_mid", C.c_double), ("area_mid", C.c_double),
        ("t_end", C.c_double), ("area_end", C.c_double),
    ]


def build() -> str:
    """Compile the oracle with its Makefile (gcc is present on both boxes)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.orc_philox_key.argtypes = [C.c_uint64, C.c_uint64, P(C.c_uint64)]
        L.orc_seedseq_key.argtypes = [P(C.c_uint32), C.c_int, P(C.c_uint32), C.c_int, P(C.c_uint64)]
        L.orc_philox_raw.argtypes = [P(C.c_uint64), C.c_int64, P(C.c_uint64)]
        L.orc_standard_exponential.argtypes = [P(C.c_uint64), C.c_int64, P(C.c_double)]
        L.orc_standard_exponential.restype = C.c_int64
        L.orc_simulate_once.argtypes = [
            C.c_int, P(C.c_double), P(C.c_int32), C.c_double, C.c_int64, C.c_double,
            C.c_uint64, C.c_uint64, P(C.c_double), P(C.c_double), P(C.c_double), P(RepSummary)]
        L.orc_simulate_reps.argtypes = [
            C.c_int, P(C.c_double), P(C.c_int32), C.c_double, C.c_int64, C.c_double,
            C.c_uint64, C.c_int64, C.c_int64, C.c_int, P(C.c_double), P(C.c_double),
            P(RepSummary)]
        L.orc_gbp.argtypes = [
            C.c_int, P(C.c_int64), P(C.c_double), P(C.c_double), P(C.c_int32), C.c_int64,
            C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, P(C.c_int32),
            P(C.c_int32), P(C.c_int32), P(C.c_double), P(C.c_int32), P(C.c_int32),
            P(C.c_int32), P(C.c_double), P(C.c_int32)]
        L.orc_gca.argtypes = [
            C.c_int, P(C.c_int64), P(C.c_double), P(C.c_double), P(C.c_int32), C.c_int64,
            C.c_int64, C.c_int64, P(C.c_int32), P(C.c_int32), P(C.c_int64), C.c_int32,
            C.c_int32, P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_double),
            P(C.c_int32), P(C.c_int64)]
        L.orc_simulate_ext.argtypes = [
            C.c_int, P(C.c_double), P(C.c_int32), C.c_int, C.c_int64, C.c_int64, P(C.c_double),
            P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double),
            P(RepSummary)]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


# ---- RNG ------------------------------------------------------------------

def philox_key(seed: int, rep: int) -> np.ndarray:
    """SeedSequence(entropy=seed, spawn_key=(rep,)) -> Philox key (sim.py:141-143)."""
    out = np.zeros(2, np.uint64)
    lib().orc_philox_key(seed, rep, _p(out, C.c_uint64))
    return out


def philox_raw(key, n: int) -> np.ndarray:
    key = np.ascontiguousarray(key, np.uint64)
    out = np.empty(n, np.uint64)
    lib().orc_philox_raw(_p(key, C.c_uint64), n, _p(out, C.c_uint64))
    return out


def standard_exponential(key, n: int):
    """Generator(Philox(key)).exponential(1.0, n) and the words it consumed."""
    key = np.ascontiguousarray(key, np.uint64)
    out = np.empty(n, np.float64)
    words = lib().orc_standard_exponential(_p(key, C.c_uint64), n, _p(out, C.c_double))
    return out, int(words)


# ---- simulator --------------------------------------------------------------

def simulate_once(rates, caps, lam, n, warmup_fraction, seed, rep, collect_jobs=False):
    """sim.py:_simulate_once (Poisson, jffc).  Returns a dict of RepResult fields."""
    rates = np.ascontiguousarray(rates, np.float64)
    caps = np.ascontiguousarray(caps, np.int32)
    K = len(rates)
    warm = int(warmup_fraction * n)
    resp = np.empty(max(n - warm, 1), np.float64)
    busy = np.empty(K, np.float64)
    jobs = np.empty((n, 4), np.float64) if collect_jobs else None
    s = RepSummary()
    st = lib().orc_simulate_once(
        K, _p(rates, C.c_double), _p(caps, C.c_int32), lam, n, warmup_fraction, seed, rep,
        _p(resp, C.c_double), _p(busy, C.c_double),
        _p(jobs, C.c_double) if jobs is not None else None, C.byref(s))
    if st != OK:
        raise RuntimeError(f"oracle simulate_once status {st}")
    out = {f: getattr(s, f) for f, _ in RepSummary._fields_}
    out["responses"] = resp[: s.counted].copy()
    out["busy_time_s"] = busy
    out["jobs"] = jobs
    return out


POLICY_CODE = {"jffc": 0, "jsq": 1, "sa-jsq": 2, "jiq": 3, "sed": 4}
HBLK = 4096


def poisson_inputs(lam, n, seed, rep, horizon=None):
    """_materialize, Poisson branch (sim.py:136-160): (arrivals, sizes).
    Without a horizon: cumsum(exponential(1/lam, n)); with one: 4096-draw
    blocks cumsum(block) + total while total < t_end and fewer than n drawn,
    then arrivals <= t_end, at most n; sizes drawn after every block."""
    key = philox_key(seed, rep)
    scale = 1.0 / lam
    if horizon is None:
        S, _ = standard_exponential(key, 2 * n)
        return np.cumsum(scale * S[:n]), 1.0 * S[n:]
    S, _ = standard_exponential(key, HBLK * (-(-n // HBLK)) + n)
    chunks, total, count, pos = [], 0.0, 0, 0
    while total < horizon and count < n:
        block = np.cumsum(scale * S[pos:pos + HBLK]) + total
        pos += HBLK
        chunks.append(block)
        total = block[-1]
        count += block.size
    arrivals = np.concatenate(chunks)
    arrivals = arrivals[arrivals <= horizon][:n]
    return arrivals, 1.0 * S[pos:pos + arrivals.size]


def trace_durations(tin, tout, chains_hops, server_params):
    """ServiceTimeModel.request_service_time (workload.py:150-164) for every
    (job, chain): chains_hops[k] = [(server, blocks_at_dst), ...] (tail hop
    excluded); server_params[s] = (rtt+overhead ms, block overhead ms,
    prefill ms, decode ms).  Returns an [n, K] array."""
    tin = np.asarray(tin, np.float64)
    tout_i = np.asarray(tout, np.int64)
    tout = tout_i.astype(np.float64)
    out = np.empty((tin.size, len(chains_hops)))
    for k, hops in enumerate(chains_hops):
        total = np.zeros(tin.size)
        for s, m in hops:
            ptm, ovh, pre, dec = server_params[s]
            total = total + tout * ptm / 1000.0
            total = total + ((ovh + pre * tin) + dec * (tout_i - 1).astype(np.float64)) / 1000.0 * m
        out[:, k] = total
    return out


def simulate_ext(rates, caps, policy, arrivals, warm, sizes=None, durations=None,
                 collect_jobs=False):
    """sim.py:_simulate_once on explicit inputs, any policy.  Returns a dict
    of RepResult fields (as simulate_once)."""
    rates = np.ascontiguousarray(rates, np.float64)
    caps = np.ascontiguousarray(caps, np.int32)
    arr = np.ascontiguousarray(arrivals, np.float64)
    K, n = len(rates), arr.size
    sz = None if sizes is None else np.ascontiguousarray(sizes, np.float64)
    dur = None if durations is None else np.ascontiguousarray(durations, np.float64)
    resp = np.empty(max(n - warm, 1), np.float64)
    busy = np.empty(K, np.float64)
    jobs = np.empty((n, 4), np.float64) if collect_jobs else None
    s = RepSummary()
    st = lib().orc_simulate_ext(
        K, _p(rates, C.c_double), _p(caps, C.c_int32), POLICY_CODE[policy], n, warm,
        _p(arr, C.c_double), _p(sz, C.c_double) if sz is not None else None,
        _p(dur, C.c_double) if dur is not None else None, _p(resp, C.c_double),
        _p(busy, C.c_double), _p(jobs, C.c_double) if jobs is not None else None, C.byref(s))
    if st != OK:
        raise RuntimeError(f"oracle simulate_ext status {st}")
    out = {f: getattr(s, f) for f, _ in RepSummary._fields_}
    out["responses"] = resp[: s.counted].copy()
    out["busy_time_s"] = busy
    out["jobs"] = jobs
    return out


def simulate_reps(rates, caps, lam, n, warmup_fraction, seed, rep_begin, rep_end, threads=None):
    rates = np.ascontiguousarray(rates, np.float64)
    caps = np.ascontiguousarray(caps, np.int32)
    K = len(rates)
    R = rep_end - rep_begin
    warm = int(warmup_fraction * n)
    resp = np.empty((R, n - warm), np.float64)
    busy = np.empty((R, K), np.float64)
    summ = (RepSummary * R)()
    threads = threads or os.cpu_count() or 1
    st = lib().orc_simulate_reps(
        K, _p(rates, C.c_double), _p(caps, C.c_int32), lam, n, warmup_fraction, seed,
        rep_begin, rep_end, threads, _p(resp, C.c_double), _p(busy, C.c_double), summ)
    if st != OK:
        raise RuntimeError(f"oracle simulate_reps status {st}")
    return resp, busy, summ


def _nanmean(values) -> float:
    x = np.asarray(values, dtype=float)
    finite = x[~np.isnan(x)]
    return float(finite.mean()) if finite.size else math.nan


def run_sim_stats(rates, caps, lam, n, warmup_fraction, seed, replications, threads=None):
    """numpy restatement of run_sim's aggregation (sim.py:397-456), jffc/Poisson."""
    from scipy import stats as sst

    resp, busy, summ = simulate_reps(rates, caps, lam, n, warmup_fraction, seed, 0,
                                     replications, threads)
    merged = np.sort(resp.ravel())
    rep_means = tuple(float(r.mean()) for r in resp)
    rep_occ = tuple(s.mean_occupancy for s in summ)
    counted = int(sum(s.counted for s in summ))
    # the reference's per-rep sums are np.float64, so builtin sum() takes the
    # generic (naive, left-to-right) path, not CPython's compensated float path
    total_wait = sum(np.float64(s.wait_sum) for s in summ)
    total_service = sum(np.float64(s.service_sum) for s in summ)
    mean_occ = _nanmean(rep_occ)
    lam_eff = _nanmean([s.lambda_effective for s in summ])
    mean_resp = float(merged.mean())
    util = tuple(
        _nanmean([busy[r, k] / (caps[k] * summ[r].window_s) if summ[r].window_s > 0 else math.nan
                  for r in range(replications)])
        for k in range(len(caps)))
    little = (abs(mean_occ - lam_eff * mean_resp) / mean_occ
              if mean_occ and not math.isnan(mean_occ) else math.nan)

    def ci(values):
        x = np.asarray(values, dtype=float)
        if x.size < 2 or np.any(np.isnan(x)):
            return math.nan
        return float(sst.t.ppf(0.975, x.size - 1) * x.std(ddof=1) / math.sqrt(x.size))

    total_rate = sum(r * c for r, c in zip(rates, caps))
    return dict(
        policy="jffc", jobs_counted=counted, mean_response_s=mean_resp,
        median_response_s=float(np.quantile(merged, 0.5)),
        p95_response_s=float(np.quantile(merged, 0.95)),
        p99_response_s=float(np.quantile(merged, 0.99)),
        mean_waiting_s=float(total_wait / counted), mean_service_s=float(total_service / counted),
        mean_occupancy=mean_occ, response_ci_half_width_s=ci(rep_means),
        occupancy_ci_half_width=ci(rep_occ), per_chain_utilization=util,
        lambda_effective=lam_eff, little_law_gap=little,
        unstable=bool(lam >= total_rate), seed=seed, replications=replications,
        rep_mean_response_s=rep_means, rep_mean_occupancy=rep_occ,
        occ_first_half=_nanmean([s.occ_first_half for s in summ]),
        occ_second_half=_nanmean([s.occ_second_half for s in summ]),
        end_queue_len=max(s.end_queue_len for s in summ))


# ---- composition --------------------------------------------------------------

def id_ranks(ids) -> np.ndarray:
    """Rank of each id in Python str order (placement.py:87-90, cache_alloc.py:34)."""
    order = sorted(range(len(ids)), key=lambda i: ids[i])
    rank = np.empty(len(ids), np.int32)
    for r, i in enumerate(order):
        rank[i] = r
    return rank


def gbp(mem, tau_c, tau_p, ids, L, s_m, s_c, capacity, arrival_rate, load_target):
    """greedy_block_placement (placement.py:67-132).  Returns (status, dict)."""
    J = len(mem)
    mem = np.ascontiguousarray(mem, np.int64)
    tc = np.ascontiguousarray(tau_c, np.float64)
    tp = np.ascontiguousarray(tau_p, np.float64)
    rk = id_ranks(ids)
    first = np.zeros(J, np.int32)
    count = np.zeros(J, np.int32)
    mb = np.zeros(J, np.int32)
    bt = np.zeros(J, np.float64)
    members = np.zeros(max(J, 1), np.int32)
    offs = np.zeros(J + 1, np.int32)
    nch = C.c_int32()
    rate = C.c_double()
    sat = C.c_int32()
    st = lib().orc_gbp(J, _p(mem, C.c_int64), _p(tc, C.c_double), _p(tp, C.c_double),
                       _p(rk, C.c_int32), L, s_m, s_c, capacity, arrival_rate, load_target,
                       _p(first, C.c_int32), _p(count, C.c_int32), _p(mb, C.c_int32),
                       _p(bt, C.c_double), _p(members, C.c_int32), _p(offs, C.c_int32),
                       C.byref(nch), C.byref(rate), C.byref(sat))
    chains = [tuple(int(x) for x in members[offs[k]:offs[k + 1]]) for k in range(nch.value)]
    return st, dict(first=first, count=count, max_blocks=mb, bound_time=bt, chains=chains,
                    scaled_rate=rate.value, rate_satisfied=bool(sat.value))


def gca(mem, tau_c, tau_p, ids, L, s_m, s_c, first, count, residual=None):
    """greedy_cache_allocation (cache_alloc.py:65-135).  Returns (status, dict)."""
    J = len(mem)
    mem = np.ascontiguousarray(mem, np.int64)
    tc = np.ascontiguousarray(tau_c, np.float64)
    tp = np.ascontiguousarray(tau_p, np.float64)
    rk = id_ranks(ids)
    first = np.ascontiguousarray(first, np.int32)
    count = np.ascontiguousarray(count, np.int32)
    res = None if residual is None else np.ascontiguousarray(residual, np.int64)
    U = int((count > 0).sum())
    max_chains = max(U * (U + 2) + 4, 16)
    max_members = max_chains * (min(U, int(L)) + 1)
    members = np.zeros(max_members, np.int32)
    offs = np.zeros(max_chains + 1, np.int32)
    caps = np.zeros(max_chains, np.int32)
    times = np.zeros(max_chains, np.float64)
    nch = C.c_int32()
    ne = C.c_int64()
    st = lib().orc_gca(J, _p(mem, C.c_int64), _p(tc, C.c_double), _p(tp, C.c_double),
                       _p(rk, C.c_int32), L, s_m, s_c, _p(first, C.c_int32),
                       _p(count, C.c_int32), _p(res, C.c_int64) if res is not None else None,
                       max_chains, max_members, _p(members, C.c_int32), _p(offs, C.c_int32),
                       _p(caps, C.c_int32), _p(times, C.c_double), C.byref(nch), C.byref(ne))
    K = nch.value
    chains = [tuple(int(x) for x in members[offs[k]:offs[k + 1]]) for k in range(K)]
    return st, dict(chains=chains, caps=caps[:K].copy(), times=times[:K].copy(),
                    n_edges=ne.value)


# ---- occupancy bounds (analysis.py:67-147), numpy restatement -------------

def death_rates(rates, caps):
    """death_rate_bounds(rates, n) for n = 1..C (analysis.py:67-81): arrays
    (fast, slow) of the sequential per-chain float sums."""
    C_tot = int(sum(caps))
    fast = np.zeros(C_tot)
    slow = np.zeros(C_tot)
    for n in range(1, C_tot + 1):
        u = lo = 0.0
        ahead, behind = 0, C_tot
        for mu, c in zip(rates, caps):
            u += mu * min(c, max(n - ahead, 0))
            ahead += c
            behind -= c
            lo += mu * min(c, max(n - behind, 0))
        fast[n - 1], slow[n - 1] = u, lo
    return fast, slow


def _logsumexp(a):
    """scipy 1.18 special.logsumexp for a 1-D real array without weights:
    maximal terms split out, log1p(s/m) + log(m) + max."""
    a = np.asarray(a, np.float64)
    amax = a.max()
    is_max = a == amax
    m = float(is_max.sum())
    s = np.exp(np.where(is_max, -np.inf, a) - amax).sum()
    if s != 0:
        s = s / m
    return np.log1p(s) + np.log(m) + amax


def birth_death_mean_occupancy(lam, death, nu):
    """analysis.py:84-109 (caller checks lam < nu, death > 0)."""
    d = np.asarray(death, np.float64)
    C_tot = d.size
    rho = lam / nu
    log_w = np.concatenate(([0.0], np.cumsum(np.log(lam) - np.log(d))))
    tail = log_w[C_tot] + math.log(nu) - math.log(nu - lam)
    log_z = _logsumexp(np.concatenate((log_w[:C_tot], [tail])))
    n = np.arange(1, C_tot)
    head = float(np.sum(n * np.exp(log_w[1:C_tot] - log_z))) if C_tot > 1 else 0.0
    queued = math.exp(log_w[C_tot] - log_z) * (rho / (1 - rho) ** 2 + C_tot / (1 - rho))
    return head + queued


def occupancy_bounds(rates, caps, lam):
    """analysis.py:121-147 -> (lower_occ, upper_occ, lower_resp, upper_resp),
    or None when lam >= total rate (UnstableError in the reference)."""
    nu = sum(r * c for r, c in zip(rates, caps))
    if lam >= nu:
        return None
    fast, slow = death_rates(rates, caps)
    lo = birth_death_mean_occupancy(lam, fast, nu)
    hi = birth_death_mean_occupancy(lam, slow, nu)
    return lo, hi, lo / lam, hi / lam
