"""The rest of run_sim's signature on the GPU.

``simulate_ext(config)`` runs every replication of a ``SimConfig`` that the
fast JFFC/Poisson path does not cover -- dedicated-queue policies
(jsq / sa-jsq / jiq / sed, chainserve sim.py:104-117,279-286), sampled and
trace workloads (sim.py:161-178,199-203; workload.py:150-164) and the
time-horizon Poisson mode (sim.py:146-158,187-190) -- through ``cs_sim_ext``
(csrc/sim_ext.cu), then the same device statistics pass.  ``sim.run_sim``
dispatches here; results are bit-exact with the reference's _simulate_once.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from .model import GB, TAIL_ID

POLICY_CODE = {"jffc": 0, "jsq": 1, "sa-jsq": 2, "jiq": 3, "sed": 4}
WL_POISSON, WL_HORIZON, WL_SAMPLED, WL_TRACE = range(4)
HBLK = 4096
REP_QUEUE_OVERFLOW, REP_EMPTY_HORIZON, REP_WARMUP_ALL = 16, 17, 18
STREAM_PAD = 512


class ExtArgs(C.Structure):
    """cs_sim_ext_args (include/chainserve_b200.h)."""

    _fields_ = [
        ("points", C.c_void_p), ("n_points", C.c_int32), ("policy", C.c_int32),
        ("workload", C.c_int32), ("max_chains", C.c_int32), ("max_capacity", C.c_int32),
        ("rates", C.c_void_p), ("caps", C.c_void_p), ("streams", C.c_void_p), ("lds", C.c_int64),
        ("horizon_time_s", C.c_double), ("warmup_cut_s", C.c_double),
        ("arrivals", C.c_void_p), ("sizes", C.c_void_p), ("tokens_in", C.c_void_p),
        ("tokens_out", C.c_void_p), ("hop_begin", C.c_void_p), ("hop_server", C.c_void_p),
        ("hop_blocks", C.c_void_p), ("server_param", C.c_void_p),
        ("rep_begin", C.c_int32), ("n_reps", C.c_int32), ("n_reps_total", C.c_int32),
        ("n_jobs", C.c_int64), ("warm", C.c_int64),
        ("responses", C.c_void_p), ("ldr", C.c_int64), ("busy", C.c_void_p), ("ldb", C.c_int32),
        ("summary", C.c_void_p), ("jobs", C.c_void_p), ("rep_jobs", C.c_void_p),
        ("rep_status", C.c_void_p), ("queue_workspace", C.c_void_p), ("queue_capacity", C.c_int32),
    ]


def workload_kind(cfg) -> int:
    wl = cfg.workload
    if hasattr(wl, "records"):
        return WL_TRACE
    if hasattr(wl, "sizes") and hasattr(wl, "arrivals_s"):
        return WL_SAMPLED
    return WL_HORIZON if cfg.horizon_time_s is not None else WL_POISSON


def needs_ext(cfg) -> bool:
    return cfg.policy != "jffc" or workload_kind(cfg) != WL_POISSON


def _trace_tables(cfg):
    """Per-chain hop lists and per-server constants of
    ServiceTimeModel.request_service_time (workload.py:150-164): the
    per-server values are formed with the reference's own expressions
    (derive_tau_c / derive_tau_p, workload.py:39-60,108-120)."""
    model = cfg.service_model
    sid_index: dict[str, int] = {}
    params: list[float] = []
    hop_begin, hop_srv, hop_m = [0], [], []
    for chain in cfg.chains:
        for e in chain.edges:
            if e.dst == TAIL_ID:
                continue
            if e.dst not in sid_index:
                prof = model.profiles[e.dst]
                per_token_ms = model.rtt.rtt_ms(model.orchestrator, e.dst) + model.rtt.overhead_ms
                prefill_ms = prof.per_block_flops_gflop / prof.flops_tflops
                decode_ms = (model.service.block_bytes / GB) / prof.mem_bandwidth_gb_per_ms
                sid_index[e.dst] = len(sid_index)
                params += [per_token_ms, prof.per_block_overhead_ms, prefill_ms, decode_ms]
            hop_srv.append(sid_index[e.dst])
            hop_m.append(int(e.blocks_at_dst))
        hop_begin.append(len(hop_srv))
    return (np.asarray(hop_begin, np.int32), np.asarray(hop_srv or [0], np.int32),
            np.asarray(hop_m or [0], np.int32), np.asarray(params or [0.0], np.float64))


def _workload_arrays(cfg, kind):
    """_materialize for the sampled / trace workloads (sim.py:161-178)."""
    n, t_end = cfg.horizon_jobs, cfg.horizon_time_s
    if kind == WL_SAMPLED:
        arr = np.asarray(cfg.workload.arrivals_s, dtype=float)
        sz = np.asarray(cfg.workload.sizes, dtype=float)
        if t_end is not None:
            keep = arr <= t_end
            arr, sz = arr[keep], sz[keep]
        arr, sz = arr[:n], sz[:n]
        if arr.size == 0:
            raise ValueError("sampled workload is empty")
        return arr, sz, None, None
    recs = [r for r in cfg.workload.records if t_end is None or r.arrival_s <= t_end][:n]
    if not recs:
        raise ValueError("trace workload is empty")
    arr = np.asarray([r.arrival_s for r in recs], dtype=float)
    tin = np.asarray([r.input_tokens for r in recs], dtype=np.int64)
    tout = np.asarray([r.output_tokens for r in recs], dtype=np.int64)
    if np.any(tin <= 0) or np.any(tout <= 0):
        raise ValueError("token counts must be positive")
    return arr, None, tin.astype(np.int32), tout.astype(np.int32)


def simulate_ext(cfg, return_responses: bool = False, queue_capacity: int = 1024):
    """All replications of `cfg` on the GPU.  Returns (summaries[R],
    busy[R, K], order_stats {rank: value}, job records per rep or None,
    responses per rep or None)."""
    from .sim import QUANTILES, _quantile_ranks

    lib = N.load()
    import torch

    dev = torch.device("cuda")
    stream = torch.cuda.current_stream()
    kind = workload_kind(cfg)
    K, R = len(cfg.rates), cfg.replications
    policy = POLICY_CODE[cfg.policy]
    d = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    keep = []  # device buffers referenced by the args struct

    a = ExtArgs()
    a.policy, a.workload = policy, kind
    a.max_chains, a.max_capacity = K, int(sum(cfg.capacities))
    lam = float(cfg.workload.rate) if kind in (WL_POISSON, WL_HORIZON) else 1.0
    pt = N.SimPoint(K, 0, lam)
    for name, arr, dt in (("points", np.frombuffer(pt, np.uint8), torch.uint8),
                          ("rates", np.asarray(cfg.rates, np.float64), torch.float64),
                          ("caps", np.asarray(cfg.capacities, np.int32), torch.int32)):
        t = d(arr, dt)
        keep.append(t)
        setattr(a, name, t.data_ptr())
    a.n_points = 1
    n = cfg.horizon_jobs
    warm = int(cfg.warmup_fraction * n)
    if kind in (WL_SAMPLED, WL_TRACE):
        arr, sz, tin, tout = _workload_arrays(cfg, kind)
        n = int(arr.size)
        if cfg.horizon_time_s is None:
            warm = int(cfg.warmup_fraction * n)
        else:
            warm = int(np.searchsorted(arr, cfg.warmup_fraction * cfg.horizon_time_s, side="left"))
            if warm >= n:
                raise ValueError("warmup consumed every arrival in the time horizon")
        t = d(arr, torch.float64)
        keep.append(t)
        a.arrivals = t.data_ptr()
        if kind == WL_SAMPLED:
            t = d(sz, torch.float64)
            keep.append(t)
            a.sizes = t.data_ptr()
        else:
            hb, hs, hm, sp = _trace_tables(cfg)
            for name, arr_, dt in (("tokens_in", tin, torch.int32), ("tokens_out", tout, torch.int32),
                                   ("hop_begin", hb, torch.int32), ("hop_server", hs, torch.int32),
                                   ("hop_blocks", hm, torch.int32), ("server_param", sp, torch.float64)):
                t = d(arr_, dt)
                keep.append(t)
                setattr(a, name, t.data_ptr())
    else:
        # exponential streams of replications 0..R-1 (sim.py:141-145)
        L = 2 * n if kind == WL_POISSON else HBLK * (-(-n // HBLK)) + n
        w = N.seed_words(cfg.seed)
        reps = np.arange(R, dtype=np.uint64)
        keys = np.zeros((R, 2), np.uint64)
        N.check(lib.cs_philox_keys(N.ptr(w, C.c_uint32), len(w), N.ptr(reps, C.c_uint64), R,
                                   N.ptr(keys, C.c_uint64)), "cs_philox_keys")
        d_keys = d(keys.view(np.int64), torch.int64)
        d_S = torch.empty(R * L + STREAM_PAD, dtype=torch.float64, device=dev)
        keep += [d_keys, d_S]
        N.check(lib.cs_exp_streams(d_keys.data_ptr(), R, L, d_S.data_ptr(), L,
                                   lib.cs_host_log1p_variant(), stream.cuda_stream), "cs_exp_streams")
        a.streams, a.lds = d_S.data_ptr(), L
        if kind == WL_HORIZON:
            a.horizon_time_s = float(cfg.horizon_time_s)
            a.warmup_cut_s = cfg.warmup_fraction * cfg.horizon_time_s
    a.rep_begin, a.n_reps, a.n_reps_total = 0, R, R
    a.n_jobs, a.warm = n, warm
    ldr = n if kind == WL_HORIZON else n - warm
    d_resp = torch.empty(max(R * ldr, 1), dtype=torch.float64, device=dev)
    d_busy = torch.zeros(R * K, dtype=torch.float64, device=dev)
    d_summ = torch.zeros(R * C.sizeof(N.RepSummary), dtype=torch.uint8, device=dev)
    d_jobs = torch.zeros(R * n * 4, dtype=torch.float64, device=dev) if cfg.collect_jobs else None
    d_rjobs = torch.zeros(R, dtype=torch.int64, device=dev)
    d_rst = torch.zeros(R, dtype=torch.int32, device=dev)
    a.responses, a.ldr, a.busy, a.ldb = d_resp.data_ptr(), ldr, d_busy.data_ptr(), K
    a.summary, a.rep_jobs, a.rep_status = d_summ.data_ptr(), d_rjobs.data_ptr(), d_rst.data_ptr()
    a.jobs = d_jobs.data_ptr() if d_jobs is not None else None
    q = 1
    while q < min(queue_capacity, n):
        q *= 2
    qmax = 1
    while qmax < n:
        qmax *= 2
    while True:
        d_q = None
        if policy != 0:
            d_q = torch.empty(R * K * q * 16, dtype=torch.uint8, device=dev)
            a.queue_workspace, a.queue_capacity = d_q.data_ptr(), q
        N.check(lib.cs_sim_ext(C.byref(a), stream.cuda_stream), "cs_sim_ext")
        rst = d_rst.cpu().numpy()
        if policy != 0 and np.any(rst == REP_QUEUE_OVERFLOW) and q < qmax:
            q = min(q * 8, qmax)  # a dedicated queue outgrew its ring: rerun with room
            continue
        break
    if np.any(rst == REP_EMPTY_HORIZON):
        raise ValueError("no arrivals fall inside the time horizon")
    if np.any(rst == REP_WARMUP_ALL):
        raise ValueError("warmup consumed every arrival in the time horizon")
    if np.any(rst != 0):
        raise AssertionError(f"cs_sim_ext: replication status {sorted(set(rst.tolist()))}")

    summ = d_summ.cpu().numpy().view(N.SUMMARY_DTYPE).copy()
    counts = summ["counted"].astype(np.int64)
    N_total = int(counts.sum())
    rank_list = sorted({r for qq in QUANTILES for r in _quantile_ranks(N_total, qq)[:2]})
    ranks = np.asarray(rank_list, np.int64)
    out_vals = np.zeros(len(rank_list), np.float64)
    sums = None
    if kind == WL_HORIZON:  # ragged rows: pairwise sums here, +inf padding for the select
        d_counts = d(counts, torch.int64)
        d_sums = torch.empty(R, dtype=torch.float64, device=dev)
        N.check(lib.cs_ragged_rows(d_resp.data_ptr(), R, ldr, d_counts.data_ptr(), d_sums.data_ptr(),
                                   stream.cuda_stream), "cs_ragged_rows")
        sums = d_sums.cpu().numpy()
    m = ldr
    if N_total > 0:
        N.check(lib.cs_rep_stats(d_resp.data_ptr(), 1, R, m, ldr, d_summ.data_ptr(),
                                 N.ptr(ranks, C.c_int64), len(rank_list),
                                 N.ptr(out_vals, C.c_double), None, stream.cuda_stream), "cs_rep_stats")
    summ = d_summ.cpu().numpy().view(N.SUMMARY_DTYPE).copy()
    if sums is not None:
        summ["resp_sum"] = sums
        with np.errstate(invalid="ignore", divide="ignore"):
            summ["resp_mean"] = sums / counts
    busy = d_busy.cpu().numpy().reshape(R, K)
    order_stats = {rank_list[i]: float(out_vals[i]) for i in range(len(rank_list))}
    n_rep = d_rjobs.cpu().numpy()
    jobs = None
    if d_jobs is not None:
        jh = d_jobs.cpu().numpy().reshape(R, n, 4)
        jobs = [jh[r, :int(n_rep[r])] for r in range(R)]
    resp = None
    if return_responses:
        rh = d_resp.cpu().numpy().reshape(R, ldr)
        resp = [rh[r, :int(counts[r])].copy() for r in range(R)]
    return summ, busy, order_stats, jobs, resp
