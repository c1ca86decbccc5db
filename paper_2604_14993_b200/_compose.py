"""Host driver of the batched composition kernels (compose.cu).

Packs instances into structure-of-arrays device buffers (torch CUDA tensors
are only the allocator here), launches cs_gbp_batch / cs_gca_batch through
the C-ABI and unpacks the results.  One call processes any number of
(instance, capacity, lambda, rho) points.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as N
from .model import ServerSpec, ServiceSpec


def id_ranks(ids: Sequence[str]) -> np.ndarray:
    """Rank of each id in Python string order (sorted by (float, str) at
    placement.py:87-90; node order at cache_alloc.py:31-37)."""
    order = sorted(range(len(ids)), key=ids.__getitem__)
    rank = np.empty(len(ids), np.int32)
    rank[order] = np.arange(len(ids), dtype=np.int32)
    return rank


@dataclass
class Fleet:
    """SoA image of one server list."""

    servers: tuple[ServerSpec, ...]
    mem: np.ndarray
    tau_c: np.ndarray
    tau_p: np.ndarray
    rank: np.ndarray

    @classmethod
    def of(cls, servers: Sequence[ServerSpec]) -> "Fleet":
        servers = tuple(servers)
        mem = np.array([s.memory_bytes for s in servers], dtype=np.int64) if servers else np.zeros(0, np.int64)
        return cls(servers, mem,
                   np.array([float(s.comm_time_s) for s in servers], dtype=np.float64),
                   np.array([float(s.per_block_compute_s) for s in servers], dtype=np.float64),
                   id_ranks([s.id for s in servers]))


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise N.NativeUnavailable("no CUDA device visible: the chainserve B200 engine has no CPU path")
    return torch


def _dev(torch, a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", non_blocking=False)


def _empty(torch, n, dtype):
    return torch.empty(max(int(n), 1), dtype=dtype, device="cuda")


@dataclass
class GbpOut:
    status: np.ndarray
    first: np.ndarray
    count: np.ndarray
    max_blocks: np.ndarray
    bound_time: np.ndarray
    order: np.ndarray
    chain_end: np.ndarray
    n_chains: np.ndarray
    scaled_rate: np.ndarray
    rate_satisfied: np.ndarray
    server_base: np.ndarray
    n_servers: np.ndarray


def _check_int64(name, v):
    if not -(2**63) <= v < 2**63:
        raise NotImplementedError(f"{name}={v} exceeds the engine's 64-bit integer range")


def gbp_batch(fleets: Sequence[Fleet], services: Sequence[ServiceSpec], capacities: Sequence[int],
              arrival_rates: Sequence[float], load_targets: Sequence[float],
              fleet_of_point: Sequence[int] | None = None) -> GbpOut:
    """greedy_block_placement for every point (fleet_of_point maps point -> fleet)."""
    lib = N.load()
    torch = _torch()
    P = len(capacities)
    if fleet_of_point is None:
        fleet_of_point = list(range(P))
    # every point gets its own copy of its fleet's SoA slice (outputs are per server)
    bases, sizes = [], []
    mem, tc, tp, rk = [], [], [], []
    off = 0
    for p in range(P):
        f = fleets[fleet_of_point[p]]
        bases.append(off)
        sizes.append(len(f.servers))
        mem.append(f.mem)
        tc.append(f.tau_c)
        tp.append(f.tau_p)
        rk.append(f.rank)
        off += len(f.servers)
    pts = (N.ComposePoint * max(P, 1))()
    for p in range(P):
        svc = services[p]
        per_block = svc.block_bytes + svc.cache_slot_bytes * int(capacities[p])
        _check_int64("s_m + s_c * c", per_block)
        pts[p] = N.ComposePoint(sizes[p], bases[p], svc.block_count, svc.block_bytes,
                                svc.cache_slot_bytes, int(capacities[p]), float(arrival_rates[p]),
                                float(load_targets[p]))
    S = max(off, 1)
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs and off else np.zeros(1, dt)
    d_mem, d_tc, d_tp, d_rk = (_dev(torch, cat(mem, np.int64)), _dev(torch, cat(tc, np.float64)),
                               _dev(torch, cat(tp, np.float64)), _dev(torch, cat(rk, np.int32)))
    d_pts = torch.frombuffer(bytearray(bytes(pts)), dtype=torch.uint8).to("cuda")
    i32, f64 = torch.int32, torch.float64
    o_first, o_count, o_mb = _empty(torch, S, i32), _empty(torch, S, i32), _empty(torch, S, i32)
    o_bt, o_order, o_end = _empty(torch, S, f64), _empty(torch, S, i32), _empty(torch, S, i32)
    o_nch, o_rate, o_sat, o_st = (_empty(torch, P, i32), _empty(torch, P, f64),
                                  _empty(torch, P, i32), _empty(torch, P, i32))
    stream = torch.cuda.current_stream().cuda_stream
    max_servers = max(sizes) if sizes else 1
    st = lib.cs_gbp_batch(d_pts.data_ptr(), P, max(max_servers, 1), d_mem.data_ptr(), d_tc.data_ptr(),
                          d_tp.data_ptr(), d_rk.data_ptr(), o_first.data_ptr(), o_count.data_ptr(),
                          o_mb.data_ptr(), o_bt.data_ptr(), o_order.data_ptr(), o_end.data_ptr(),
                          o_nch.data_ptr(), o_rate.data_ptr(), o_sat.data_ptr(), o_st.data_ptr(),
                          stream)
    N.check(st, "cs_gbp_batch")
    h = lambda t: t.cpu().numpy()
    return GbpOut(h(o_st)[:P], h(o_first)[:off], h(o_count)[:off], h(o_mb)[:off], h(o_bt)[:off],
                  h(o_order)[:off], h(o_end)[:off], h(o_nch)[:P], h(o_rate)[:P], h(o_sat)[:P],
                  np.asarray(bases, np.int64), np.asarray(sizes, np.int64))


@dataclass
class GcaOut:
    status: np.ndarray
    n_chains: np.ndarray
    n_edges: np.ndarray
    chain_srv: np.ndarray   # [P, max_chains, max_hops]
    chain_len: np.ndarray   # [P, max_chains]
    caps: np.ndarray
    times: np.ndarray


def gca_batch(fleets: Sequence[Fleet], services: Sequence[ServiceSpec],
              firsts: Sequence[np.ndarray], counts: Sequence[np.ndarray],
              residuals: Sequence[np.ndarray | None] | None = None,
              fleet_of_point: Sequence[int] | None = None, max_chains: int | None = None) -> GcaOut:
    """greedy_cache_allocation for every placement."""
    lib = N.load()
    torch = _torch()
    P = len(firsts)
    if fleet_of_point is None:
        fleet_of_point = list(range(P))
    bases, sizes = [], []
    mem, tc, tp, rk, fi, co, rs = [], [], [], [], [], [], []
    off = 0
    any_res = residuals is not None and any(r is not None for r in residuals)
    max_used, max_L = 1, 1
    for p in range(P):
        f = fleets[fleet_of_point[p]]
        bases.append(off)
        sizes.append(len(f.servers))
        mem.append(f.mem)
        tc.append(f.tau_c)
        tp.append(f.tau_p)
        rk.append(f.rank)
        fi.append(np.asarray(firsts[p], np.int32))
        c = np.asarray(counts[p], np.int32)
        co.append(c)
        max_used = max(max_used, int((c > 0).sum()))
        max_L = max(max_L, services[p].block_count)
        if any_res:
            r = residuals[p]
            rs.append(np.asarray(r, np.int64) if r is not None else np.full(len(f.servers), -1, np.int64))
        off += len(f.servers)
    if any_res:
        for p in range(P):
            if residuals[p] is None:
                raise ValueError("residual_slots must be given for every point or none")
    pts = (N.ComposePoint * max(P, 1))()
    for p in range(P):
        svc = services[p]
        pts[p] = N.ComposePoint(sizes[p], bases[p], svc.block_count, svc.block_bytes,
                                svc.cache_slot_bytes, 1, 0.0, 0.5)
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs and off else np.zeros(1, dt)
    d = lambda a: _dev(torch, a)
    d_mem, d_tc, d_tp, d_rk = d(cat(mem, np.int64)), d(cat(tc, np.float64)), d(cat(tp, np.float64)), d(cat(rk, np.int32))
    d_fi, d_co = d(cat(fi, np.int32)), d(cat(co, np.int32))
    d_rs = d(cat(rs, np.int64)) if any_res else None
    d_pts = torch.frombuffer(bytearray(bytes(pts)), dtype=torch.uint8).to("cuda")
    max_hops = max(1, min(max_used, max_L))
    if max_chains is None:
        # iterations are bounded by |E|+1 (cache_alloc.py:107); E <= U*(U+1)
        max_chains = max(4, max_used * (max_used + 1) + 1)
        max_chains = min(max_chains, 1 << 16)
    i32, f64, i64 = torch.int32, torch.float64, torch.int64
    o_srv = _empty(torch, P * max_chains * max_hops, i32)
    o_len, o_caps, o_times = (_empty(torch, P * max_chains, i32), _empty(torch, P * max_chains, i32),
                              _empty(torch, P * max_chains, f64))
    o_nch, o_ne, o_st = _empty(torch, P, i32), _empty(torch, P, i64), _empty(torch, P, i32)
    stream = torch.cuda.current_stream().cuda_stream
    st = lib.cs_gca_batch(d_pts.data_ptr(), P, max(max(sizes) if sizes else 1, 1), max_L,
                          d_mem.data_ptr(), d_tc.data_ptr(), d_tp.data_ptr(), d_rk.data_ptr(),
                          d_fi.data_ptr(), d_co.data_ptr(), d_rs.data_ptr() if d_rs is not None else None,
                          max_chains, max_hops, o_srv.data_ptr(), o_len.data_ptr(), o_caps.data_ptr(),
                          o_times.data_ptr(), o_nch.data_ptr(), o_ne.data_ptr(), o_st.data_ptr(), stream)
    N.check(st, "cs_gca_batch")
    h = lambda t: t.cpu().numpy()
    return GcaOut(h(o_st)[:P], h(o_nch)[:P], h(o_ne)[:P],
                  h(o_srv)[:P * max_chains * max_hops].reshape(P, max_chains, max_hops),
                  h(o_len)[:P * max_chains].reshape(P, max_chains),
                  h(o_caps)[:P * max_chains].reshape(P, max_chains),
                  h(o_times)[:P * max_chains].reshape(P, max_chains))
