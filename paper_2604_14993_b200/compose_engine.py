"""Device-resident batched composition: many (instance, c, lambda, rho) points
through GBP-CR placement and GCA chain composition in two launches.

The fleets are structure-of-arrays in HBM (memory bytes, tau_c, tau_p, id
rank per server); ``cs_gbp_batch`` writes the placements that
``cs_gca_batch`` reads in place, so nothing returns to the host between the
two stages.  torch provides the allocations and the stream.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .model import GB
from .workload import HI_TIER, LO_TIER, derive_tau_p


def fleet_soa(J: int, L: int = 80, seed: int = 7, block_bytes: int = int(1.32 * GB),
              hi_fraction: float = 0.2):
    """Vectorised workload.fleet(): the same Philox draws (random(), uniform(5,60)
    alternate per server, one 64-bit word each), as (mem, tau_c, tau_p)."""
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))
    u = rng.random(2 * J)
    hi = u[0::2] < hi_fraction
    rtt = 5.0 + 55.0 * u[1::2]  # numpy random_uniform: low + (high-low) * next_double
    mem = np.where(hi, HI_TIER.memory_bytes, LO_TIER.memory_bytes).astype(np.int64)
    tc = 20 * (rtt + 18) / 1000
    tp = np.where(hi, derive_tau_p(HI_TIER, block_bytes, 2000, 20),
                  derive_tau_p(LO_TIER, block_bytes, 2000, 20))
    return mem, tc, tp


@dataclass
class ComposeTimes:
    gbp_ms: float
    gca_ms: float


class ComposeEngine:
    """P points, each one instance of J servers (ids ranked by position)."""

    def __init__(self, mem: np.ndarray, tau_c: np.ndarray, tau_p: np.ndarray, J: int, L: int,
                 block_bytes: int, cache_slot_bytes: int, capacity, arrival_rate, load_target,
                 max_chains: int = 512):
        import torch

        self.torch = torch
        self.lib = N.load()
        P = len(mem) // J
        self.P, self.J, self.L = P, J, L
        cap = np.broadcast_to(np.asarray(capacity, np.int64), (P,))
        lam = np.broadcast_to(np.asarray(arrival_rate, np.float64), (P,))
        rho = np.broadcast_to(np.asarray(load_target, np.float64), (P,))
        pts = (N.ComposePoint * P)()
        for p in range(P):
            pts[p] = N.ComposePoint(J, p * J, L, block_bytes, cache_slot_bytes, int(cap[p]),
                                    float(lam[p]), float(rho[p]))
        dev = "cuda"
        self.d_pts = torch.frombuffer(bytearray(bytes(pts)), dtype=torch.uint8).to(dev)
        self.d_mem = torch.from_numpy(np.ascontiguousarray(mem, np.int64)).to(dev)
        self.d_tc = torch.from_numpy(np.ascontiguousarray(tau_c, np.float64)).to(dev)
        self.d_tp = torch.from_numpy(np.ascontiguousarray(tau_p, np.float64)).to(dev)
        self.d_rank = torch.from_numpy(np.tile(np.arange(J, dtype=np.int32), P)).to(dev)
        i32, f64, i64 = torch.int32, torch.float64, torch.int64
        S = P * J
        self.first, self.count = torch.empty(S, dtype=i32, device=dev), torch.empty(S, dtype=i32, device=dev)
        self.max_blocks = torch.empty(S, dtype=i32, device=dev)
        self.bound_time = torch.empty(S, dtype=f64, device=dev)
        self.order, self.chain_end = torch.empty(S, dtype=i32, device=dev), torch.empty(S, dtype=i32, device=dev)
        self.g_nch, self.g_rate = torch.empty(P, dtype=i32, device=dev), torch.empty(P, dtype=f64, device=dev)
        self.g_sat, self.g_st = torch.empty(P, dtype=i32, device=dev), torch.empty(P, dtype=i32, device=dev)
        self.max_chains = max_chains
        self.max_hops = min(J, L)
        self.c_srv = torch.empty(P * max_chains * self.max_hops, dtype=i32, device=dev)
        self.c_len = torch.empty(P * max_chains, dtype=i32, device=dev)
        self.c_caps = torch.empty(P * max_chains, dtype=i32, device=dev)
        self.c_times = torch.empty(P * max_chains, dtype=f64, device=dev)
        self.c_nch, self.c_ne = torch.empty(P, dtype=i32, device=dev), torch.empty(P, dtype=i64, device=dev)
        self.c_st = torch.empty(P, dtype=i32, device=dev)
        self.stream = torch.cuda.current_stream()

    def gbp(self):
        st = self.lib.cs_gbp_batch(
            self.d_pts.data_ptr(), self.P, self.J, self.d_mem.data_ptr(), self.d_tc.data_ptr(),
            self.d_tp.data_ptr(), self.d_rank.data_ptr(), self.first.data_ptr(), self.count.data_ptr(),
            self.max_blocks.data_ptr(), self.bound_time.data_ptr(), self.order.data_ptr(),
            self.chain_end.data_ptr(), self.g_nch.data_ptr(), self.g_rate.data_ptr(),
            self.g_sat.data_ptr(), self.g_st.data_ptr(), self.stream.cuda_stream)
        N.check(st, "cs_gbp_batch")

    def gca(self):
        st = self.lib.cs_gca_batch(
            self.d_pts.data_ptr(), self.P, self.J, self.L, self.d_mem.data_ptr(), self.d_tc.data_ptr(),
            self.d_tp.data_ptr(), self.d_rank.data_ptr(), self.first.data_ptr(), self.count.data_ptr(),
            None, self.max_chains, self.max_hops, self.c_srv.data_ptr(), self.c_len.data_ptr(),
            self.c_caps.data_ptr(), self.c_times.data_ptr(), self.c_nch.data_ptr(), self.c_ne.data_ptr(),
            self.c_st.data_ptr(), self.stream.cuda_stream)
        N.check(st, "cs_gca_batch")

    def run(self, timed: bool = False) -> ComposeTimes | None:
        torch = self.torch
        if not timed:
            self.gbp()
            self.gca()
            return None
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(self.stream)
        self.gbp()
        ev[1].record(self.stream)
        self.gca()
        ev[2].record(self.stream)
        ev[2].synchronize()
        return ComposeTimes(ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]))

    def results(self):
        h = lambda t: t.cpu().numpy()
        return dict(gbp_status=h(self.g_st), n_chains_gbp=h(self.g_nch), gca_status=h(self.c_st),
                    n_chains=h(self.c_nch), n_edges=h(self.c_ne),
                    caps=h(self.c_caps).reshape(self.P, self.max_chains),
                    times=h(self.c_times).reshape(self.P, self.max_chains),
                    first=h(self.first).reshape(self.P, self.J), count=h(self.count).reshape(self.P, self.J),
                    chain_len=h(self.c_len).reshape(self.P, self.max_chains),
                    chain_srv=h(self.c_srv).reshape(self.P, self.max_chains, self.max_hops))
