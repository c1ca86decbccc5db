"""Device-resident sweep engine: preallocated HBM buffers + the three stage
launches (streams -> JFFC simulation -> statistics) on one CUDA stream.

``run_sim_batch`` (host buffers in/out) is the drop-in path; ``SweepEngine``
is for repeated sweeps of one shape (benchmarks, design-parameter loops):
inputs stay resident in HBM and only the per-replication summaries and the
order statistics come back.  torch provides the device allocations and the
stream; all compute is the engine's own kernels via the C-ABI.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as N
from .sim import QUANTILES, _quantile_ranks


@dataclass
class StageTimes:
    streams_ms: float
    sim_ms: float
    stats_ms: float


class SweepEngine:
    """P sweep points x R replications of n jobs, seed `seed`, reps
    [rep_begin, rep_begin + R) (a shard of n_reps_total when sharded)."""

    # streams, sim; stats: 2 sample selections (hist0, compact, 3x2 digit rounds),
    # leaf-sum+bracket pass, tree combine, 4x2 digit rounds on the candidates
    KERNELS_PER_STEP = 1 + 1 + 2 * (1 + 1 + 6) + 1 + 1 + 8

    def __init__(self, rates_list: Sequence[Sequence[float]], caps_list: Sequence[Sequence[int]],
                 lams: Sequence[float], n_jobs: int, warmup_fraction: float, seed: int, reps: int,
                 rep_begin: int = 0, log1p_variant: int = -1, device: int | None = None,
                 distributed: bool = False, total_reps: int | None = None):
        import torch

        self.torch = torch
        self.lib = N.load()
        if device is not None:
            torch.cuda.set_device(device)
        self.P, self.R, self.n = len(lams), reps, n_jobs
        self.warm = int(warmup_fraction * n_jobs)
        self.m = n_jobs - self.warm
        self.ldr = (self.m + 1) & ~1
        self.lds = 2 * n_jobs
        self.seed, self.rep_begin = seed, rep_begin
        self.log1p_variant = self.lib.cs_host_log1p_variant() if log1p_variant < 0 else log1p_variant
        pts = (N.SimPoint * self.P)()
        rates, caps = [], []
        self.max_chains, self.max_cap = 1, 1
        for p in range(self.P):
            pts[p] = N.SimPoint(len(rates_list[p]), len(rates), float(lams[p]))
            rates.extend(float(x) for x in rates_list[p])
            caps.extend(int(x) for x in caps_list[p])
            self.max_chains = max(self.max_chains, len(rates_list[p]))
            self.max_cap = max(self.max_cap, int(sum(caps_list[p])))
        self.ldb = self.max_chains
        dev = "cuda"
        f64, i64 = torch.float64, torch.int64
        self.d_pts = torch.frombuffer(bytearray(bytes(pts)), dtype=torch.uint8).to(dev)
        self.d_rates = torch.tensor(rates, dtype=f64, device=dev)
        self.d_caps = torch.tensor(caps, dtype=torch.int32, device=dev)
        # Philox keys of replications rep_begin.. (host SeedSequence, exact)
        w = N.seed_words(seed)
        reps_a = np.arange(rep_begin, rep_begin + reps, dtype=np.uint64)
        keys = np.zeros(2 * reps, np.uint64)
        N.check(self.lib.cs_philox_keys(N.ptr(w, C.c_uint32), len(w), N.ptr(reps_a, C.c_uint64),
                                        reps, N.ptr(keys, C.c_uint64)), "cs_philox_keys")
        self.h_keys = keys
        self.d_keys = torch.from_numpy(keys.view(np.int64)).to(dev)
        self.d_S = torch.empty(reps * self.lds + 512, dtype=f64, device=dev)  # + CS_STREAM_PAD
        self.d_resp = torch.empty(self.P * reps * self.ldr, dtype=f64, device=dev)
        self.d_busy = torch.empty(self.P * reps * self.ldb, dtype=f64, device=dev)
        self.d_summ = torch.empty(self.P * reps * C.sizeof(N.RepSummary), dtype=torch.uint8, device=dev)
        wsb = self.lib.cs_jffc_sim_workspace_bytes(self.P, reps, self.max_chains, self.max_cap, n_jobs)
        self.d_ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
        self.ws_bytes = wsb
        # sharded (distributed=True): ranks index the union of all shards' responses
        self.distributed = distributed
        N_total = (total_reps if distributed and total_reps else reps) * self.m
        self.rank_list = sorted({r for q in QUANTILES for r in _quantile_ranks(N_total, q)[:2]})
        self.ranks = np.asarray(self.rank_list * self.P, np.int64)
        self.out_vals = np.zeros(len(self.ranks), np.float64)
        self.h_summ = np.zeros(self.P * reps, N.SUMMARY_DTYPE)
        self.stream = torch.cuda.current_stream()

    # -- stages -----------------------------------------------------------
    def streams(self):
        st = self.lib.cs_exp_streams(self.d_keys.data_ptr(), self.R, self.lds, self.d_S.data_ptr(),
                                     self.lds, self.log1p_variant, self.stream.cuda_stream)
        N.check(st, "cs_exp_streams")

    def simulate(self):
        st = self.lib.cs_jffc_sim(
            self.d_pts.data_ptr(), self.P, self.d_rates.data_ptr(), self.d_caps.data_ptr(),
            self.max_chains, self.max_cap, self.d_S.data_ptr(), self.lds, 0, self.R, self.R, self.n,
            self.warm, self.d_resp.data_ptr(), self.ldr, self.d_busy.data_ptr(), self.ldb,
            self.d_summ.data_ptr(), None, self.d_ws.data_ptr(), self.ws_bytes, self.stream.cuda_stream)
        N.check(st, "cs_jffc_sim")

    def statistics(self):
        fn = self.lib.cs_rep_stats_dist if self.distributed else self.lib.cs_rep_stats
        st = fn(self.d_resp.data_ptr(), self.P, self.R, self.m, self.ldr, self.d_summ.data_ptr(),
                N.ptr(self.ranks, C.c_int64), len(self.rank_list), N.ptr(self.out_vals, C.c_double),
                None, self.stream.cuda_stream)
        N.check(st, "cs_rep_stats")

    def step(self, timed: bool = False) -> StageTimes | None:
        """One full sweep on the device; optional per-stage CUDA-event times."""
        torch = self.torch
        if not timed:
            self.streams()
            self.simulate()
            self.statistics()
            return None
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(self.stream)
        self.streams()
        ev[1].record(self.stream)
        self.simulate()
        ev[2].record(self.stream)
        self.statistics()
        ev[3].record(self.stream)
        ev[3].synchronize()
        return StageTimes(ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]))

    def summaries(self) -> np.ndarray:
        self.h_summ[:] = self.d_summ.cpu().numpy().view(N.SUMMARY_DTYPE)
        return self.h_summ.reshape(self.P, self.R)

    def busy(self) -> np.ndarray:
        return self.d_busy.cpu().numpy().reshape(self.P, self.R, self.ldb)

    def order_stats(self) -> list[dict]:
        k = len(self.rank_list)
        return [{self.rank_list[i]: float(self.out_vals[p * k + i]) for i in range(k)}
                for p in range(self.P)]
