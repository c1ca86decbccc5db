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
import os
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
        self.ldr = (self.m + 15) & ~15  # whole 128-byte lines per row (simulator flushes lines)
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
        # simulator workspace per buffer set (the segmented path's prefix is
        # written by the streams stage of the same set)
        self.ws_bytes = self.lib.cs_jffc_sim_workspace_bytes(self.P, reps, self.max_chains, self.max_cap, n_jobs)
        # buffer sets: one for step(), a second one for the pipelined sweep
        self.sets = [self._alloc_set()]
        self.d_S, self.d_resp = self.sets[0]["S"], self.sets[0]["resp"]
        self.d_busy, self.d_summ = self.sets[0]["busy"], self.sets[0]["summ"]
        # sharded (distributed=True): ranks index the union of all shards' responses
        self.distributed = distributed
        N_total = (total_reps if distributed and total_reps else reps) * self.m
        self.rank_list = sorted({r for q in QUANTILES for r in _quantile_ranks(N_total, q)[:2]})
        self.ranks = np.asarray(self.rank_list * self.P, np.int64)
        self.out_vals = np.zeros(len(self.ranks), np.float64)
        self.h_summ = np.zeros(self.P * reps, N.SUMMARY_DTYPE)
        self.stream = torch.cuda.current_stream()

    def _alloc_set(self):
        torch, dev, f64 = self.torch, "cuda", self.torch.float64
        return {"S": torch.empty(self.R * self.lds + 512, dtype=f64, device=dev),  # + CS_STREAM_PAD
                "resp": torch.empty(self.P * self.R * self.ldr, dtype=f64, device=dev),
                "busy": torch.empty(self.P * self.R * self.ldb, dtype=f64, device=dev),
                "summ": torch.empty(self.P * self.R * C.sizeof(N.RepSummary), dtype=torch.uint8,
                                    device=dev),
                "ws": torch.empty(max(self.ws_bytes, 16), dtype=torch.uint8, device=dev),
                "flags": C.c_int32(0)}  # simulation flags cs_sim_streams returns

    # -- stages (buffer set b, CUDA stream st) ------------------------------
    def streams(self, b: int = 0, st=None, whole_sm: bool = False):
        st = st or self.stream
        B = self.sets[b]
        rc = self.lib.cs_sim_streams_ex(self.d_keys.data_ptr(), self.R, self.lds, B["S"].data_ptr(), self.lds,
                                        self.log1p_variant, self.d_pts.data_ptr(), self.P, self.max_chains,
                                        self.max_cap, self.n, self.warm, B["ws"].data_ptr(), self.ws_bytes,
                                        N.CS_STREAMS_WHOLE_SM if whole_sm else 0, C.byref(B["flags"]),
                                        st.cuda_stream)
        N.check(rc, "cs_sim_streams")

    def simulate(self, b: int = 0, st=None):
        st = st or self.stream
        B = self.sets[b]
        rc = self.lib.cs_jffc_sim_ex(
            self.d_pts.data_ptr(), self.P, self.d_rates.data_ptr(), self.d_caps.data_ptr(),
            self.max_chains, self.max_cap, B["S"].data_ptr(), self.lds, 0, self.R, self.R, self.n,
            self.warm, B["resp"].data_ptr(), self.ldr, B["busy"].data_ptr(), self.ldb,
            B["summ"].data_ptr(), None, B["ws"].data_ptr(), self.ws_bytes,
            B["flags"].value, st.cuda_stream)
        N.check(rc, "cs_jffc_sim_ex")

    def statistics(self, b: int = 0, st=None):
        st = st or self.stream
        B = self.sets[b]
        fn = self.lib.cs_rep_stats_dist if self.distributed else self.lib.cs_rep_stats
        rc = fn(B["resp"].data_ptr(), self.P, self.R, self.m, self.ldr, B["summ"].data_ptr(),
                N.ptr(self.ranks, C.c_int64), len(self.rank_list), N.ptr(self.out_vals, C.c_double),
                None, st.cuda_stream)
        N.check(rc, "cs_rep_stats")

    def run_pipelined(self, steps: int, after_stats=None) -> int:
        """`steps` complete sweeps over two buffer sets and two CUDA streams,
        in one deterministic order per sweep k: the simulation (a cooperative
        launch of whole-SM blocks: ceil(units / 16) SMs, 128 of 148 on config
        2), beside it on the SMs it leaves free the exponential streams of
        sweep k+1 (lower priority; they finish beside the statistics), then
        the statistics of sweep k.  Every sweep is computed in full; the
        caller's stream waits for all of them.  ``after_stats(b, stream)``
        runs after each sweep's statistics (e.g. the cross-GPU gather of its
        summaries; the statistics' NCCL collectives are in the same stream).
        Returns the last sweep's set."""
        torch = self.torch
        if len(self.sets) < 2:
            self.sets.append(self._alloc_set())
            # lower number = higher priority (torch clamps to the device's range):
            # the simulation and the statistics chain first, the streams fill in
            self.pipe = [torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-8)]
        s_gen, s_sim = self.pipe
        cur = torch.cuda.current_stream()
        for s_ in self.pipe:
            s_.wait_stream(cur)
        ev_sim = [torch.cuda.Event(), torch.cuda.Event()]
        ev_gen = [torch.cuda.Event(), torch.cuda.Event()]
        if steps > 0:
            self.streams(0, s_gen)
            ev_gen[0].record(s_gen)
        for k in range(steps):
            b = k & 1
            s_sim.wait_event(ev_gen[b])
            self.simulate(b, s_sim)
            ev_sim[b].record(s_sim)
            if k + 1 < steps:
                # set (k+1)&1 was last simulated by sweep k-1 (its statistics
                # read only the responses): the streams of sweep k+1 start
                # beside the simulation of sweep k, on the SMs it leaves free
                s_gen.wait_event(ev_sim[(k + 1) & 1])
                self.streams((k + 1) & 1, s_gen, whole_sm=True)
                ev_gen[(k + 1) & 1].record(s_gen)
            self.statistics(b, s_sim)
            if after_stats is not None:
                after_stats(b, s_sim)
        for s_ in self.pipe:
            cur.wait_stream(s_)
        return (steps - 1) & 1

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

    def summaries(self, b: int = 0) -> np.ndarray:
        self.h_summ[:] = self.sets[b]["summ"].cpu().numpy().view(N.SUMMARY_DTYPE)
        return self.h_summ.reshape(self.P, self.R)

    def busy(self, b: int = 0) -> np.ndarray:
        return self.sets[b]["busy"].cpu().numpy().reshape(self.P, self.R, self.ldb)

    def order_stats(self) -> list[dict]:
        k = len(self.rank_list)
        return [{self.rank_list[i]: float(self.out_vals[p * k + i]) for i in range(k)}
                for p in range(self.P)]
