"""Workload types and the calibration helpers used to build instances.

Restates the parts of chainserve/workload.py that sit on the compose ->
simulate path or generate its instances: ``PoissonWorkload`` (the simulator's
input type, workload.py:177-185), the trace/sampled workload types (accepted
by ``SimConfig`` but simulated only in a later round),
and the timing model (workload.py:23-167) that turns GPU profiles and RTTs
into ``ServerSpec`` lists.  Plus the synthetic fleet generators the benchmark
configurations are defined on.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from .model import GB, TAIL_ID, ServerChain, ServerSpec, ServiceSpec


@dataclass(frozen=True)
class GpuProfile:
    flops_tflops: float
    mem_bandwidth_gb_per_ms: float
    memory_bytes: int
    per_block_overhead_ms: float = 1.0
    per_block_flops_gflop: float = 5.0

    def __post_init__(self):
        if min(self.flops_tflops, self.mem_bandwidth_gb_per_ms, self.memory_bytes,
               self.per_block_overhead_ms, self.per_block_flops_gflop) <= 0:
            raise ValueError("profile figures must all be positive")


def derive_tau_p(profile: GpuProfile, block_bytes: int, mean_input_tokens: float,
                 mean_output_tokens: float) -> float:
    """Per-block compute seconds: overhead + prefill + decode (workload.py:39-62)."""
    if mean_input_tokens < 0:
        raise ValueError("mean_input_tokens must be >= 0")
    if mean_output_tokens < 1:
        raise ValueError("mean_output_tokens must be >= 1")
    prefill_ms = profile.per_block_flops_gflop / profile.flops_tflops
    decode_ms = (block_bytes / GB) / profile.mem_bandwidth_gb_per_ms
    total_ms = (profile.per_block_overhead_ms + prefill_ms * mean_input_tokens
                + decode_ms * (mean_output_tokens - 1))
    return total_ms / 1000.0


class RttMatrix:
    """Symmetric RTTs in ms with a per-message overhead (workload.py:65-106)."""

    def __init__(self, nodes: Sequence[str], rtt_ms, overhead_ms: float = 18.0):
        self.nodes = tuple(nodes)
        self.values_ms = np.asarray(rtt_ms, dtype=float)
        self.overhead_ms = float(overhead_ms)
        n = len(self.nodes)
        if self.values_ms.shape != (n, n):
            raise ValueError(f"matrix shape {self.values_ms.shape} does not match {n} nodes")
        if len(set(self.nodes)) != n:
            raise ValueError("duplicate node ids")
        if np.any(self.values_ms < 0) or np.any(np.diag(self.values_ms) != 0):
            raise ValueError("RTT values must be >= 0 with a zero diagonal")
        if not np.array_equal(self.values_ms, self.values_ms.T):
            raise ValueError("RTT matrix must be symmetric")
        if self.overhead_ms < 0:
            raise ValueError("overhead_ms must be >= 0")
        self._index = {v: i for i, v in enumerate(self.nodes)}

    def rtt_ms(self, a: str, b: str) -> float:
        return float(self.values_ms[self._index[a], self._index[b]])


def derive_tau_c(rtt: RttMatrix, orchestrator: str, node: str, mean_output_tokens: float) -> float:
    """One relay per generated token: tokens * (rtt + overhead) ms (workload.py:109-121)."""
    if mean_output_tokens < 0:
        raise ValueError("mean_output_tokens must be >= 0")
    return mean_output_tokens * (rtt.rtt_ms(orchestrator, node) + rtt.overhead_ms) / 1000.0


@dataclass(frozen=True)
class ServiceTimeModel:
    service: ServiceSpec
    profiles: Mapping[str, GpuProfile]
    rtt: RttMatrix
    orchestrator: str

    def tau_p_s(self, server_id: str, input_tokens: float, output_tokens: float) -> float:
        return derive_tau_p(self.profiles[server_id], self.service.block_bytes, input_tokens,
                            output_tokens)

    def tau_c_s(self, server_id: str, output_tokens: float) -> float:
        return derive_tau_c(self.rtt, self.orchestrator, server_id, output_tokens)

    def server_specs(self, mean_input_tokens: float, mean_output_tokens: float):
        return tuple(
            ServerSpec(sid, p.memory_bytes, self.tau_c_s(sid, mean_output_tokens),
                       self.tau_p_s(sid, mean_input_tokens, mean_output_tokens))
            for sid, p in self.profiles.items())

    def request_service_time(self, chain: ServerChain, input_tokens: int, output_tokens: int) -> float:
        if input_tokens <= 0 or output_tokens <= 0:
            raise ValueError("token counts must be positive")
        total = 0.0
        for e in chain.edges:
            if e.dst != TAIL_ID:
                total += self.tau_c_s(e.dst, output_tokens)
                total += self.tau_p_s(e.dst, input_tokens, output_tokens) * e.blocks_at_dst
        return total


@dataclass(frozen=True)
class TraceRecord:
    arrival_s: float
    input_tokens: int
    output_tokens: int


@dataclass(frozen=True)
class PoissonWorkload:
    """Poisson arrivals at ``rate`` with unit-mean exponential sizes (workload.py:177-185)."""

    rate: float

    def __post_init__(self):
        if self.rate <= 0:
            raise ValueError("rate must be positive")


@dataclass(frozen=True)
class SampledWorkload:
    arrivals_s: tuple[float, ...]
    sizes: tuple[float, ...]

    def __post_init__(self):
        if len(self.arrivals_s) != len(self.sizes):
            raise ValueError("arrivals and sizes must align")
        if any(b < a for a, b in zip(self.arrivals_s, self.arrivals_s[1:])):
            raise ValueError("arrival times must be nondecreasing")


@dataclass(frozen=True)
class TraceWorkload:
    records: tuple[TraceRecord, ...]

    @property
    def arrivals_s(self) -> tuple[float, ...]:
        return tuple(r.arrival_s for r in self.records)


# --------------------------------------------------------------------------
# synthetic instances of the benchmark configurations
# --------------------------------------------------------------------------
HI_TIER = GpuProfile(flops_tflops=120, mem_bandwidth_gb_per_ms=1.02, memory_bytes=40 * GB)
LO_TIER = GpuProfile(flops_tflops=80, mem_bandwidth_gb_per_ms=0.51, memory_bytes=20 * GB)
PETALS_SERVICE = ServiceSpec(block_count=70, block_bytes=int(1.32 * GB), cache_slot_bytes=int(0.11 * GB))


def _philox(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))


def petals_instance(J: int = 10, eta: float = 0.2, seed: int = 101):
    """Geo-distributed PETALS-style fleet of BASELINE config 1 (L=70, BLOOM-176B-like).

    Same construction as the reference's test fixture wan_gpu_fixture
    (pkg/tests/conftest.py:81-97): a Philox(seed) RTT matrix over
    orchestrator + J nodes (upper triangle, U(5,60) ms rounded to 1e-3), the
    first int(eta*J) nodes on the 40 GB tier, calibrated at 2000 input / 20
    output tokens.  Returns (service, servers, model).
    """
    rng = _philox(seed)
    n_hi = int(eta * J)
    nodes = ["orch"] + [f"n{i:02d}" for i in range(J)]
    rtt = np.zeros((J + 1, J + 1))
    for i in range(J + 1):
        for j in range(i + 1, J + 1):
            rtt[i, j] = rtt[j, i] = round(float(rng.uniform(5, 60)), 3)
    model = ServiceTimeModel(PETALS_SERVICE,
                             {f"n{i:02d}": (HI_TIER if i < n_hi else LO_TIER) for i in range(J)},
                             RttMatrix(nodes, rtt, overhead_ms=18.0), "orch")
    return PETALS_SERVICE, model.server_specs(2000, 20), model


def fleet(J: int, L: int = 80, seed: int = 7, block_bytes: int = int(1.32 * GB),
          cache_slot_bytes: int = int(0.11 * GB), hi_fraction: float = 0.2):
    """Two-tier heterogeneous fleet of SURVEY.md §8(d) (configs 3-4).

    rng = Philox(SeedSequence(seed)); per server: hi tier if rng.random() <
    hi_fraction, rtt ~ U(5, 60) ms, tau_c = 20*(rtt+18)/1000 s, tau_p from
    derive_tau_p(profile, block_bytes, 2000, 20).  Returns (service, servers).
    """
    rng = _philox(seed)
    service = ServiceSpec(L, block_bytes, cache_slot_bytes)
    servers = []
    for i in range(J):
        prof = HI_TIER if rng.random() < hi_fraction else LO_TIER
        rtt = float(rng.uniform(5, 60))
        servers.append(ServerSpec(f"n{i:04d}", prof.memory_bytes, 20 * (rtt + 18) / 1000,
                                  derive_tau_p(prof, block_bytes, 2000, 20)))
    return service, tuple(servers)
