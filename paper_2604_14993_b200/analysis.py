"""``ChainRates``: the compose -> simulate handoff type (chainserve/analysis.py:27-64).

The occupancy bounds and capacity-bound tuning of analysis.py are the
SURVEY.md §8(f) "next" row 1 and are not part of this round's engine.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

from .model import ComposedSystem, py_sum


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
