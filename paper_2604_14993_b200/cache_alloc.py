"""GCA chain composition -- CUDA-backed drop-in for chainserve/cache_alloc.py.

``greedy_cache_allocation(placement, residual_slots=None)`` keeps the
reference signature (cache_alloc.py:65-68); the shortest-path extraction loop
runs in compose.cu:gca_kernel (frontier-ordered DAG DP, one CTA per
placement).  ``greedy_cache_allocation_batch`` composes many placements in one
launch.
"""

from __future__ import annotations

from typing import Mapping, Sequence

import numpy as np

from . import _compose as CE
from .model import (
    TAIL_ID,
    BlockPlacement,
    ComposedSystem,
    ServerChain,
    cache_slots,
    chain_edges,
)


def _node_order(placement: BlockPlacement) -> dict[str, int]:
    """Lexicographic tie-break order: head, used ids by str, tail (cache_alloc.py:31-37)."""
    order = {"__head__": 0}
    for i, sid in enumerate(sorted(placement.used_ids()), start=1):
        order[sid] = i
    order[TAIL_ID] = len(order)
    return order


def _residual_array(placement: BlockPlacement, residual_slots: Mapping[str, int] | None):
    if residual_slots is None:
        return None
    arr = np.zeros(len(placement.servers), np.int64)
    for i, (srv, m) in enumerate(zip(placement.servers, placement.block_count)):
        if m > 0:
            r = residual_slots[srv.id]  # KeyError for a missing used server, as the reference
            budget = cache_slots(placement, srv.id)
            if not 0 <= r <= budget:
                raise ValueError(f"server {srv.id}: residual {r} outside [0, {budget}]")
            arr[i] = r
    return arr


def _system(placement: BlockPlacement, out: CE.GcaOut, p: int) -> ComposedSystem:
    st = int(out.status[p])
    if st == 2:
        raise ValueError("greedy_cache_allocation: invalid placement/residuals")
    if st == 3:
        raise AssertionError("allocation failed (cap < 1 or no termination within the edge budget)")
    if st != 0:
        raise RuntimeError(f"greedy_cache_allocation: engine status {st}")
    servers = placement.servers
    chains, caps = [], []
    for k in range(int(out.n_chains[p])):
        n = int(out.chain_len[p, k])
        ids = tuple(servers[int(j)].id for j in out.chain_srv[p, k, :n])
        chains.append(ServerChain(ids, chain_edges(placement, ids), float(out.times[p, k])))
        caps.append(int(out.caps[p, k]))
    return ComposedSystem(placement, tuple(chains), tuple(caps))


def greedy_cache_allocation(placement: BlockPlacement,
                            residual_slots: Mapping[str, int] | None = None) -> ComposedSystem:
    """Algorithm 2 (GCA): saturate successively fastest admissible chains."""
    res = _residual_array(placement, residual_slots)
    fleet = CE.Fleet.of(placement.servers)
    out = CE.gca_batch([fleet], [placement.service], [np.asarray(placement.first_block)],
                       [np.asarray(placement.block_count)], [res] if res is not None else None)
    return _system(placement, out, 0)


def greedy_cache_allocation_batch(placements: Sequence[BlockPlacement],
                                  residual_slots: Sequence[Mapping[str, int] | None] | None = None
                                  ) -> list[ComposedSystem]:
    if residual_slots is None:
        res = None
    else:
        res = [_residual_array(pl, r) for pl, r in zip(placements, residual_slots)]
    fleets = [CE.Fleet.of(pl.servers) for pl in placements]
    out = CE.gca_batch(fleets, [pl.service for pl in placements],
                       [np.asarray(pl.first_block) for pl in placements],
                       [np.asarray(pl.block_count) for pl in placements], res)
    return [_system(pl, out, p) for p, pl in enumerate(placements)]
