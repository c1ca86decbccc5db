"""The JSON artifacts of the compose -> simulate path.

Same files as the reference's ``chainserve.config`` (config.py:21-133), so a
chains.json written by either side loads in the other:

* a system file: ``block_count``, ``block_bytes``, ``cache_slot_bytes`` and a
  ``servers`` list (``id``, ``memory_bytes``, ``comm_time_s``,
  ``per_block_compute_s``); a server list may also stand alone;
* chains.json (written by ``compose``): the service, the servers, the
  placement (``{server id: {first_block, block_count}}`` for the used
  servers), the chains (server ids, service time, rate, capacity) and the
  total rate -- self-contained, so ``simulate`` needs nothing else;
* every artifact carries a provenance record: the SHA-256 of each input file
  plus the run parameters.

Pure host IO; the composition and simulation themselves run on the GPU.
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path
from typing import Sequence

from .model import BlockPlacement, ComposedSystem, ServerSpec, ServiceSpec, build_chain

ARTIFACT_VERSION = "0.1.0"  # the reference's artifact format version

_SERVER_FIELDS = (("id", str), ("memory_bytes", int), ("comm_time_s", float), ("per_block_compute_s", float))
_SERVICE_FIELDS = ("block_count", "block_bytes", "cache_slot_bytes")


def sha256_of(path) -> str:
    h = hashlib.sha256()
    h.update(Path(path).read_bytes())
    return h.hexdigest()


def provenance(inputs: dict, **parameters) -> dict:
    """Input file hashes + run parameters (identical inputs, identical artifacts)."""
    return {"artifact": "chainserve", "version": ARTIFACT_VERSION,
            "inputs": {name: sha256_of(path) for name, path in inputs.items()},
            "parameters": parameters}


def save_json(path, payload: dict) -> None:
    Path(path).write_text(json.dumps(payload, indent=2, sort_keys=True) + "\n")


def _server(d: dict) -> ServerSpec:
    return ServerSpec(**{name: cast(d[name]) for name, cast in _SERVER_FIELDS})


def _service(d: dict) -> ServiceSpec:
    return ServiceSpec(**{name: int(d[name]) for name in _SERVICE_FIELDS})


def load_system(path) -> tuple[ServiceSpec, tuple[ServerSpec, ...]]:
    """A system file: the service definition and (optionally) its servers."""
    data = json.loads(Path(path).read_text())
    return _service(data), tuple(_server(s) for s in data.get("servers", []))


def load_servers(path) -> tuple[ServerSpec, ...]:
    """A server list: a bare array or ``{"servers": [...]}``."""
    data = json.loads(Path(path).read_text())
    return tuple(_server(s) for s in (data["servers"] if isinstance(data, dict) else data))


def service_to_dict(service: ServiceSpec) -> dict:
    return {name: getattr(service, name) for name in _SERVICE_FIELDS}


def servers_to_list(servers: Sequence[ServerSpec]) -> list[dict]:
    return [{name: getattr(s, name) for name, _ in _SERVER_FIELDS} for s in servers]


def placement_to_dict(placement: BlockPlacement) -> dict:
    """Used servers only: ``{id: {"first_block": a, "block_count": m}}``."""
    out = {}
    for srv, first, count in zip(placement.servers, placement.first_block, placement.block_count):
        if count > 0:
            out[srv.id] = {"first_block": first, "block_count": count}
    return out


def system_to_dict(system: ComposedSystem, capacity_parameter: int | None = None) -> dict:
    """The self-contained chains file body."""
    pl = system.placement
    chains = [{"servers": list(chain.server_ids), "service_time_s": chain.service_time_s,
               "service_rate_per_s": chain.rate, "capacity": cap}
              for chain, cap in zip(system.chains, system.capacities)]
    return {"capacity_parameter": capacity_parameter, "service": service_to_dict(pl.service),
            "servers": servers_to_list(pl.servers), "placement": placement_to_dict(pl),
            "chains": chains, "total_service_rate_per_s": system.total_rate}


def load_composed(path) -> tuple[ComposedSystem, dict]:
    """Rebuild the composed system of a chains file (chains re-derived from
    their server lists, exactly as composition built them); also returns the
    raw file contents."""
    data = json.loads(Path(path).read_text())
    service = _service(data["service"])
    servers = tuple(_server(s) for s in data["servers"])
    index = {s.id: i for i, s in enumerate(servers)}
    first, count = [0] * len(servers), [0] * len(servers)
    for sid, entry in data["placement"].items():
        first[index[sid]] = int(entry["first_block"])
        count[index[sid]] = int(entry["block_count"])
    placement = BlockPlacement(service, servers, tuple(first), tuple(count))
    chains = tuple(build_chain(placement, c["servers"]) for c in data["chains"])
    return ComposedSystem(placement, chains, tuple(int(c["capacity"]) for c in data["chains"])), data
