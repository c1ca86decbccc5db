"""Golden artifacts of the reference's own CLI (run here, where
/root/reference exists): the PETALS fixture system file, then
``chainserve compose --c 7`` and ``chainserve simulate`` on it.  The engine's
CLI must write the same chains.json / placement.json (byte for byte) and the
same stats.json (to the stated tolerances).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cli.py
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

ARGS = json.load(open(os.path.join(HERE, "cli", "args.json")))  # shared with tests/test_cli.py
ARGS_COMPOSE, ARGS_SIMULATE = ARGS["compose"], ARGS["simulate"]


def main():
    from chainserve import cli  # the reference

    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import wan_gpu_fixture  # the reference's own fixture

    out = os.path.join(HERE, "cli")
    os.makedirs(out, exist_ok=True)
    service, servers, _ = wan_gpu_fixture(10, 0.2, 101)
    system = {"block_count": service.block_count, "block_bytes": service.block_bytes,
              "cache_slot_bytes": service.cache_slot_bytes,
              "servers": [{"id": s.id, "memory_bytes": s.memory_bytes, "comm_time_s": s.comm_time_s,
                           "per_block_compute_s": s.per_block_compute_s} for s in servers]}
    cwd = os.getcwd()
    os.chdir(out)  # relative paths: the provenance hashes file contents only
    try:
        with open("system.json", "w") as fh:
            json.dump(system, fh, indent=2)
        assert cli.main(["compose", "--service", "system.json", *ARGS_COMPOSE, "--out", "."]) == 0
        assert cli.main(["simulate", "--chains", "chains.json", *ARGS_SIMULATE, "--out", "."]) == 0
    finally:
        os.chdir(cwd)


if __name__ == "__main__":
    main()
