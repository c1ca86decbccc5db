"""The chains.json artifacts and the compose / simulate command line
(SURVEY.md §8(f)4), against artifacts the reference's own CLI wrote
(tests/golden/make_golden_cli.py: PETALS fixture, c = 7).

CPU: the chains file loads into the same composed system (chains re-derived
from their server lists: bit-exact service times and rates) and writes back
the same JSON body.  GPU: ``compose`` writes chains.json / placement.json
byte for byte as the reference; ``simulate`` writes the same stats.json
(quantiles, counts and rep means bit-exact; the segmented simulator's per-job
sums <= 1e-12 relative; the merged mean <= 1e-12)."""

import json
import os
import shutil

import pytest

from conftest import ROOT, close_rel

GOLD = os.path.join(ROOT, "tests", "golden", "cli")


def test_chains_file_round_trip(tmp_path):
    from paper_2604_14993_b200 import config as K

    ref = json.load(open(os.path.join(GOLD, "chains.json")))
    system, raw = K.load_composed(os.path.join(GOLD, "chains.json"))
    assert raw == ref
    body = K.system_to_dict(system, capacity_parameter=ref["capacity_parameter"])
    for k, v in body.items():
        assert v == ref[k], k  # floats compare exactly (same IEEE operations)
    K.save_json(tmp_path / "again.json", {"provenance": ref["provenance"], "evaluation": ref["evaluation"], **body})
    assert (tmp_path / "again.json").read_text() == open(os.path.join(GOLD, "chains.json")).read()
    service, servers = K.load_system(os.path.join(GOLD, "system.json"))
    assert service == system.placement.service and servers == system.placement.servers
    assert K.load_servers(os.path.join(GOLD, "system.json")) == servers


def test_cli_refuses_out_of_scope_modes(tmp_path, capsys):
    from paper_2604_14993_b200 import cli

    rc = cli.main(["simulate", "--chains", os.path.join(GOLD, "chains.json"), "--trace", "t.csv",
                   "--out", str(tmp_path)])
    assert rc == 1 and "outside this engine's scope" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_compose_and_simulate_match_the_reference(tmp_path, monkeypatch):
    from paper_2604_14993_b200 import cli

    shutil.copy(os.path.join(GOLD, "system.json"), tmp_path / "system.json")
    monkeypatch.chdir(tmp_path)  # relative paths, as the golden run
    args = json.load(open(os.path.join(GOLD, "args.json")))
    assert cli.main(["compose", "--service", "system.json", *args["compose"], "--out", "."]) == 0
    for f in ("chains.json", "placement.json"):
        assert (tmp_path / f).read_text() == open(os.path.join(GOLD, f)).read(), f
    assert cli.main(["simulate", "--chains", "chains.json", *args["simulate"], "--out", "."]) == 0
    got, ref = json.load(open(tmp_path / "stats.json")), json.load(open(os.path.join(GOLD, "stats.json")))
    assert got.keys() == ref.keys()
    sums = {"mean_waiting_s", "mean_service_s", "mean_occupancy", "occ_first_half", "occ_second_half",
            "little_law_gap", "mean_response_s", "response_ci_half_width_s", "occupancy_ci_half_width",
            "rep_mean_occupancy", "per_chain_utilization"}
    for k, v in ref.items():
        g = got[k]
        if k in sums:
            gl, vl = (g, v) if isinstance(v, list) else ([g], [v])
            assert all(close_rel(a, b) for a, b in zip(gl, vl)), (k, g, v)
        else:
            assert g == v, (k, g, v)
