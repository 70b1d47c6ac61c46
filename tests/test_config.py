"""Host-side configuration mirror (config.hpp / config.cpp semantics) and the
product's phase classifier (metrics.cpp:41-81) against reference outputs."""
import ctypes as C
import json
import os

import pytest

from paper_2601_22705_b200 import abi, config, engine
from tests.golden_cases import CASES, case_scenario
from tests.golden_hash import hx
from tests.helpers import GOLDEN, load_presets, oracle_run

PRESETS_DIR = "/root/reference/proj/configs"


@pytest.mark.skipif(not os.path.isdir(PRESETS_DIR), reason="reference presets absent")
def test_presets_parse_like_the_fixture():
    fixture = load_presets()
    for f in sorted(os.listdir(PRESETS_DIR)):
        if f.endswith(".toml"):
            s = config.load_scenario(os.path.join(PRESETS_DIR, f))
            assert config.scenario_to_dict(s) == fixture[f[:-5]]


def test_fixture_round_trip():
    for name, d in load_presets().items():
        assert config.scenario_to_dict(config.scenario_from_dict(d)) == d


@pytest.mark.parametrize("text,kind,cap", [
    ("uncontrolled", abi.POLICY_UNCONTROLLED, 1), ("aimd", abi.POLICY_AIMD, 1),
    ("agent_cap:8", abi.POLICY_AGENT_CAP, 8), ("request_cap:16", abi.POLICY_REQUEST_CAP, 16)])
def test_parse_policy(text, kind, cap):
    p = config.parse_policy(text, config.ControllerConfig())
    assert (p.kind, p.cap) == (kind, cap)


@pytest.mark.parametrize("text", ["bogus", "agent_cap", "agent_cap:0", "aimd:3", "request_cap:x"])
def test_parse_policy_errors(text):
    with pytest.raises(config.ConfigError):
        config.parse_policy(text, config.ControllerConfig())


def test_unknown_keys_are_rejected():
    with pytest.raises(config.ConfigError):
        config.parse_scenario("[cache]\ncapacity = 4\nbogus = 1\n")
    with pytest.raises(config.ConfigError):
        config.parse_scenario("nope = 1\n")


def test_offload_pseudo_policy_resolves_like_resolve_run():
    s = config.c1_toy()
    pol, eng = s.resolved("offload")
    assert pol.kind == abi.POLICY_UNCONTROLLED and eng.eviction == "offload"


GOLD = json.load(open(os.path.join(GOLDEN, "reference_runs.json")))
PHASE_CASES = [c["id"] for c in CASES if c["id"].startswith(("preset_", "c1_", "eng_"))]


@pytest.mark.parametrize("cid", PHASE_CASES)
def test_product_phase_classifier_matches_reference(cid):
    case = next(c for c in CASES if c["id"] == cid)
    s, pol = case_scenario(case, load_presets())
    pop = engine.Population(s.workload, s.seed)  # keeps the plan buffer alive
    run = oracle_run(s, pol, pop=pop.c)
    rows = (abi.TraceRow * max(1, len(run["trace"])))()
    for i, r in enumerate(run["trace"]):
        rows[i] = abi.TraceRow(**r)
    out = (abi.PhaseLabel * 3)()
    n = C.c_size_t()
    pp = s.resolved(pol)[1].to_abi().phases
    rc = engine.lib().kvg_classify_phases(rows, len(run["trace"]), run["result"]["makespan"],
                                          C.byref(pp), out, 3, C.byref(n))
    assert rc == 0
    got = [[out[i].phase, hx(out[i].start), hx(out[i].end)] for i in range(n.value)]
    assert got == GOLD[cid]["result"]["phases"]
