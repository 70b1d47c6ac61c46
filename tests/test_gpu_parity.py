"""GPU engine vs the CPU oracle (pinned to the reference) — bit-exact.

Every case runs the same seeded inputs through libkvgpu.so (sm_100a kernels
behind the C ABI) and through oracle/libkvoracle.so, and requires identical
SimulationResult scalars (doubles compared bit for bit), trace rows, per-agent
stats including completion time/event, and the per-dispatch event log
(match lengths, eviction sets, insert outcomes, finishes).
"""
import os

import pytest

from paper_2601_22705_b200 import abi, config, engine
from tests.helpers import load_presets, oracle_run
from tests.parity import diff_all

pytestmark = pytest.mark.gpu

PRESETS = "/root/reference/proj/configs"
HERE = os.path.dirname(os.path.abspath(__file__))
AGENT_ALL = abi.AGENT_FIELDS + ("finish_time", "finish_ordinal")


def preset(name):
    return config.scenario_from_dict(load_presets()[name])


def gpu_run(s, policy=None, warps=0, log=False, verify=None):
    spec = engine.SimSpec.from_scenario(s, policy)
    b = engine.Batch([spec], warps_per_sim=warps, log_capacity=(1 << 20) if log else 0,
                     verify=verify)
    st = b.run()
    out = dict(status=st, result=b.result(0), trace=b.trace(0), agents=b.agent_stats(0))
    if log:
        out["log"] = b.log(0)
    b.close()
    return out


CASES = [
    ("smoke", "uncontrolled"), ("smoke", "aimd"), ("smoke", "agent_cap:2"),
    ("smoke", "request_cap:1"),
    ("thrash", "uncontrolled"), ("thrash", "aimd"), ("thrash", "request_cap:16"),
    ("thrash", "agent_cap:8"),
    ("ample", "aimd"), ("ample", "uncontrolled"),
    ("sweep-sensitivity", "aimd"), ("sweep-sensitivity-ulow", "aimd"),
]


@pytest.mark.parametrize("name,policy", CASES)
@pytest.mark.parametrize("warps,verify", [(1, True), (4, True), (0, False)],
                         ids=["table-w1", "table-w4", "chain"])
def test_presets_bit_exact(name, policy, warps, verify):
    """table: page table + block-hash probe on every match (verify on);
    chain: the benchmarked path (chain LRU, no page table) — its eviction
    victims are logged in the reference's order by construction."""
    s = preset(name)
    g = gpu_run(s, policy, warps=warps, log=True, verify=verify)
    o = oracle_run(s, policy, log=True)
    assert g["status"] == o["status"]
    assert diff_all(g, o, AGENT_ALL) == []
    assert g["log"] == o["log"]
    assert g["result"]["lookups"] == o["result"]["lookups"]
    assert g["result"]["agent_steps"] == o["result"]["agent_steps"]


@pytest.mark.parametrize("policy", ["uncontrolled", "aimd"])
@pytest.mark.parametrize("verify", [True, False], ids=["table", "chain"])
def test_c1_toy_bit_exact(policy, verify):
    s = config.c1_toy(policy)
    g = gpu_run(s, policy, log=True, verify=verify)
    o = oracle_run(s, policy, log=True)
    assert diff_all(g, o, AGENT_ALL) == []
    assert g["log"] == o["log"]
    assert g["result"]["evicted_pages"] == o["result"]["evicted_pages"]
