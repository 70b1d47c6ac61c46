"""GPU engine, offload mode (EvictionMode::kOffload), vs the reference — bit-exact.

The device runs the node-level radix tree (csrc/tree.cuh) with a cooperative
frontier scan; every offload fixture recorded from the unmodified reference
(tests/golden/offload_runs.json: presets, C1, scaled C3 with thousands of
quirk-Q1 states and corrupted children_with_device counters, randomized
rounds) must come out identical: SimulationResult scalars (offloaded /
reloaded tokens, link busy time, makespan = max(last completion, link)), the
full trace (incl. transfers in flight per tick) and agent stats. The
per-dispatch event log (match / host_matched, reload outcomes, every eviction
victim in order, inserts) must equal the CPU oracle's."""
import json
import os

import pytest

from paper_2601_22705_b200 import abi, engine
from tests.golden_hash import run_record
from tests.helpers import GOLDEN, load_presets, oracle_run
from tests.offload_cases import OFFLOAD_CASES, offload_scenario
from tests.parity import diff_all

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(GOLDEN, "offload_runs.json")))
AGENT_ALL = abi.AGENT_FIELDS + ("finish_time", "finish_ordinal")


def gpu_run(case, warps=0, log=False):
    s, pol = offload_scenario(case, load_presets())
    spec = engine.SimSpec.from_scenario(s, pol)
    b = engine.Batch([spec], warps_per_sim=warps, log_capacity=(1 << 22) if log else 0)
    st = b.run()
    out = dict(status=st, result=b.result(0), trace=b.trace(0), agents=b.agent_stats(0))
    if log:
        out["log"] = b.log(0)
    b.close()
    return out, s, pol


def check(rec, gold):
    assert rec["status"] == gold["status"]
    assert rec["result"] == gold["result"]
    assert rec["n_trace"] == gold["n_trace"]
    assert rec["trace_sha"] == gold["trace_sha"]
    assert rec["agents_sha"] == gold["agents_sha"]


@pytest.mark.parametrize("cid", [c["id"] for c in OFFLOAD_CASES])
def test_gpu_offload_reproduces_reference(cid):
    case = next(c for c in OFFLOAD_CASES if c["id"] == cid)
    run, _, _ = gpu_run(case)
    check(run_record(run), GOLD[cid])


@pytest.mark.parametrize("cid", ["off_preset_thrash", "off_c3s16", "off_c1_offload",
                                 "off_c3s32_aimd"])
def test_gpu_offload_event_log_equals_oracle(cid):
    case = next(c for c in OFFLOAD_CASES if c["id"] == cid)
    g, s, pol = gpu_run(case, log=True)
    pop = engine.Population(s.workload, s.seed)
    o = oracle_run(s, pol, log=True, pop=pop.c)
    assert diff_all(g, o, AGENT_ALL) == []
    assert g["log"] == o["log"]


@pytest.mark.parametrize("cid", ["off_preset_thrash", "off_c3s32"])
@pytest.mark.parametrize("warps", [1, 8, 32])
def test_gpu_offload_warps_do_not_change_results(cid, warps):
    case = next(c for c in OFFLOAD_CASES if c["id"] == cid)
    run, _, _ = gpu_run(case, warps=warps)
    check(run_record(run), GOLD[cid])


def test_offload_and_discard_sims_in_one_batch():
    from tests.golden_cases import CASES, case_scenario
    gold_d = json.load(open(os.path.join(GOLDEN, "reference_runs.json")))
    pres = load_presets()
    picks = [c for c in OFFLOAD_CASES if c["id"] != "off_c3s64"]
    dcases = [c for c in CASES if c["id"] in ("preset_thrash_aimd", "c1_uncontrolled", "rand_3")]
    specs = []
    for c in picks:
        s, pol = offload_scenario(c, pres)
        specs.append(engine.SimSpec.from_scenario(s, pol))
    for c in dcases:
        s, pol = case_scenario(c, pres)
        specs.append(engine.SimSpec.from_scenario(s, pol))
    b = engine.Batch(specs)
    b.run()
    for i, c in enumerate(picks + dcases):
        run = dict(status=b.result(i)["status"], result=b.result(i), trace=b.trace(i),
                   agents=b.agent_stats(i))
        check(run_record(run), (GOLD if c in picks else gold_d)[c["id"]])
    b.close()
