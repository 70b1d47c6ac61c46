"""GPU engine vs the reference's recorded outputs (tests/golden/), bit-exact:
every SimulationResult scalar and phase, the full trace and per-agent stats,
for every golden case — presets x policies, the engine test suite analogs,
seeded random configs, BASELINE C1, C2 (full 1024 agents), scaled C2/C3/C5
shapes, C4 sample sims — and independently of the warps-per-sim mode."""
import json
import os

import pytest

from paper_2601_22705_b200 import engine
from tests.golden_cases import CASES, case_scenario
from tests.golden_hash import run_record
from tests.helpers import GOLDEN, load_presets

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(GOLDEN, "reference_runs.json")))


def gpu_record(case, warps=0, verify=None):
    s, pol = case_scenario(case, load_presets())
    spec = engine.SimSpec.from_scenario(s, pol)
    b = engine.Batch([spec], warps_per_sim=warps, verify=verify)
    st = b.run()
    run = dict(status=st, result=b.result(0), trace=b.trace(0), agents=b.agent_stats(0))
    b.close()
    return run_record(run)


def check(rec, gold):
    assert rec["status"] == gold["status"]
    assert rec["result"] == gold["result"]
    assert rec["n_trace"] == gold["n_trace"]
    assert rec["trace_sha"] == gold["trace_sha"]
    assert rec["agents_sha"] == gold["agents_sha"]


@pytest.mark.parametrize("cid", [c["id"] for c in CASES])
@pytest.mark.parametrize("verify", [False, True], ids=["held", "probe"])
def test_gpu_reproduces_reference(cid, verify):
    # held: the benchmarked configuration (prefix matches from the held
    # state); probe: every match also re-derived by the block-hash probe
    case = next(c for c in CASES if c["id"] == cid)
    check(gpu_record(case, verify=verify), GOLD[cid])


@pytest.mark.parametrize("cid", ["preset_thrash_uncontrolled", "preset_thrash_aimd",
                                 "c1_uncontrolled", "c3s128_aimd_h03", "rand_9", "eng_pausing"])
@pytest.mark.parametrize("warps", [1, 2, 8, 32])
def test_warps_per_sim_do_not_change_results(cid, warps):
    case = next(c for c in CASES if c["id"] == cid)
    check(gpu_record(case, warps), GOLD[cid])


def test_whole_golden_catalogue_in_one_batch():
    """All cases as ONE batch (mixed sizes, warps groups, launch order)."""
    pres = load_presets()
    specs, pops = [], []
    for c in CASES:
        s, pol = case_scenario(c, pres)
        specs.append(engine.SimSpec.from_scenario(s, pol))
    b = engine.Batch(specs)
    b.run()
    for i, c in enumerate(CASES):
        run = dict(status=b.result(i)["status"], result=b.result(i), trace=b.trace(i),
                   agents=b.agent_stats(i))
        check(run_record(run), GOLD[c["id"]])
    b.close()


def test_catalogue_batch_outputs_are_in_caller_order():
    """kvg_batch_outputs on a mixed-warp batch (launch order differs from
    caller order): results[i], and the stats / trace slices located by
    kvg_batch_offsets, belong to simulation i."""
    import numpy as np

    from tests.golden_hash import result_record
    pres = load_presets()
    specs = []
    for c in CASES:
        s, pol = case_scenario(c, pres)
        specs.append(engine.SimSpec.from_scenario(s, pol))
    b = engine.Batch(specs, verify=False, host_outputs=True)
    b.run()
    res, stats, rows = b.outputs()
    for i, c in enumerate(CASES):
        g = GOLD[c["id"]]
        r = b.result(i)
        assert int(res[i]["status"]) == g["status"]
        assert np.float64(res[i]["makespan"]).tobytes() == np.float64(r["makespan"]).tobytes()
        assert result_record(r) == g["result"]
        assert len(rows[i]) == g["n_trace"]
        assert len(stats[i]) == specs[i].population.c.agents
        ref_rows = b.trace_array(i)
        assert rows[i].tobytes() == ref_rows.tobytes()
    b.close()
