"""Full-size parity pins (tests/golden/full_runs.json, generated from the
unmodified reference by tests/golden/make_golden_full.py):

  * all 4,096 simulations of the BASELINE C4 sweep (per-simulation digest of
    result + trace + agent stats), through the engine exactly as bench.py
    runs it (verify off: prefix matches come from the held state) and with
    the block-hash probe re-deriving every match (verify on);
  * full-size C3 (2,048 agents, DeepSeek-V3 MLA sizing, aimd h_thresh 0.3);
  * the C5 shape at 1,024 and 4,096 agents (aimd and agent_cap).

The CPU restatement (oracle/) is pinned against the same fixtures first.
"""
import json
import os

import numpy as np
import pytest

from paper_2601_22705_b200 import config, engine
from tests.golden_cases import FULL_CASES, full_case_scenario
from tests.golden_hash import sim_digest
from tests.helpers import GOLDEN, oracle_run

FULL = json.load(open(os.path.join(GOLDEN, "full_runs.json")))
C4_SAMPLE = [0, 1, 63, 777, 1024, 2048, 3333, 4095]


def _oracle_digest(s, pol=None, pop=None):
    o = oracle_run(s, pol, pop=pop)
    tr = np.ctypeslib.as_array(o["raw_trace"])[: o["n_trace"]]
    ag = np.ctypeslib.as_array(o["raw_agents"])[: s.workload.agents]
    return sim_digest(o["status"], o["result"], tr, ag)


def test_fixture_shape():
    assert len(FULL["c4_seed42"]) == 4096
    assert len(set(FULL["c4_seed42"])) > 200  # the grid really varies the runs (221 distinct)
    for case in FULL_CASES:
        assert FULL[case["id"]]["status"] == 0


@pytest.mark.parametrize("k", C4_SAMPLE)
def test_oracle_c4_sweep_sims_match_reference(k):
    s = config.c4_sweep(k + 1)[k]
    assert _oracle_digest(s) == FULL["c4_seed42"][k]


def test_oracle_full_c3_matches_reference():
    case = next(c for c in FULL_CASES if c["id"] == "c3_aimd_h03")
    s, pol = full_case_scenario(case)
    assert _oracle_digest(s, pol) == FULL["c3_aimd_h03"]["digest"]


@pytest.mark.slow
@pytest.mark.parametrize("cid", ["c5s1024_aimd", "c5s1024_cap256"])
def test_oracle_scaled_c5_matches_reference(cid):
    case = next(c for c in FULL_CASES if c["id"] == cid)
    s, pol = full_case_scenario(case)
    assert _oracle_digest(s, pol) == FULL[cid]["digest"]


# ------------------------------------------------------------------ GPU

def _batch_digests(b: engine.Batch) -> list[str]:
    res, stats, rows = b.outputs()
    out = []
    for i in range(b.n):
        r = b.result(i)
        out.append(sim_digest(r["status"], r, rows[i], stats[i]))
    return out


@pytest.fixture(scope="module")
def c4_specs():
    pop = engine.Population(config.c1_toy().workload, 42)
    return [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep(4096)]


@pytest.mark.gpu
@pytest.mark.parametrize("verify", [False, True])
def test_gpu_full_c4_sweep_every_sim_matches_reference(c4_specs, verify):
    # verify=False is the benchmarked configuration (bench.py)
    b = engine.Batch(c4_specs, verify=verify, host_outputs=True)
    assert b.run() == 0
    got = _batch_digests(b)
    b.close()
    bad = [k for k in range(4096) if got[k] != FULL["c4_seed42"][k]]
    assert bad == [], f"{len(bad)} sims differ, first {bad[:8]}"


@pytest.mark.gpu
def test_gpu_full_c4_verify_on_equals_verify_off(c4_specs):
    outs = []
    for verify in (False, True):
        b = engine.Batch(c4_specs, verify=verify, host_outputs=True)
        b.run()
        res, stats, rows = b.outputs()
        outs.append((res.copy(), [s.copy() for s in stats], [r.copy() for r in rows]))
        b.close()
    (ra, sa, ta), (rb, sb, tb) = outs
    skip = {"device_cycles", "evict_scanned"}  # chains (verify off) vs pages (verify on)
    for f in ra.dtype.names:
        if f not in skip:
            assert (ra[f] == rb[f]).all(), f
    for k in range(4096):
        assert sa[k].tobytes() == sb[k].tobytes() and ta[k].tobytes() == tb[k].tobytes(), k


@pytest.mark.gpu
@pytest.mark.parametrize("cid", [c["id"] for c in FULL_CASES])
@pytest.mark.parametrize("verify", [False, True])
def test_gpu_full_size_configs_match_reference(cid, verify):
    case = next(c for c in FULL_CASES if c["id"] == cid)
    s, pol = full_case_scenario(case)
    b = engine.Batch([engine.SimSpec.from_scenario(s, pol)], verify=verify, host_outputs=True)
    assert b.run() == 0
    r = b.result(0)
    from tests.golden_hash import result_record
    assert result_record(r) == FULL[cid]["result"]
    assert _batch_digests(b)[0] == FULL[cid]["digest"]
    b.close()
