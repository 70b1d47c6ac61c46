"""Pins the CPU oracle to the reference (CPU suite, no GPU).

Each case's oracle run must reproduce, bit for bit, what the UNMODIFIED
reference produced when tests/golden/make_golden.py ran it: every
SimulationResult scalar, the phase labels, the full trace (TraceRecord +
TickHits), per-agent stats, and — where recorded — the hash of the per-event
state-digest sequence (cache + controller state after every event, taken
through the reference's paranoid-mode hooks).
"""
import json
import os

import pytest

from paper_2601_22705_b200 import engine
from tests.golden_cases import CASES, case_scenario
from tests.golden_hash import run_record
from tests.helpers import GOLDEN, load_presets, oracle_run

GOLD = json.load(open(os.path.join(GOLDEN, "reference_runs.json")))
# the 64-agent C2-shape LRU stall storm takes ~50 s in the oracle; it is
# checked against the same fixture on the GPU (tests/test_gpu_golden.py)
CPU_SKIP = {"c2s64_uncontrolled"}


@pytest.mark.parametrize("cid", [c["id"] for c in CASES if c["id"] not in CPU_SKIP])
def test_oracle_reproduces_reference(cid):
    case = next(c for c in CASES if c["id"] == cid)
    s, pol = case_scenario(case, load_presets())
    pop = engine.Population(s.workload, s.seed)  # bit-identical (test_population.py)
    run = oracle_run(s, pol, digests=case.get("digests", True), pop=pop.c)
    rec, gold = run_record(run), GOLD[cid]
    assert rec["status"] == gold["status"]
    assert rec["result"] == gold["result"]
    assert rec["n_trace"] == gold["n_trace"]
    assert rec["trace_sha"] == gold["trace_sha"]
    assert rec["agents_sha"] == gold["agents_sha"]
    if "digest_sha" in gold:
        assert rec["n_events"] == gold["n_events"]
        assert rec["digest_sha"] == gold["digest_sha"]
