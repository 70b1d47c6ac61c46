"""Pins the offload-mode oracle (node-level TreeCache, oracle/kvoracle.cpp) to
the unmodified reference (CPU suite, no GPU).

Every case must reproduce bit for bit what the reference produced when
tests/golden/make_golden_offload.py ran it — results, trace, agent stats and
the hash of the per-event state digests — through thousands of quirk-Q1
states (device node below a host node) and corrupted children_with_device
counters (cache_tree.cpp:94-102, 321-368). The cache-level
programs replay engine-style match/pin/reload/insert sequences with the
reference's ordered victim lists."""
import ctypes as C
import json
import os

import pytest

from paper_2601_22705_b200 import abi, engine
from tests.golden_hash import hx, run_record
from tests.helpers import GOLDEN, load_presets, oracle_lib, oracle_run
from tests.offload_cases import OFFLOAD_CASES, offload_scenario

GOLD = json.load(open(os.path.join(GOLDEN, "offload_runs.json")))
PROGS = json.load(open(os.path.join(GOLDEN, "offload_cache_fuzz.json")))
SLOW = {"off_c3s64"}  # ~25 s in the oracle: GPU suite checks it against the same fixture


@pytest.mark.parametrize("cid", [c["id"] for c in OFFLOAD_CASES if c["id"] not in SLOW])
def test_oracle_offload_reproduces_reference(cid):
    case = next(c for c in OFFLOAD_CASES if c["id"] == cid)
    s, pol = offload_scenario(case, load_presets())
    pop = engine.Population(s.workload, s.seed)
    run = oracle_run(s, pol, digests=True, pop=pop.c)
    rec, gold = run_record(run), GOLD[cid]
    assert rec["status"] == gold["status"]
    assert rec["result"] == gold["result"]
    assert rec["trace_sha"] == gold["trace_sha"]
    assert rec["agents_sha"] == gold["agents_sha"]
    assert rec["n_events"] == gold["n_events"]
    assert rec["digest_sha"] == gold["digest_sha"]


def test_offload_fixtures_exercise_the_quirks():
    assert sum(g["q1_states"] for g in GOLD.values()) > 10000
    assert sum(g["cwd_states"] for g in GOLD.values()) > 10000


@pytest.mark.parametrize("k", range(len(PROGS)))
def test_oracle_offload_cache_program(k):
    prog = PROGS[k]
    lib = oracle_lib()
    h = lib.kvo_cache_new(prog["capacity"], prog["page_size"], abi.EVICT_OFFLOAD, prog["prompt"],
                          prog["shared"])
    assert h
    vic = (abi.Victim * 65536)()
    try:
        for (kind, a, ln, arg, arg2), exp in zip(prog["ops"], prog["expect"]):
            op = abi.CacheOp(kind=kind, agent=a, len=ln, arg=arg, arg2=arg2)
            res = abi.CacheOpResult()
            nv = C.c_size_t()
            rc = lib.kvo_cache_op(h, C.byref(op), C.byref(res), vic, 65536, C.byref(nv))
            got = [rc, res.r0, res.r1, res.clock, res.used, [vic[i].key for i in range(nv.value)]]
            assert got == exp, (kind, a, ln, arg, arg2)
        m, r = C.c_double(), C.c_double()
        lib.kvo_cache_stats(h, C.byref(m), C.byref(r), None)
        assert [hx(m.value), hx(r.value)] == prog["hit"]
    finally:
        lib.kvo_cache_free(h)
