"""The device CacheTree seam (kvg_cache_*) against the reference CacheTree's
recorded behaviour: 40 randomized programs / 13K ops (tests/golden/
cache_fuzz.json): match and insert results, clock, pool usage and the exact
ordered victim list of every eviction."""
import json
import os

import pytest

from paper_2601_22705_b200 import engine
from tests.golden_hash import hx
from tests.helpers import GOLDEN

pytestmark = pytest.mark.gpu
PROGS = json.load(open(os.path.join(GOLDEN, "cache_fuzz.json")))


@pytest.mark.parametrize("k", range(len(PROGS)))
def test_device_cache_program(k):
    prog = PROGS[k]
    c = engine.DeviceCache(prog["capacity"], prog["page_size"], prog["prompt"],
                           bool(prog["shared"]), max_agents=prog["agents"])
    try:
        out = c.execute([tuple(op) for op in prog["ops"]])
        for (kind, a, ln, arg), exp, got in zip(prog["ops"], prog["expect"], out):
            g = [got["status"], got["r0"], got["r1"], got["clock"], got["used"], got["victims"]]
            assert g == exp, (kind, a, ln, arg)
        m, r = c.hit_window()
        assert [hx(m), hx(r)] == prog["hit"]
    finally:
        c.close()


def test_device_cache_op_by_op_equals_batched():
    prog = PROGS[3]
    c1 = engine.DeviceCache(prog["capacity"], prog["page_size"], prog["prompt"],
                            bool(prog["shared"]), max_agents=prog["agents"])
    c2 = engine.DeviceCache(prog["capacity"], prog["page_size"], prog["prompt"],
                            bool(prog["shared"]), max_agents=prog["agents"])
    batched = c1.execute([tuple(op) for op in prog["ops"]])
    single = [c2.execute([tuple(op)])[0] for op in prog["ops"]]
    assert [(x["r0"], x["clock"], x["used"], x["victims"]) for x in batched] == \
        [(x["r0"], x["clock"], x["used"], x["victims"]) for x in single]


OFF = json.load(open(os.path.join(GOLDEN, "offload_cache_fuzz.json")))


@pytest.mark.parametrize("k", range(len(OFF)))
def test_device_offload_cache_program(k):
    """Offload-mode seam (node-level tree on the device) against the
    reference's engine-style reload programs (tests/golden/
    offload_cache_fuzz.json): match / host_matched, reload promotions and the
    offloaded tokens their evictions push, inserts, ordered victims."""
    from paper_2601_22705_b200 import abi
    prog = OFF[k]
    c = engine.DeviceCache(prog["capacity"], prog["page_size"], prog["prompt"],
                           bool(prog["shared"]), max_agents=prog["agents"],
                           eviction=abi.EVICT_OFFLOAD)
    try:
        out = c.execute([tuple(op) for op in prog["ops"]])
        for op, exp, got in zip(prog["ops"], prog["expect"], out):
            g = [got["status"], got["r0"], got["r1"], got["clock"], got["used"], got["victims"]]
            assert g == exp, op
        m, r = c.hit_window()
        assert [hx(m), hx(r)] == prog["hit"]
    finally:
        c.close()
