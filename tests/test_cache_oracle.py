"""CacheTree-level differential: the oracle's flat per-page cache against the
reference CacheTree's recorded behaviour (tests/golden/cache_fuzz.json) over
40 randomized programs, 13K ops: match/insert results, clock, pool usage and
the ordered eviction victim list of every op (acceptance criterion 2 style,
acceptance.cpp:133-209; test_cache_tree.cpp:276-340)."""
import ctypes as C
import json
import os

import pytest

from paper_2601_22705_b200 import abi
from tests.golden_hash import hx
from tests.helpers import GOLDEN, oracle_lib

PROGS = json.load(open(os.path.join(GOLDEN, "cache_fuzz.json")))


@pytest.mark.parametrize("k", range(len(PROGS)))
def test_oracle_cache_program(k):
    prog = PROGS[k]
    lib = oracle_lib()
    h = lib.kvo_cache_new(prog["capacity"], prog["page_size"], 0, prog["prompt"], prog["shared"])
    assert h
    vic = (abi.Victim * 65536)()
    try:
        for (kind, a, ln, arg), exp in zip(prog["ops"], prog["expect"]):
            op = abi.CacheOp(kind=kind, agent=a, len=ln, arg=arg)
            res = abi.CacheOpResult()
            nv = C.c_size_t()
            rc = lib.kvo_cache_op(h, C.byref(op), C.byref(res), vic, 65536, C.byref(nv))
            got = [rc, res.r0, res.r1, res.clock, res.used, [vic[i].key for i in range(nv.value)]]
            assert got == exp, (kind, a, ln, arg)
        m, r = C.c_double(), C.c_double()
        lib.kvo_cache_stats(h, C.byref(m), C.byref(r), None)
        assert [hx(m.value), hx(r.value)] == prog["hit"]
    finally:
        lib.kvo_cache_free(h)
