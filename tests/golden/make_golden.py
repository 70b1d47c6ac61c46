"""Generates the committed golden fixtures from the REFERENCE itself.

Run in the build container (needs /root/reference and oracle/_ref/libkvref.so):
    python tests/golden/make_golden.py

  scenarios.json       the reference presets (proj/configs/*.toml) parsed into
                       Scenario dicts, so tests on the GPU box need no /root/reference
  reference_runs.json  per case: every SimulationResult scalar (doubles as hex
                       bit patterns), a hash of the full trace, of the agent stats,
                       and of the per-event state-digest sequence (paranoid hooks)
  cache_fuzz.json      CacheTree differential sequences with the reference's
                       per-op results and ordered eviction victims
"""
import hashlib
import json
import os
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2601_22705_b200 import config  # noqa: E402
from tests.golden_cases import CASES, cache_fuzz_program, case_scenario  # noqa: E402
from tests.golden_hash import hx, run_record  # noqa: E402
from tests.helpers import ref_lib, ref_run  # noqa: E402
from paper_2601_22705_b200 import abi  # noqa: E402
import ctypes as C  # noqa: E402

PRESETS = "/root/reference/proj/configs"


def main():
    scen = {}
    for f in sorted(os.listdir(PRESETS)):
        if f.endswith(".toml"):
            scen[f[:-5]] = config.scenario_to_dict(config.load_scenario(os.path.join(PRESETS, f)))
    with open(os.path.join(HERE, "scenarios.json"), "w") as fh:
        json.dump(scen, fh, indent=1, sort_keys=True)
    runs = {}
    for case in CASES:
        s, pol = case_scenario(case, scen)
        r = ref_run(s, pol, digests=case.get("digests", True))
        runs[case["id"]] = run_record(r)
        print(case["id"], r["result"]["makespan"], len(r["trace"]))
    with open(os.path.join(HERE, "reference_runs.json"), "w") as fh:
        json.dump(runs, fh, indent=1, sort_keys=True)
    # CacheTree differential programs
    lib = ref_lib()
    fuzz = []
    for prog in cache_fuzz_program():
        h = lib.kvr_cache_new(prog["capacity"], prog["page_size"], 0, prog["prompt"], prog["shared"])
        outs, concrete = [], []
        vic = (C.c_uint64 * 65536)()
        last_match = {}
        pins = {}
        for (k, a, ln, arg) in prog["ops"]:
            if k == "PIN_LAST_MATCH":
                k, arg = 4, last_match.get(a, 0)
                pins.setdefault(a, []).append(arg)
            elif k == "DISCARD_IF_UNPINNED":
                if pins.get(a):
                    continue
                k = 6
            elif k == "UNPIN_ONE":
                if not pins.get(a):
                    continue
                L = pins[a].pop()
                k, ln, arg = 5, L, L
            op = abi.CacheOp(kind=k, agent=a, len=ln, arg=arg)
            res = abi.CacheOpResult()
            nv = C.c_size_t()
            rc = lib.kvr_cache_op(h, C.byref(op), C.byref(res), vic, 65536, C.byref(nv))
            assert rc == 0, (prog["seed"], k, a, ln, arg, lib.kvr_last_error())
            assert lib.kvr_cache_check(h) == 0, lib.kvr_last_error()
            if k == 1:
                last_match[a] = res.r0
            concrete.append([k, a, ln, arg])
            outs.append([rc, res.r0, res.r1, res.clock, res.used, list(vic[: nv.value])])
        # release outstanding pins so the program ends in a clean state
        for a, lst in pins.items():
            for L in lst:
                op = abi.CacheOp(kind=5, agent=a, len=L, arg=L)
                res = abi.CacheOpResult()
                nv = C.c_size_t()
                rc = lib.kvr_cache_op(h, C.byref(op), C.byref(res), vic, 65536, C.byref(nv))
                assert rc == 0
                concrete.append([5, a, L, L])
                outs.append([rc, res.r0, res.r1, res.clock, res.used, []])
        m, r = C.c_double(), C.c_double()
        lib.kvr_cache_stats(h, C.byref(m), C.byref(r), None, None)
        lib.kvr_cache_free(h)
        prog = dict(prog)
        prog["ops"] = concrete
        prog["expect"] = outs
        prog["hit"] = [hx(m.value), hx(r.value)]
        fuzz.append(prog)
    with open(os.path.join(HERE, "cache_fuzz.json"), "w") as fh:
        json.dump(fuzz, fh)
    print("cache programs:", len(fuzz), "ops:", sum(len(p["ops"]) for p in fuzz))


if __name__ == "__main__":
    main()
