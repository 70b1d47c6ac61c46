"""Generates the offload-mode golden fixtures from the REFERENCE itself.

Run in the build container (needs oracle/_ref/libkvref.so, built from the
unmodified /root/reference sources by oracle/Makefile):
    python tests/golden/make_golden_offload.py

  offload_runs.json        per case (tests/offload_cases.py): every
                           SimulationResult scalar, trace / agent-stat hashes,
                           the per-event state-digest hash, and how many events
                           ended in a Q1 state / with a corrupted
                           children_with_device counter
  offload_cache_fuzz.json  engine-style offload CacheTree programs (reload,
                           self-eviction) with the reference's per-op results
                           and ordered victims
"""
import ctypes as C
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2601_22705_b200 import abi  # noqa: E402
from tests.golden_hash import hx, run_record  # noqa: E402
from tests.helpers import load_presets, ref_lib, ref_run  # noqa: E402
from tests.offload_cases import OFFLOAD_CASES, offload_fuzz_programs, offload_scenario  # noqa: E402


def op(lib, h, kind, a, ln, arg=0, arg2=0):
    o = abi.CacheOp(kind=kind, agent=a, len=ln, arg=arg, arg2=arg2)
    res = abi.CacheOpResult()
    vic = (C.c_uint64 * 65536)()
    nv = C.c_size_t()
    rc = lib.kvr_cache_op(h, C.byref(o), C.byref(res), vic, 65536, C.byref(nv))
    return [rc, res.r0, res.r1, res.clock, res.used, list(vic[: nv.value])]


def fuzz(lib):
    out = []
    for prog in offload_fuzz_programs():
        h = lib.kvr_cache_new(prog["capacity"], prog["page_size"], abi.EVICT_OFFLOAD,
                              prog["prompt"], prog["shared"])
        ops, exp = [], []
        pinned = [0] * prog["agents"]
        lens = [prog["prompt"]] * prog["agents"]
        ps = prog["page_size"]

        def run(kind, a, ln, arg=0, arg2=0):
            r = op(lib, h, kind, a, ln, arg, arg2)
            assert r[0] == 0, (prog["seed"], kind, a, ln, arg, arg2, lib.kvr_last_error())
            ops.append([kind, a, ln, arg, arg2])
            exp.append(r)
            return r

        for (k, a, ln, arg) in prog["ops"]:
            if k == "STEP":  # dispatch_member, engine.cpp:337-396 (no token append)
                lens[a] = ln
                m, hm = run(abi.OP_MATCH, a, ln)[1:3]
                run(abi.OP_PIN, a, ln, m)
                if pinned[a]:
                    run(abi.OP_UNPIN, a, ln, pinned[a])
                pinned[a] = m
                if hm > 0:
                    promoted = run(abi.OP_RELOAD, a, ln, m, hm)[1]
                    if promoted > 0:
                        run(abi.OP_PIN, a, ln, m + promoted)
                        run(abi.OP_UNPIN, a, ln, m)
                        pinned[a] = m + promoted
                        continue
                ok = run(abi.OP_INSERT, a, ln)[1]
                if ok:
                    stored = ln // ps * ps
                    run(abi.OP_PIN, a, ln, stored)
                    run(abi.OP_UNPIN, a, ln, m)
                    pinned[a] = stored
                else:
                    run(abi.OP_UNPIN, a, ln, m)
                    pinned[a] = 0
            elif k == "RELEASE":
                if pinned[a]:
                    run(abi.OP_UNPIN, a, lens[a], pinned[a])
                    pinned[a] = 0
            elif k == "DISCARD_IF_UNPINNED":
                if not pinned[a]:
                    run(abi.OP_DISCARD, a, ln, arg)
            else:
                run(k, a, ln, arg)
        for a in range(prog["agents"]):
            if pinned[a]:
                run(abi.OP_UNPIN, a, lens[a], pinned[a])
        m, r = C.c_double(), C.c_double()
        off = C.c_uint64()
        lib.kvr_cache_stats(h, C.byref(m), C.byref(r), None, C.byref(off))
        lib.kvr_cache_free(h)
        p = {k: v for k, v in prog.items() if k != "ops"}
        p.update(ops=ops, expect=exp, hit=[hx(m.value), hx(r.value)], offloaded=off.value)
        out.append(p)
    return out


def main():
    lib = ref_lib()
    lib.kvr_last_q1_states.restype = C.c_uint64
    lib.kvr_last_cwd_states.restype = C.c_uint64
    presets = load_presets()
    runs = {}
    for case in OFFLOAD_CASES:
        s, pol = offload_scenario(case, presets)
        t0 = time.time()
        r = ref_run(s, pol, digests=True)
        rec = run_record(r)
        rec["q1_states"] = lib.kvr_last_q1_states()
        rec["cwd_states"] = lib.kvr_last_cwd_states()
        runs[case["id"]] = rec
        print(case["id"], r["result"]["makespan"], rec["n_events"], rec["q1_states"],
              rec["cwd_states"], f"{time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(HERE, "offload_runs.json"), "w") as fh:
        json.dump(runs, fh, indent=1, sort_keys=True)
    progs = fuzz(lib)
    with open(os.path.join(HERE, "offload_cache_fuzz.json"), "w") as fh:
        json.dump(progs, fh)
    print("offload cache programs:", len(progs), "ops:", sum(len(p["ops"]) for p in progs))


if __name__ == "__main__":
    main()
