"""Bindings used by the tests to drive the three implementations on identical
inputs: the reference (oracle/_ref/libkvref.so, unmodified reference sources),
the CPU restatement (oracle/libkvoracle.so) and the GPU engine (libkvgpu.so
through the package API). TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2601_22705_b200 import abi
from paper_2601_22705_b200.config import Scenario

REPO = abi.REPO_DIR
REF_SO = os.path.join(REPO, "oracle", "_ref", "libkvref.so")
ORACLE_SO = os.path.join(REPO, "oracle", "libkvoracle.so")
GOLDEN = os.path.join(REPO, "tests", "golden")

_ref = None
_orc = None


def ref_lib():
    global _ref
    if _ref is None:
        # RTLD_GLOBAL: the reference's iostream writers (export_trace & co.)
        # crash when libstdc++ arrives only as a dependency of a local library
        C.CDLL("libstdc++.so.6", mode=C.RTLD_GLOBAL)
        lib = C.CDLL(REF_SO)
        P = C.POINTER
        lib.kvr_last_error.restype = C.c_char_p
        lib.kvr_build_population.argtypes = [P(abi.WorkloadConfig), C.c_uint64,
                                             P(abi.StepPlan), C.c_size_t,
                                             P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]
        lib.kvr_run.argtypes = [P(abi.WorkloadConfig), C.c_uint64, P(abi.Policy),
                                P(abi.CostParams), P(abi.EngineParams), P(abi.SimResult),
                                P(abi.TraceRow), C.c_size_t, P(C.c_size_t),
                                P(abi.AgentStats), C.c_size_t,
                                P(C.c_uint64), C.c_size_t, P(C.c_size_t), P(C.c_double)]
        lib.kvr_run_many.argtypes = [C.c_size_t, P(abi.WorkloadConfig), P(C.c_uint64),
                                     P(abi.Policy), P(abi.CostParams), P(abi.EngineParams),
                                     C.c_uint, P(C.c_double), P(C.c_uint64), P(C.c_double)]
        lib.kvr_run_artifacts.argtypes = [P(abi.WorkloadConfig), C.c_uint64, P(abi.Policy),
                                          P(abi.CostParams), P(abi.EngineParams), C.c_char_p,
                                          C.c_char_p, C.c_char_p]
        lib.kvr_cache_new.restype = C.c_void_p
        lib.kvr_cache_new.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32]
        lib.kvr_cache_free.argtypes = [C.c_void_p]
        lib.kvr_cache_op.argtypes = [C.c_void_p, P(abi.CacheOp), P(abi.CacheOpResult),
                                     P(C.c_uint64), C.c_size_t, P(C.c_size_t)]
        lib.kvr_cache_stats.argtypes = [C.c_void_p, P(C.c_double), P(C.c_double),
                                        P(C.c_uint64), P(C.c_uint64)]
        lib.kvr_cache_digest.restype = C.c_uint64
        lib.kvr_cache_digest.argtypes = [C.c_void_p]
        lib.kvr_cache_check.argtypes = [C.c_void_p]
        _ref = lib
    return _ref


def _rows(arr, n):
    return [abi.struct_to_dict(arr[i]) for i in range(n)]


def ref_run(s: Scenario, policy_text: str | None = None, digests: bool = False,
            trace_cap: int = 1 << 16, dig_cap: int = 1 << 20):
    lib = ref_lib()
    pol, eng = s.resolved(policy_text)
    wl, cost, ep = s.workload.to_abi(), s.cost.to_abi(), eng.to_abi()
    res = abi.SimResult()
    for _ in range(4):
        trace = (abi.TraceRow * trace_cap)()
        agents = (abi.AgentStats * max(1, s.workload.agents))()
        dig = (C.c_uint64 * dig_cap)() if digests else None
        nt, nd, wall = C.c_size_t(), C.c_size_t(), C.c_double()
        rc = lib.kvr_run(C.byref(wl), s.seed, C.byref(pol), C.byref(cost), C.byref(ep),
                         C.byref(res), trace, trace_cap, C.byref(nt), agents,
                         s.workload.agents, dig, dig_cap if digests else 0,
                         C.byref(nd), C.byref(wall))
        if rc not in (abi.KVG_OK, abi.KVG_ERR_HORIZON):
            raise RuntimeError(f"reference failed ({rc}): {lib.kvr_last_error().decode()}")
        if nt.value <= trace_cap and (not digests or nd.value <= dig_cap):
            break
        trace_cap = max(trace_cap, nt.value)
        dig_cap = max(dig_cap, nd.value)
    return dict(status=rc, result=abi.struct_to_dict(res), trace=_rows(trace, nt.value),
                agents=_rows(agents, s.workload.agents),
                digests=np.ctypeslib.as_array(dig)[:nd.value].copy() if digests else None,
                wall=wall.value)


def ref_population(s: Scenario):
    lib = ref_lib()
    n = s.workload.agents * s.workload.steps
    plans = (abi.StepPlan * max(1, n))()
    h, sp, peak = C.c_uint64(), C.c_uint64(), C.c_uint64()
    wl = s.workload.to_abi()
    rc = lib.kvr_build_population(C.byref(wl), s.seed, plans, n, C.byref(h), C.byref(sp),
                                  C.byref(peak))
    assert rc == 0, lib.kvr_last_error()
    return plans, n, h.value, sp.value, peak.value


def oracle_lib():
    global _orc
    if _orc is None:
        lib = C.CDLL(ORACLE_SO)
        P = C.POINTER
        lib.kvo_last_error.restype = C.c_char_p
        lib.kvo_run.argtypes = [P(abi.SimDesc), P(abi.SimResult), P(abi.TraceRow), C.c_size_t,
                                P(C.c_size_t), P(abi.AgentStats), C.c_size_t, P(C.c_uint64),
                                C.c_size_t, P(C.c_size_t), P(abi.LogRecord), C.c_size_t,
                                P(C.c_size_t)]
        lib.kvo_cache_new.restype = C.c_void_p
        lib.kvo_cache_new.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32]
        lib.kvo_cache_free.argtypes = [C.c_void_p]
        lib.kvo_cache_op.argtypes = [C.c_void_p, P(abi.CacheOp), P(abi.CacheOpResult),
                                     P(abi.Victim), C.c_size_t, P(C.c_size_t)]
        lib.kvo_cache_stats.argtypes = [C.c_void_p, P(C.c_double), P(C.c_double), P(C.c_uint64)]
        lib.kvo_cache_digest.restype = C.c_uint64
        lib.kvo_cache_digest.argtypes = [C.c_void_p]
        _orc = lib
    return _orc


class RefPopulation:
    """A population built by the REFERENCE's build_population, held in an ABI
    struct (keeps the plan buffer alive)."""

    def __init__(self, s: Scenario):
        plans, n, h, sp, peak = ref_population(s)
        self.plans = plans
        self.pop = abi.Population(agents=s.workload.agents, steps=s.workload.steps,
                                  prompt_tokens=s.workload.prompt_tokens,
                                  shared_prompt=int(s.workload.shared_prompt),
                                  shared_prompt_tokens=sp, stream_hash=h,
                                  peak_aggregate_tokens=peak,
                                  plans=C.cast(plans, C.POINTER(abi.StepPlan)))


def make_desc(s: Scenario, pop: abi.Population, policy_text: str | None = None) -> abi.SimDesc:
    pol, eng = s.resolved(policy_text)
    return abi.SimDesc(population=C.pointer(pop), policy=pol, cost=s.cost.to_abi(),
                       engine=eng.to_abi())


def oracle_run(s: Scenario, policy_text: str | None = None, digests: bool = False,
               log: bool = False, pop: abi.Population | None = None):
    lib = oracle_lib()
    holder = None
    if pop is None:
        holder = RefPopulation(s)
        pop = holder.pop
    desc = make_desc(s, pop, policy_text)
    res = abi.SimResult()
    nt, nd, nl = C.c_size_t(), C.c_size_t(), C.c_size_t()
    d1 = (C.c_uint64 * 1)() if digests else None
    l1 = (abi.LogRecord * 1)() if log else None
    rc = lib.kvo_run(C.byref(desc), C.byref(res), None, 0, C.byref(nt), None, 0,
                     d1, 0, C.byref(nd), l1, 0, C.byref(nl))
    if rc not in (abi.KVG_OK, abi.KVG_ERR_HORIZON):
        raise RuntimeError(f"oracle failed ({rc}): {lib.kvo_last_error().decode()}")
    # second pass with exact buffers (the oracle is deterministic)
    trace = (abi.TraceRow * max(1, nt.value))()
    agents = (abi.AgentStats * max(1, s.workload.agents))()
    dig = (C.c_uint64 * max(1, nd.value))() if digests else None
    lg = (abi.LogRecord * max(1, nl.value))() if log else None
    rc = lib.kvo_run(C.byref(desc), C.byref(res), trace, nt.value, C.byref(nt), agents,
                     s.workload.agents, dig, nd.value if digests else 0, C.byref(nd),
                     lg, nl.value if log else 0, C.byref(nl))
    return dict(status=rc, result=abi.struct_to_dict(res), trace=_rows(trace, nt.value),
                agents=_rows(agents, s.workload.agents),
                digests=np.ctypeslib.as_array(dig)[:nd.value].copy() if digests else None,
                log=[(r.kind, r.agent, r.clock, r.a, r.b) for r in lg[:nl.value]] if log else None,
                raw_result=res, raw_trace=trace, n_trace=nt.value, raw_agents=agents)


def load_presets() -> dict:
    import json
    with open(os.path.join(GOLDEN, "scenarios.json")) as fh:
        return json.load(fh)


def ref_artifacts(s: Scenario, policy_text: str | None, out_dir: str, label: str):
    """The reference's own trace.csv / summary.txt / phases.csv for one run
    (execute_run's finalize through the unmodified metrics.cpp writers)."""
    lib = ref_lib()
    os.makedirs(out_dir, exist_ok=True)
    pol, eng = s.resolved(policy_text)
    wl, cost, ep = s.workload.to_abi(), s.cost.to_abi(), eng.to_abi()
    rc = lib.kvr_run_artifacts(C.byref(wl), s.seed, C.byref(pol), C.byref(cost), C.byref(ep),
                               s.name.encode(), label.encode(), out_dir.encode())
    assert rc == 0, lib.kvr_last_error()


def ref_run_many_out(scen: list, threads: int | None = None, stride: int = 4096):
    """The reference's run_simulation over many scenarios on host threads,
    with every output: [(status, result dict, trace rows, agent stats)], the
    arrays as numpy structured arrays in the ABI layouts."""
    lib = ref_lib()
    P = C.POINTER
    lib.kvr_run_many_out.argtypes = [C.c_size_t, P(abi.WorkloadConfig), P(C.c_uint64),
                                     P(abi.Policy), P(abi.CostParams), P(abi.EngineParams),
                                     C.c_uint, P(abi.SimResult), P(abi.TraceRow), C.c_size_t,
                                     P(C.c_size_t), P(abi.AgentStats), P(C.c_size_t)]
    n = len(scen)
    wls = (abi.WorkloadConfig * n)()
    seeds = (C.c_uint64 * n)()
    pols = (abi.Policy * n)()
    costs = (abi.CostParams * n)()
    engs = (abi.EngineParams * n)()
    aoff = (C.c_size_t * n)()
    na = 0
    for i, s in enumerate(scen):
        pol, eng = s.resolved()
        wls[i] = s.workload.to_abi()
        seeds[i] = s.seed
        pols[i] = pol
        costs[i] = s.cost.to_abi()
        engs[i] = eng.to_abi()
        aoff[i] = na
        na += s.workload.agents
    threads = threads or os.cpu_count() or 1
    while True:
        res = (abi.SimResult * n)()
        trace = np.zeros(n * stride, dtype=np.ctypeslib.as_array((abi.TraceRow * 1)()).dtype)
        agents = np.zeros(max(1, na), dtype=np.ctypeslib.as_array((abi.AgentStats * 1)()).dtype)
        nt = (C.c_size_t * n)()
        rc = lib.kvr_run_many_out(n, wls, seeds, pols, costs, engs, threads, res,
                                  trace.ctypes.data_as(P(abi.TraceRow)), stride, nt,
                                  agents.ctypes.data_as(P(abi.AgentStats)), aoff)
        if rc != 0:
            raise RuntimeError(lib.kvr_last_error().decode())
        mx = max(nt[i] for i in range(n))
        if mx <= stride:
            break
        stride = mx
    out = []
    for i, s in enumerate(scen):
        r = abi.struct_to_dict(res[i])
        out.append((r["status"], r, trace[i * stride: i * stride + nt[i]],
                    agents[aoff[i]: aoff[i] + s.workload.agents]))
    return out
