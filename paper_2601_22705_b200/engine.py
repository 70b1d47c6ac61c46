"""Python mirror of the reference hot-path seam, over the C ABI (libkvgpu.so).

    run_simulation(population, policy, cost, params)   ~ engine.hpp:75-78
    build_population(workload, seed)                   ~ workload.hpp:128
    Batch([...]).run()                                  ~ run_rows (experiment.cpp:75-108)
    DeviceCache(...)                                    ~ CacheTree (cache_tree.hpp:94-198)

The library is the product: there is no CPU fallback. Loading fails loudly if
libkvgpu.so is missing, and every compute call fails with KVG_ERR_CUDA when no
GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import abi
from .config import Scenario

_lib = None
_RESULT_DTYPE = None


class EngineError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{abi.STATUS_NAMES.get(status, status)}] {msg}")
        self.status = status


class HorizonError(EngineError):
    """Simulated time exceeded the horizon (errors.hpp:33-36); partial results kept."""


def lib():
    """Loads libkvgpu.so (build it with `python -m paper_2601_22705_b200.build`)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(abi.LIB_PATH):
        raise ImportError(f"{abi.LIB_PATH} is missing: the B200 engine has no CPU fallback; "
                          "run `python -m paper_2601_22705_b200.build`")
    L = C.CDLL(abi.LIB_PATH)
    P = C.POINTER
    L.kvg_version.restype = C.c_char_p
    L.kvg_last_error.restype = C.c_char_p
    L.kvg_build_population.argtypes = [P(abi.WorkloadConfig), C.c_uint64, P(abi.Population)]
    L.kvg_population_free.argtypes = [P(abi.Population)]
    L.kvg_population_free.restype = None
    L.kvg_cost_params_init.argtypes = [P(abi.CostParams)]
    L.kvg_controller_config_init.argtypes = [P(abi.ControllerConfig)]
    L.kvg_engine_params_init.argtypes = [P(abi.EngineParams)]
    L.kvg_batch_options_init.argtypes = [P(abi.BatchOptions)]
    L.kvg_batch_create.argtypes = [C.c_int, P(abi.SimDesc), C.c_size_t, P(abi.BatchOptions),
                                   P(C.c_void_p)]
    L.kvg_batch_run.argtypes = [C.c_void_p]
    L.kvg_batch_launch.argtypes = [C.c_void_p]
    L.kvg_batch_wait.argtypes = [C.c_void_p]
    L.kvg_batch_last_ms.argtypes = [C.c_void_p, P(C.c_double)]
    L.kvg_batch_timing.argtypes = [C.c_void_p, P(C.c_double), P(C.c_double)]
    L.kvg_batch_geometry.argtypes = [C.c_void_p, P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
    L.kvg_batch_result.argtypes = [C.c_void_p, C.c_size_t, P(abi.SimResult)]
    L.kvg_batch_trace.argtypes = [C.c_void_p, C.c_size_t, P(abi.TraceRow), C.c_size_t,
                                  P(C.c_size_t)]
    L.kvg_batch_agent_stats.argtypes = [C.c_void_p, C.c_size_t, P(abi.AgentStats), C.c_size_t,
                                        P(C.c_size_t)]
    L.kvg_batch_log.argtypes = [C.c_void_p, C.c_size_t, P(abi.LogRecord), C.c_size_t,
                                P(C.c_size_t)]
    L.kvg_batch_results.argtypes = [C.c_void_p, P(abi.SimResult), C.c_size_t]
    L.kvg_batch_outputs.argtypes = [C.c_void_p, P(P(abi.SimResult)), P(P(abi.TraceRow)),
                                    P(P(abi.AgentStats))]
    L.kvg_batch_offsets.argtypes = [C.c_void_p, C.c_size_t, P(C.c_size_t), P(C.c_size_t)]
    L.kvg_batch_trace_view.argtypes = [C.c_void_p, C.c_size_t, P(P(abi.TraceRow)),
                                       P(C.c_size_t)]
    L.kvg_batch_free.argtypes = [C.c_void_p]
    L.kvg_batch_free.restype = None
    L.kvg_run_batch.argtypes = [C.c_int, P(abi.SimDesc), C.c_size_t, P(abi.SimResult)]
    L.kvg_classify_phases.argtypes = [P(abi.TraceRow), C.c_size_t, C.c_double,
                                      P(abi.PhaseParams), P(abi.PhaseLabel), C.c_size_t,
                                      P(C.c_size_t)]
    L.kvg_policy_name.argtypes = [P(abi.Policy), C.c_char_p, C.c_size_t]
    L.kvg_summarize.argtypes = [P(abi.SimResult), P(abi.TraceRow), C.c_size_t, C.c_char_p,
                                C.c_char_p, C.c_uint64, C.c_uint32, P(abi.Summary)]
    L.kvg_write_run_artifacts.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint64,
                                          C.c_uint32, P(abi.SimResult), P(abi.TraceRow),
                                          C.c_size_t, P(abi.Summary)]
    L.kvg_controllers_create.argtypes = [C.c_int, C.c_size_t, P(abi.Policy), P(C.c_uint32),
                                         P(C.c_void_p)]
    L.kvg_controllers_free.argtypes = [C.c_void_p]
    L.kvg_controllers_free.restype = None
    L.kvg_controllers_update_window.argtypes = [C.c_void_p, P(C.c_double), P(C.c_double),
                                                P(C.c_double)]
    L.kvg_controllers_admission_pass.argtypes = [C.c_void_p, P(C.c_uint8), P(abi.Command),
                                                 P(C.c_size_t), P(C.c_int32)]
    L.kvg_controllers_apply.argtypes = [C.c_void_p, P(abi.CtlEvent), C.c_size_t, P(C.c_int32)]
    L.kvg_controllers_state.argtypes = [C.c_void_p, P(C.c_double), P(C.c_double),
                                        P(C.c_uint64), P(C.c_size_t), P(C.c_size_t),
                                        P(C.c_size_t)]
    L.kvg_controllers_active.argtypes = [C.c_void_p, C.c_size_t, P(C.c_uint32), C.c_size_t,
                                         P(C.c_size_t)]
    L.kvg_cache_create.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64,
                                   C.c_uint32, C.c_uint32, P(C.c_void_p)]
    L.kvg_cache_exec.argtypes = [C.c_void_p, P(abi.CacheOp), C.c_size_t, P(abi.CacheOpResult)]
    L.kvg_cache_victims.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, P(abi.Victim)]
    L.kvg_cache_hit_window.argtypes = [C.c_void_p, P(C.c_double), P(C.c_double)]
    L.kvg_cache_free.argtypes = [C.c_void_p]
    L.kvg_cache_free.restype = None
    L.kvg_cache_configure.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
    L.kvg_cache_match_batch.argtypes = [C.c_void_p, P(C.c_uint32), P(C.c_uint64), C.c_size_t,
                                        P(abi.CacheOpResult)]
    L.kvg_cache_last_ms.argtypes = [C.c_void_p, P(C.c_double), P(C.c_uint32)]
    _lib = L
    return L


def _check(status: int, allow_horizon: bool = False):
    if status == abi.KVG_OK or (allow_horizon and status == abi.KVG_ERR_HORIZON):
        return status
    msg = lib().kvg_last_error().decode()
    if status == abi.KVG_ERR_HORIZON:
        raise HorizonError(status, msg)
    raise EngineError(status, msg)


class Population:
    """Owning wrapper of kvg_population built by the library (bit-identical to
    the reference's build_population, workload.cpp:153-204)."""

    def __init__(self, workload, seed: int):
        self.c = abi.Population()
        wl = workload.to_abi() if hasattr(workload, "to_abi") else workload
        _check(lib().kvg_build_population(C.byref(wl), int(seed), C.byref(self.c)))

    @property
    def stream_hash(self) -> int:
        return self.c.stream_hash

    @property
    def peak_aggregate_tokens(self) -> int:
        return self.c.peak_aggregate_tokens

    def plans(self) -> np.ndarray:
        n = self.c.agents * self.c.steps
        if n == 0:
            return np.zeros((0,), dtype=np.uint8)
        buf = C.cast(self.c.plans, C.POINTER(C.c_uint8 * (n * C.sizeof(abi.StepPlan)))).contents
        return np.frombuffer(buf, dtype=np.uint8).copy()

    def __del__(self):
        if _lib is not None and getattr(self, "c", None) is not None and self.c.plans:
            _lib.kvg_population_free(C.byref(self.c))


def build_population(workload, seed: int) -> Population:
    return Population(workload, seed)


@dataclass
class SimSpec:
    """One simulation: a population plus policy / cost / engine parameters."""
    population: Population
    policy: abi.Policy
    cost: abi.CostParams
    engine: abi.EngineParams

    @property
    def desc(self) -> abi.SimDesc:
        """The C descriptor of this simulation (built once, cached)."""
        d = self.__dict__.get("_desc")
        if d is None:
            d = abi.SimDesc(population=C.pointer(self.population.c), policy=self.policy,
                            cost=self.cost, engine=self.engine)
            self.__dict__["_desc"] = d
        return d

    @property
    def desc_bytes(self) -> bytes:
        """The descriptor's bytes (cached): batches pack them with one join."""
        b = self.__dict__.get("_desc_bytes")
        if b is None:
            b = bytes(self.desc)
            self.__dict__["_desc_bytes"] = b
        return b

    @staticmethod
    def from_scenario(s: Scenario, policy_text: str | None = None,
                      population: Population | None = None) -> "SimSpec":
        pol, eng = s.resolved(policy_text)
        pop = population if population is not None else Population(s.workload, s.seed)
        return SimSpec(pop, pol, s.cost.to_abi(), eng.to_abi())


HOST_OUTPUTS_COPY = 2


class Batch:
    """A set of independent simulations executed on one GPU in one launch."""

    def __init__(self, specs: list[SimSpec], device: int = 0, warps_per_sim: int = 0,
                 log_capacity: int = 0, trace_capacity: int = 0, host_outputs: bool | int = False,
                 verify: bool | None = None):
        """host_outputs: False / 0 outputs stay in HBM; True / 1 delivered to
        pinned host memory by run() / wait(), trace rows streamed by the kernel;
        2 (HOST_OUTPUTS_COPY) the same with the rows copied by one DMA after
        the kernel (for pipelined launch / wait).
        verify: re-derive every prefix match with the block-hash probe and
        check it against the incrementally held state (default: the
        KVG_VERIFY environment variable; the GPU test suite sets it)."""
        if verify is None:
            verify = os.environ.get("KVG_VERIFY", "0") == "1"
        self.specs = specs
        if specs:
            # the descriptors hold pointers into the specs' populations, which
            # self.specs keeps alive
            self.descs = (abi.SimDesc * len(specs)).from_buffer_copy(
                b"".join([sp.desc_bytes for sp in specs]))
        else:
            self.descs = (abi.SimDesc * 1)()
        opt = abi.BatchOptions(warps_per_sim=warps_per_sim, log_capacity=log_capacity,
                               trace_capacity=trace_capacity, host_outputs=int(host_outputs),
                               verify=int(bool(verify)))
        h = C.c_void_p()
        _check(lib().kvg_batch_create(device, self.descs, len(specs), C.byref(opt), C.byref(h)))
        self.h = h
        self.n = len(specs)

    def run(self, allow_horizon: bool = True) -> int:
        return _check(lib().kvg_batch_run(self.h), allow_horizon=allow_horizon)

    def launch(self) -> None:
        """First half of run(): enqueue on the batch's stream, return at once."""
        _check(lib().kvg_batch_launch(self.h))

    def wait(self, allow_horizon: bool = True) -> int:
        """Second half of run(): block until the launch ends, deliver results."""
        return _check(lib().kvg_batch_wait(self.h), allow_horizon=allow_horizon)

    def last_ms(self) -> float:
        v = C.c_double()
        _check(lib().kvg_batch_last_ms(self.h, C.byref(v)))
        return v.value

    def timing(self) -> tuple[float, float]:
        """(step_ms, kernel_ms) of the last run, CUDA events on the launch stream."""
        a, k = C.c_double(), C.c_double()
        _check(lib().kvg_batch_timing(self.h, C.byref(a), C.byref(k)))
        return a.value, k.value

    def geometry(self) -> dict:
        """One-warp kernel geometry: small simulations, CTAs per SM at this
        batch's shared memory (CUDA occupancy calculator), SM count, waves."""
        n, occ, sms = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib().kvg_batch_geometry(self.h, C.byref(n), C.byref(occ), C.byref(sms)))
        slots = occ.value * sms.value
        waves = -(-n.value // slots) if slots else 0
        return {"small_sims": n.value, "ctas_per_sm": occ.value, "sms": sms.value, "waves": waves}

    def result(self, i: int) -> dict:
        r = abi.SimResult()
        _check(lib().kvg_batch_result(self.h, i, C.byref(r)))
        return abi.struct_to_dict(r)

    def results_raw(self) -> list[abi.SimResult]:
        arr = (abi.SimResult * max(1, self.n))()
        _check(lib().kvg_batch_results(self.h, arr, self.n))
        return list(arr)[: self.n]

    def results_array(self) -> np.ndarray:
        """Every simulation's result as one numpy structured array (no
        per-simulation Python objects; the dtype is built once)."""
        global _RESULT_DTYPE
        if _RESULT_DTYPE is None:
            _RESULT_DTYPE = np.ctypeslib.as_array((abi.SimResult * 1)()).dtype
        out = np.empty(max(1, self.n), dtype=_RESULT_DTYPE)
        _check(lib().kvg_batch_results(self.h, out.ctypes.data_as(C.POINTER(abi.SimResult)),
                                       self.n))
        return out[: self.n]

    def outputs(self):
        """Zero-copy numpy views of the host output block: (results[n],
        [agent-stats slice per simulation], [trace-row slice per simulation])."""
        r, t, st = C.POINTER(abi.SimResult)(), C.POINTER(abi.TraceRow)(), \
            C.POINTER(abi.AgentStats)()
        _check(lib().kvg_batch_outputs(self.h, C.byref(r), C.byref(t), C.byref(st)))
        res = np.ctypeslib.as_array(r, shape=(max(1, self.n),))[: self.n]
        stats, rows = [], []
        for i in range(self.n):
            si, ti = C.c_size_t(), C.c_size_t()
            _check(lib().kvg_batch_offsets(self.h, i, C.byref(si), C.byref(ti)))
            na = self.specs[i].population.c.agents
            stats.append(np.ctypeslib.as_array(
                C.cast(C.byref(st.contents, si.value * C.sizeof(abi.AgentStats)),
                       C.POINTER(abi.AgentStats)), shape=(max(1, na),))[:na])
            p, nt = C.POINTER(abi.TraceRow)(), C.c_size_t()
            _check(lib().kvg_batch_trace_view(self.h, i, C.byref(p), C.byref(nt)))
            view = C.cast(C.byref(t.contents, ti.value * C.sizeof(abi.TraceRow)),
                          C.POINTER(abi.TraceRow))
            assert C.addressof(view.contents) == C.addressof(p.contents) or nt.value == 0
            rows.append(np.ctypeslib.as_array(view, shape=(max(1, nt.value),))[:nt.value])
        return res, stats, rows

    def trace(self, i: int) -> list[dict]:
        n = C.c_size_t()
        _check(lib().kvg_batch_trace(self.h, i, None, 0, C.byref(n)))
        rows = (abi.TraceRow * max(1, n.value))()
        _check(lib().kvg_batch_trace(self.h, i, rows, n.value, C.byref(n)))
        return [abi.struct_to_dict(rows[k]) for k in range(n.value)]

    def trace_array(self, i: int) -> np.ndarray:
        """Simulation i's trace rows (one copy out of the host block)."""
        p, n = C.POINTER(abi.TraceRow)(), C.c_size_t()
        _check(lib().kvg_batch_trace_view(self.h, i, C.byref(p), C.byref(n)))
        if n.value == 0:
            return np.ctypeslib.as_array((abi.TraceRow * 1)())[:0]
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy()

    def agent_stats(self, i: int) -> list[dict]:
        na = self.specs[i].population.c.agents
        out = (abi.AgentStats * max(1, na))()
        n = C.c_size_t()
        _check(lib().kvg_batch_agent_stats(self.h, i, out, na, C.byref(n)))
        return [abi.struct_to_dict(out[k]) for k in range(na)]

    def log(self, i: int) -> list[tuple]:
        n = C.c_size_t()
        _check(lib().kvg_batch_log(self.h, i, None, 0, C.byref(n)))
        recs = (abi.LogRecord * max(1, n.value))()
        _check(lib().kvg_batch_log(self.h, i, recs, n.value, C.byref(n)))
        return [(r.kind, r.agent, r.clock, r.a, r.b) for r in recs[: n.value]]

    def write_artifacts(self, i: int, out_dir: str, name: str, policy_label: str,
                        seed: int) -> dict:
        """trace.csv, summary.txt and phases.csv of simulation i in `out_dir`,
        byte-identical to the reference's execute_run (experiment.cpp:161-170).
        Returns the Summary."""
        os.makedirs(out_dir, exist_ok=True)
        r = abi.SimResult()
        _check(lib().kvg_batch_result(self.h, i, C.byref(r)))
        n = C.c_size_t()
        _check(lib().kvg_batch_trace(self.h, i, None, 0, C.byref(n)))
        rows = (abi.TraceRow * max(1, n.value))()
        _check(lib().kvg_batch_trace(self.h, i, rows, n.value, C.byref(n)))
        s = abi.Summary()
        _check(lib().kvg_write_run_artifacts(out_dir.encode(), name.encode(),
                                             policy_label.encode(), seed,
                                             self.specs[i].population.c.agents, C.byref(r),
                                             rows, n.value, C.byref(s)))
        return abi.struct_to_dict(s)

    def close(self):
        if getattr(self, "h", None):
            lib().kvg_batch_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_simulation(population: Population, policy: abi.Policy, cost: abi.CostParams,
                   params: abi.EngineParams, device: int = 0) -> dict:
    """Mirror of kvadmit::run_simulation: one simulation, full result.
    Raises HorizonError (with .partial) when the horizon guard trips."""
    b = Batch([SimSpec(population, policy, cost, params)], device=device)
    st = b.run(allow_horizon=True)
    out = dict(result=b.result(0), trace=b.trace(0), agents=b.agent_stats(0))
    b.close()
    if st == abi.KVG_ERR_HORIZON:
        e = HorizonError(st, "simulated time exceeded the horizon")
        e.partial = out
        raise e
    return out


class DeviceCache:
    """Device-resident paged prefix cache driven through CacheTree-style ops."""

    def __init__(self, capacity: int, page_size: int = 1, prompt_tokens: int = 0,
                 shared_prompt: bool = False, max_agents: int = 64, device: int = 0,
                 eviction: int = abi.EVICT_DISCARD):
        h = C.c_void_p()
        _check(lib().kvg_cache_create(device, capacity, page_size, eviction,
                                      prompt_tokens, int(shared_prompt), max_agents,
                                      C.byref(h)))
        self.h = h

    def execute(self, ops: list[tuple]) -> list[dict]:
        """ops: (kind, agent, len, arg). Returns per-op results incl. victims
        ordered as the reference evicts them."""
        n = len(ops)
        arr = (abi.CacheOp * max(1, n))()
        for i, op in enumerate(ops):
            k, a, ln, arg = op[:4]
            arr[i] = abi.CacheOp(kind=k, agent=a, len=ln, arg=arg, arg2=op[4] if len(op) > 4 else 0)
        res = (abi.CacheOpResult * max(1, n))()
        _check(lib().kvg_cache_exec(self.h, arr, n, res))
        out = []
        for i in range(n):
            r = res[i]
            nv = r.victims_end - r.victims_begin
            vic = (abi.Victim * max(1, nv))()
            if nv:
                _check(lib().kvg_cache_victims(self.h, r.victims_begin, r.victims_end, vic))
            out.append(dict(status=r.status, r0=r.r0, r1=r.r1, clock=r.clock, used=r.used,
                            victims=[vic[j].key for j in range(nv)],
                            vrange=(r.victims_begin, r.victims_end)))
        return out

    def victim_stamps(self, res: dict) -> list[int]:
        """Last-access stamps of one op result's victims, in victim order."""
        b, e = res["vrange"]
        vic = (abi.Victim * max(1, e - b))()
        if e > b:
            _check(lib().kvg_cache_victims(self.h, b, e, vic))
        return [vic[j].stamp for j in range(e - b)]

    def hit_window(self):
        m, r = C.c_double(), C.c_double()
        _check(lib().kvg_cache_hit_window(self.h, C.byref(m), C.byref(r)))
        return m.value, r.value

    def configure(self, grid_mode: int = 0, record_victims: bool = True):
        """grid_mode: 0 auto (EVICT grid-wide on big tables), 1 never, 2 always."""
        _check(lib().kvg_cache_configure(self.h, grid_mode, int(record_victims)))

    def match_batch(self, agents, lens) -> list[dict]:
        """n match_prefix calls in one grid launch (== n KVG_OP_MATCH ops)."""
        import numpy as np
        a = np.ascontiguousarray(agents, dtype=np.uint32)
        ln = np.ascontiguousarray(lens, dtype=np.uint64)
        n = len(a)
        res = (abi.CacheOpResult * max(1, n))()
        _check(lib().kvg_cache_match_batch(self.h, a.ctypes.data_as(C.POINTER(C.c_uint32)),
                                           ln.ctypes.data_as(C.POINTER(C.c_uint64)), n, res))
        return [dict(status=res[i].status, r0=res[i].r0, r1=res[i].r1, clock=res[i].clock,
                     used=res[i].used, victims=[]) for i in range(n)]

    def last_ms(self):
        ms, blocks = C.c_double(), C.c_uint32()
        _check(lib().kvg_cache_last_ms(self.h, C.byref(ms), C.byref(blocks)))
        return ms.value, blocks.value

    def close(self):
        if getattr(self, "h", None):
            lib().kvg_cache_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceControllers:
    """N admission controllers with their state in HBM: the reference's
    standalone controller ABI (kvadmit.h:86-159) batched, one kernel per call
    over all controllers (csrc/controllers.cu)."""

    def __init__(self, policies: list, total_agents: list[int], device: int = 0):
        n = len(policies)
        self.n = n
        self.total = list(total_agents)
        self.off = [0]
        for t in self.total:
            self.off.append(self.off[-1] + t)
        pol = (abi.Policy * max(1, n))(*policies)
        tot = (C.c_uint32 * max(1, n))(*self.total)
        h = C.c_void_p()
        _check(lib().kvg_controllers_create(device, n, pol, tot, C.byref(h)))
        self.h = h

    def update_window(self, usage: list[float], hit: list[float]) -> list[float]:
        u = (C.c_double * max(1, self.n))(*usage)
        r = (C.c_double * max(1, self.n))(*hit)
        w = (C.c_double * max(1, self.n))()
        _check(lib().kvg_controllers_update_window(self.h, u, r, w))
        return list(w)[: self.n]

    def admission_pass(self, at_boundary: list[list[bool]], statuses: list | None = None
                       ) -> list[list[tuple[int, int]]]:
        """Commands per controller. A controller whose pass emitted more
        commands than agents (API misuse) reports status KVG_ERR_STATE in
        `statuses` and no commands."""
        flat = [int(b) for row in at_boundary for b in row]
        bnd = (C.c_uint8 * max(1, len(flat)))(*flat)
        cmds = (abi.Command * max(1, self.off[-1]))()
        nout = (C.c_size_t * max(1, self.n))()
        st = (C.c_int32 * max(1, self.n))()
        rc = lib().kvg_controllers_admission_pass(self.h, bnd, cmds, nout, st)
        if rc not in (abi.KVG_OK, abi.KVG_ERR_STATE):
            _check(rc)
        if statuses is not None:
            statuses[:] = list(st)[: self.n]
        return [[(cmds[self.off[i] + k].kind, cmds[self.off[i] + k].agent)
                 for k in range(nout[i])] for i in range(self.n)]

    def apply(self, events: list[tuple[int, int, int]]) -> list[int]:
        """events: (controller, kind, agent); returns per-event statuses."""
        ev = (abi.CtlEvent * max(1, len(events)))(
            *[abi.CtlEvent(controller=c, kind=k, agent=a) for c, k, a in events])
        st = (C.c_int32 * max(1, len(events)))()
        lib().kvg_controllers_apply(self.h, ev, len(events), st)
        return list(st)[: len(events)]

    def state(self) -> list[dict]:
        n = max(1, self.n)
        w, dw = (C.c_double * n)(), (C.c_double * n)()
        t = (C.c_uint64 * n)()
        a, p, q = (C.c_size_t * n)(), (C.c_size_t * n)(), (C.c_size_t * n)()
        _check(lib().kvg_controllers_state(self.h, w, dw, t, a, p, q))
        return [dict(window=w[i], display_window=dw[i], ticks=t[i], active=a[i], pending=p[i],
                     paused=q[i]) for i in range(self.n)]

    def active(self, i: int) -> list[int]:
        cap = max(4 * self.total[i], self.total[i] + 256)  # list capacity (controllers.cu)
        out = (C.c_uint32 * cap)()
        n = C.c_size_t()
        _check(lib().kvg_controllers_active(self.h, i, out, cap, C.byref(n)))
        return list(out)[: n.value]

    def close(self):
        if getattr(self, "h", None):
            lib().kvg_controllers_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
