"""ctypes mirror of include/kvgpu.h (the C boundary of the B200 engine).

Plumbing only: every struct here is a field-for-field copy of the C header so
that Python tests, the bench and the oracle bindings can hand identical
descriptors to the GPU engine (libkvgpu.so), the CPU restatement
(oracle/libkvoracle.so) and the reference harness (oracle/_ref/libkvref.so).
"""
from __future__ import annotations

import ctypes as C
import os

u32, u64, i32, f64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_double

KVG_OK, KVG_ERR_CONFIG, KVG_ERR_IO, KVG_ERR_HORIZON, KVG_ERR_STATE = 0, 1, 2, 3, 4
KVG_ERR_MISSING_BASELINE, KVG_ERR_CUDA = 5, 6
STATUS_NAMES = {0: "ok", 1: "config", 2: "io", 3: "horizon", 4: "state",
                5: "missing_baseline", 6: "cuda"}

DIST_CONSTANT, DIST_UNIFORM, DIST_LOGNORMAL = 0, 1, 2
POLICY_UNCONTROLLED, POLICY_REQUEST_CAP, POLICY_AGENT_CAP, POLICY_AIMD = 0, 1, 2, 3
EVICT_DISCARD, EVICT_OFFLOAD = 0, 1
OP_MATCH, OP_INSERT, OP_EVICT, OP_PIN, OP_UNPIN, OP_DISCARD, OP_RELOAD = 1, 2, 3, 4, 5, 6, 7
LOG_MATCH, LOG_INSERT, LOG_EVICT, LOG_VICTIM, LOG_FINISH, LOG_DISCARD = 1, 2, 3, 4, 5, 6


class Distribution(C.Structure):
    _fields_ = [("kind", u32), ("_pad", u32), ("a", f64), ("b", f64)]


class WorkloadConfig(C.Structure):
    _fields_ = [("agents", u32), ("shared_prompt", u32), ("prompt_tokens", u64),
                ("steps", u32), ("_pad", u32), ("gen_tokens", Distribution),
                ("obs_tokens", Distribution), ("tool_latency", Distribution),
                ("tool_probability", f64)]


class StepPlan(C.Structure):
    _fields_ = [("gen_tokens", u64), ("obs_tokens", u64), ("tool_latency", f64),
                ("has_tool", u32), ("_pad", u32)]


class Population(C.Structure):
    _fields_ = [("agents", u32), ("steps", u32), ("prompt_tokens", u64),
                ("shared_prompt", u32), ("_pad", u32),
                ("shared_prompt_tokens", u64), ("stream_hash", u64),
                ("peak_aggregate_tokens", u64), ("plans", C.POINTER(StepPlan))]


class ControllerConfig(C.Structure):
    _fields_ = [(n, f64) for n in ("alpha", "beta", "u_low", "u_high", "h_thresh",
                                   "w_min", "w_max", "initial_window",
                                   "control_interval", "signal_smoothing")]


class Policy(C.Structure):
    _fields_ = [("kind", u32), ("cap", u32), ("aimd", ControllerConfig)]


class CostParams(C.Structure):
    _fields_ = [(n, f64) for n in ("prefill_linear", "prefill_quadratic",
                                   "decode_base", "decode_context",
                                   "bytes_per_token", "pcie_bandwidth",
                                   "transfer_sync_overhead")]


class PhaseParams(C.Structure):
    _fields_ = [("sat_threshold", f64), ("hit_threshold", f64),
                ("hysteresis", i32), ("_pad", i32)]


class EngineParams(C.Structure):
    _fields_ = [("capacity", u64), ("page_size", u64), ("eviction", u32),
                ("paranoid", u32), ("hit_window_decay", f64), ("horizon", f64),
                ("phases", PhaseParams)]


class SimDesc(C.Structure):
    _fields_ = [("population", C.POINTER(Population)), ("policy", Policy),
                ("cost", CostParams), ("engine", EngineParams)]


class TraceRow(C.Structure):
    _fields_ = [("time", f64), ("usage", f64), ("hit_rate", f64), ("window", f64),
                ("active", u64), ("pending", u64), ("decoded_cum", u64),
                ("recompute_cum", u64), ("transfers", u64),
                ("hit_matched", f64), ("hit_requested", f64)]


class AgentStats(C.Structure):
    _fields_ = [("generated_tokens", u64), ("recompute_tokens", u64),
                ("recompute_events", u64), ("stall_events", u64),
                ("pause_events", u64), ("wait_time", f64),
                ("finish_time", f64), ("finish_ordinal", u64)]


class Ledger(C.Structure):
    _fields_ = [(n, f64) for n in ("prefill_fresh", "prefill_recompute",
                                   "decode", "transfer", "tool_wait")]


class PhaseLabel(C.Structure):
    _fields_ = [("phase", u32), ("_pad", u32), ("start", f64), ("end", f64)]


class SimResult(C.Structure):
    _fields_ = [("status", i32), ("n_phases", u32), ("ledger", Ledger),
                ("makespan", f64), ("device_busy", f64), ("link_busy", f64),
                ("decoded_tokens", u64), ("recompute_tokens", u64),
                ("recompute_events", u64), ("stall_events", u64),
                ("offloaded_tokens", u64), ("reloaded_tokens", u64),
                ("discarded_tokens", u64), ("total_wait_time", f64),
                ("ticks", u64), ("workload_hash", u64),
                ("agent_steps", u64), ("lookups", u64), ("events", u64),
                ("evict_calls", u64), ("evicted_pages", u64),
                ("cache_clock", u64), ("pool_used", u64),
                ("hit_matched", f64), ("hit_requested", f64),
                ("hit_pages", u64), ("created_pages", u64), ("refreshed_pages", u64),
                ("evict_scanned", u64), ("agent_events", u64), ("device_cycles", u64),
                ("phases", PhaseLabel * 3), ("abort_time", f64), ("unfinished", u64)]


class LogRecord(C.Structure):
    _fields_ = [("kind", u32), ("agent", u32), ("clock", u64), ("a", u64), ("b", u64)]


class BatchOptions(C.Structure):
    _fields_ = [("warps_per_sim", u32), ("log_capacity", u32),
                ("trace_capacity", u64), ("host_outputs", u32), ("verify", u32)]


class Summary(C.Structure):  # kvg_summary (metrics.hpp:85-118)
    _fields_ = [("name", C.c_char * 128), ("policy", C.c_char * 64), ("seed", u64),
                ("agents", u64), ("makespan", f64), ("throughput", f64),
                ("decoded_tokens", u64), ("recompute_tokens", u64), ("recompute_events", u64),
                ("stall_events", u64), ("recompute_fraction", f64), ("mean_hit_rate", f64),
                ("mean_usage", f64), ("ledger", Ledger), ("device_busy", f64),
                ("device_idle", f64), ("link_busy", f64), ("link_idle", f64),
                ("offloaded_tokens", u64), ("reloaded_tokens", u64), ("discarded_tokens", u64),
                ("total_wait_time", f64), ("warmup_duration", f64), ("middle_duration", f64),
                ("cooldown_duration", f64), ("middle_fraction", f64), ("warmup_hit_rate", f64),
                ("middle_hit_rate", f64), ("cooldown_hit_rate", f64),
                ("middle_usage_mean", f64), ("ticks", u64), ("workload_hash", u64)]


class Command(C.Structure):  # kvg_command == kva_command (kvadmit.h:123-126)
    _fields_ = [("kind", C.c_uint8), ("_pad", C.c_uint8 * 3), ("agent", u32)]


class CtlEvent(C.Structure):  # kvg_ctl_event
    _fields_ = [("controller", u32), ("kind", u32), ("agent", u32), ("_pad", u32)]


CMD_ADMIT, CMD_PAUSE, CMD_RESUME = 0, 1, 2
CTL_ADD_PENDING, CTL_AGENT_FINISHED, CTL_REQUEST_COMPLETE, CTL_TOOL_RETURN = 0, 1, 2, 3


class CacheOp(C.Structure):
    _fields_ = [("kind", u32), ("agent", u32), ("len", u64), ("arg", u64), ("arg2", u64)]


class CacheOpResult(C.Structure):
    _fields_ = [("status", i32), ("_pad", u32), ("r0", u64), ("r1", u64),
                ("clock", u64), ("used", u64), ("victims_begin", u64),
                ("victims_end", u64)]


class Victim(C.Structure):
    _fields_ = [("key", u64), ("stamp", u64)]


# ---------------------------------------------------------------------------
# Result field lists used by parity comparisons (bit-exact on every field).
RESULT_EXACT_FIELDS = (
    "makespan", "device_busy", "link_busy", "decoded_tokens", "recompute_tokens",
    "recompute_events", "stall_events", "offloaded_tokens", "reloaded_tokens",
    "discarded_tokens", "total_wait_time", "ticks", "workload_hash")
LEDGER_FIELDS = ("prefill_fresh", "prefill_recompute", "decode", "transfer",
                 "tool_wait")
TRACE_FIELDS = [f for f, _ in TraceRow._fields_]
AGENT_FIELDS = ("generated_tokens", "recompute_tokens", "recompute_events",
                "stall_events", "pause_events", "wait_time")

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("KVG_LIB") or os.path.join(PKG_DIR, "libkvgpu.so")


def struct_to_dict(s) -> dict:
    out = {}
    for name, typ in s._fields_:
        if name.startswith("_"):
            continue
        v = getattr(s, name)
        if isinstance(v, C.Structure):
            v = struct_to_dict(v)
        elif isinstance(v, C.Array):
            v = [struct_to_dict(x) if isinstance(x, C.Structure) else x for x in v]
        out[name] = v
    return out


def bucket_count(capacity: int, agents: int) -> int:
    """Mirror of capi.cu bucket_count: 4x worst-case live 32-page chunks, pow2."""
    live = (capacity + 31) // 32 + agents + 2
    b = 1
    while b < 4 * live:
        b <<= 1
    return max(64, b)


def table_bytes(capacity: int, agents: int) -> int:
    """Primary + alternate hash tables of one simulation (512 B per bucket)."""
    return 2 * bucket_count(capacity, agents) * 32 * 16
