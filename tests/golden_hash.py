"""Canonical hashing of simulation outputs for the committed golden fixtures.
Only fields the reference defines (SimulationResult, TraceRecord/TickHits,
AgentStats, phases) enter the hashes; doubles are hashed by bit pattern."""
from __future__ import annotations

import hashlib
import struct

from paper_2601_22705_b200 import abi


def hx(v):
    return struct.pack("<d", v).hex() if isinstance(v, float) else v


def result_record(res: dict) -> dict:
    out = {k: hx(res[k]) for k in abi.RESULT_EXACT_FIELDS}
    out["ledger"] = {k: hx(res["ledger"][k]) for k in abi.LEDGER_FIELDS}
    out["phases"] = [[p["phase"], hx(p["start"]), hx(p["end"])]
                     for p in res["phases"][: res["n_phases"]]]
    return out


def trace_sha(trace: list[dict]) -> str:
    h = hashlib.sha256()
    for r in trace:
        for f in abi.TRACE_FIELDS:
            h.update(str(hx(r[f])).encode())
    return h.hexdigest()


def agents_sha(agents: list[dict]) -> str:
    h = hashlib.sha256()
    for a in agents:
        for f in abi.AGENT_FIELDS:
            h.update(str(hx(a[f])).encode())
    return h.hexdigest()


def run_record(run: dict) -> dict:
    rec = dict(status=run["status"], result=result_record(run["result"]),
               trace_sha=trace_sha(run["trace"]), agents_sha=agents_sha(run["agents"]),
               n_trace=len(run["trace"]))
    if run.get("digests") is not None:
        rec["n_events"] = len(run["digests"])
        rec["digest_sha"] = hashlib.sha256(run["digests"].tobytes()).hexdigest()
    return rec


def sim_digest(status: int, result: dict, trace, agents) -> str:
    """One 16-hex digest of a whole simulation's reference-defined outputs,
    for full-size fixtures (thousands of simulations): the result record,
    the raw trace rows (kvg_trace_row, 88 B each: every field is a double or
    u64, so the bytes are the bit patterns) and the six AgentStats fields of
    every agent (the first 48 B of each kvg_agent_stats; the reference does
    not define finish_time / finish_ordinal). `trace` and `agents` are numpy
    structured arrays in the ABI layouts."""
    import json

    import numpy as np
    h = hashlib.sha256()
    h.update(json.dumps(dict(status=status, result=result_record(result)),
                        sort_keys=True).encode())
    h.update(np.ascontiguousarray(trace).view(np.uint8).tobytes())
    a = np.ascontiguousarray(agents).view(np.uint8).reshape(-1, 64)[:, :48]
    h.update(a.tobytes())
    return h.hexdigest()[:16]
