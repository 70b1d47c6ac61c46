"""Comparison helpers: bit-exact equality of simulation outputs."""
from __future__ import annotations

import struct

from paper_2601_22705_b200 import abi


def _bits(x):
    if isinstance(x, float):
        return struct.pack("<d", x)
    return x


def diff_results(a: dict, b: dict, fields=abi.RESULT_EXACT_FIELDS) -> list[str]:
    out = []
    for f in fields:
        if _bits(a[f]) != _bits(b[f]):
            out.append(f"{f}: {a[f]!r} != {b[f]!r}")
    for f in abi.LEDGER_FIELDS:
        if _bits(a["ledger"][f]) != _bits(b["ledger"][f]):
            out.append(f"ledger.{f}: {a['ledger'][f]!r} != {b['ledger'][f]!r}")
    return out


def diff_trace(a: list[dict], b: list[dict]) -> list[str]:
    if len(a) != len(b):
        return [f"trace length {len(a)} != {len(b)}"]
    for i, (x, y) in enumerate(zip(a, b)):
        for f in abi.TRACE_FIELDS:
            if _bits(x[f]) != _bits(y[f]):
                return [f"trace[{i}].{f}: {x[f]!r} != {y[f]!r}"]
    return []


def diff_agents(a: list[dict], b: list[dict], fields=abi.AGENT_FIELDS) -> list[str]:
    if len(a) != len(b):
        return [f"agent count {len(a)} != {len(b)}"]
    for i, (x, y) in enumerate(zip(a, b)):
        for f in fields:
            if _bits(x[f]) != _bits(y[f]):
                return [f"agent[{i}].{f}: {x[f]!r} != {y[f]!r}"]
    return []


def diff_all(a: dict, b: dict, agent_fields=abi.AGENT_FIELDS) -> list[str]:
    return (diff_results(a["result"], b["result"]) + diff_trace(a["trace"], b["trace"])
            + diff_agents(a["agents"], b["agents"], agent_fields))
