"""Experiment commands over the batched B200 engine.

    run_command(scenario, out_root)       ~ experiment.cpp:184-213
    compare_command(scenario, out_root)   ~ experiment.cpp:215-241
    sweep_command(scenario, out_root)     ~ experiment.cpp:243-287

The reference executes a command's rows through run_rows, a thread pool of
run_simulation calls (experiment.cpp:75-108). Here every row of a command is
one simulation of ONE engine batch on the GPU; the rows' artifacts
(trace.csv / summary.txt / phases.csv), manifest.json and table.txt are
byte-identical to what the reference writes, and the workload-hash replay
check (experiment.cpp:101-108) is kept.
"""
from __future__ import annotations

import copy
import json
import os
from dataclasses import dataclass, field

from . import abi, engine
from .config import Scenario


class InvariantViolation(RuntimeError):
    """errors.hpp InvariantViolation."""


class MissingBaseline(RuntimeError):
    """errors.hpp MissingBaseline."""


def format_g6(v: float) -> str:  # metrics.cpp:83-87
    return "%.6g" % v


def hash_hex(h: int) -> str:  # experiment.cpp:40-44
    return "0x%016x" % h


def sanitize_label(label: str) -> str:  # experiment.cpp:59-63
    return label.replace(":", "_").replace("=", "_")


def render_table(rows: list[list[str]]) -> str:  # metrics.cpp:284-308
    widths: list[int] = []
    for row in rows:
        widths += [0] * (len(row) - len(widths))
        for i, cell in enumerate(row):
            widths[i] = max(widths[i], len(cell))
    out = []
    for r, row in enumerate(rows):
        line = "  ".join(cell.ljust(widths[i]) for i, cell in enumerate(row)).rstrip(" ")
        out.append(line + "\n")
        if r == 0:
            out.append("-" * (sum(widths) + 2 * (len(widths) - 1)) + "\n")
    return "".join(out)


def render_comparison(runs: list[tuple[str, dict]], baseline: str) -> str:  # metrics.cpp:313-338
    base = next((s for name, s in runs if name == baseline), None)
    if base is None:
        raise MissingBaseline(f"baseline run '{baseline}' not present in comparison")
    rows = [["policy", "makespan_s", "speedup", "mean_hit", "recompute_frac", "middle_frac"]]
    for name, s in runs:
        speedup = base["makespan"] / s["makespan"] if s["makespan"] > 0 else 0.0
        rows.append([name, format_g6(s["makespan"]), "%.2fx" % speedup,
                     format_g6(s["mean_hit_rate"]), format_g6(s["recompute_fraction"]),
                     format_g6(s["middle_fraction"])])
    return render_table(rows)


def render_sweep(axis: str, runs: list[tuple[str, dict]]) -> str:  # metrics.cpp:340-352
    rows = [[axis, "makespan_s", "mean_hit", "recompute_frac", "middle_frac"]]
    for name, s in runs:
        rows.append([name, format_g6(s["makespan"]), format_g6(s["mean_hit_rate"]),
                     format_g6(s["recompute_fraction"]), format_g6(s["middle_fraction"])])
    return render_table(rows)


@dataclass
class Row:  # experiment.cpp:65-72
    label: str
    policy_text: str
    scenario: Scenario
    rel: str = ""
    dir: str = ""
    summary: dict = field(default_factory=dict)


def run_rows(rows: list[Row], device: int = 0) -> None:
    """Every row as one simulation of ONE batch (the reference's run_rows
    thread pool, experiment.cpp:75-108). Rows that share a workload and seed
    share one population. Artifacts are written for every row (partial ones
    after a horizon abort, like execute_run's finalize); then a horizon abort
    propagates, and the replay check runs."""
    pops: dict = {}
    specs = []
    for row in rows:
        os.makedirs(row.dir, exist_ok=True)
        s = row.scenario
        key = (s.seed, repr(s.workload))
        if key not in pops:
            pops[key] = engine.Population(s.workload, s.seed)
        specs.append(engine.SimSpec.from_scenario(s, row.policy_text, population=pops[key]))
    batch = engine.Batch(specs, device=device, host_outputs=True)
    try:
        status = batch.run(allow_horizon=True)
        for i, row in enumerate(rows):
            row.summary = batch.write_artifacts(i, row.dir, row.scenario.name, row.policy_text,
                                                row.scenario.seed)
        if status == abi.KVG_ERR_HORIZON:
            bad = next(r for i, r in enumerate(rows) if batch.result(i)["status"] != 0)
            raise engine.HorizonError(status, f"run {bad.label} exceeded its horizon")
    finally:
        batch.close()
    h0 = rows[0].summary["workload_hash"] if rows else 0
    for row in rows:
        if row.summary["workload_hash"] != h0:
            raise InvariantViolation(f"workload replay diverged: run {row.label} consumed a "
                                     "different action stream")


def write_manifest(dir_: str, command: str, s: Scenario, extra_key: str, extra_value: str,
                   rows: list[Row]) -> None:  # experiment.cpp:110-129
    m = {"command": command, "scenario": s.name, "seed": s.seed}
    if extra_key:
        m[extra_key] = extra_value
    m["rows"] = [{"label": r.label, "policy": r.policy_text, "dir": r.rel,
                  "workload_hash": hash_hex(r.summary["workload_hash"])} for r in rows]
    with open(os.path.join(dir_, "manifest.json"), "w", newline="") as fh:
        fh.write(json.dumps(m, indent=2, ensure_ascii=False) + "\n")


def _table_rows(rows: list[Row]) -> list[tuple[str, dict]]:
    return [(r.label, r.summary) for r in rows]


def run_command(s: Scenario, out_root: str, device: int = 0) -> str:
    d = os.path.join(out_root, s.name)
    rows = [Row(label=s.policy, policy_text=s.policy, scenario=s, rel=".", dir=d)]
    try:
        run_rows(rows, device)
    except engine.HorizonError:
        write_manifest(d, "run-aborted", s, "", "", [])
        raise
    write_manifest(d, "run", s, "", "", rows)
    sm = rows[0].summary
    return (f"run {s.name} policy={sm['policy'].decode() if isinstance(sm['policy'], bytes) else sm['policy']}"
            f" seed={s.seed}\n"
            f"  makespan {format_g6(sm['makespan'])} s, throughput "
            f"{format_g6(sm['throughput'])} tok/s\n"
            f"  hit rate {format_g6(sm['mean_hit_rate'])}, recompute fraction "
            f"{format_g6(sm['recompute_fraction'])}, middle fraction "
            f"{format_g6(sm['middle_fraction'])}\n"
            f"  artifacts in {d}\n")


def compare_command(s: Scenario, out_root: str, device: int = 0) -> str:
    if not s.compare:
        raise ValueError("compare needs a [compare] section with a baseline")
    if not s.compare.get("policies"):
        raise ValueError("compare.policies lists no policies")
    texts = [s.compare["baseline"]] + list(s.compare["policies"])
    d = os.path.join(out_root, f"{s.name}-compare")
    rows = []
    for i, t in enumerate(texts):
        rel = "%02d-" % (i + 1) + sanitize_label(t)
        rows.append(Row(label=t, policy_text=t, scenario=s, rel=rel, dir=os.path.join(d, rel)))
    run_rows(rows, device)
    write_manifest(d, "compare", s, "baseline", s.compare["baseline"], rows)
    table = render_comparison(_table_rows(rows), rows[0].label)
    with open(os.path.join(d, "table.txt"), "w", newline="") as fh:
        fh.write(table)
    return table


def sweep_command(s: Scenario, out_root: str, device: int = 0) -> str:
    if not s.sweep:
        raise ValueError("sweep needs a [sweep] section")
    axis, values = s.sweep["axis"], list(s.sweep["values"])
    d = os.path.join(out_root, f"{s.name}-sweep-{axis}")
    rows = []
    for v in values:
        sc = copy.deepcopy(s)
        if axis == "fixed_cap":
            label, pol = "cap=" + format_g6(float(v)), "agent_cap:%d" % int(v)
        else:
            label, pol = axis + "=" + format_g6(float(v)), "aimd"
            setattr(sc.controller, axis, float(v))
        rows.append(Row(label=label, policy_text=pol, scenario=sc))
    rows.append(Row(label="aimd", policy_text="aimd", scenario=s))  # adaptive reference row
    for r in rows:
        r.rel = sanitize_label(r.label)
        r.dir = os.path.join(d, r.rel)
    run_rows(rows, device)
    write_manifest(d, "sweep", s, "axis", axis, rows)
    table = render_sweep(axis, _table_rows(rows))
    with open(os.path.join(d, "table.txt"), "w", newline="") as fh:
        fh.write(table)
    return table
