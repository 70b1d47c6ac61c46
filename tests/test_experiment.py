"""Experiment commands: run / compare / sweep with
every row of a command executed as one engine batch. The directory each
command writes — per-row trace.csv / summary.txt / phases.csv, manifest.json,
table.txt — must be byte-identical to what the reference's own commands
write (tests/golden/experiments.json, recorded through the reference's C ABI
kva_cmd_run / kva_cmd_compare / kva_cmd_sweep, kvadmit.h:58-78).

CPU suite: the orchestration with the rows executed by the CPU oracle (the
artifact writers are the product's host code). GPU suite: the real thing."""
import ctypes as C
import hashlib
import json
import os

import pytest

from paper_2601_22705_b200 import abi, config, engine, experiment
from tests.helpers import GOLDEN, load_presets, oracle_run

GOLD = json.load(open(os.path.join(GOLDEN, "experiments.json")))


def tree_hashes(d):
    out = {}
    for root, _, files in os.walk(d):
        for f in files:
            p = os.path.join(root, f)
            out[os.path.relpath(p, d)] = hashlib.sha256(open(p, "rb").read()).hexdigest()
    return dict(sorted(out.items()))


def oracle_rows(rows, device=0):
    """run_rows with the CPU oracle executing each row (CPU-suite stand-in)."""
    for row in rows:
        os.makedirs(row.dir, exist_ok=True)
        s = row.scenario
        pop = engine.Population(s.workload, s.seed)
        o = oracle_run(s, row.policy_text, pop=pop.c)
        summ = abi.Summary()
        rc = engine.lib().kvg_write_run_artifacts(
            row.dir.encode(), s.name.encode(), row.policy_text.encode(), s.seed,
            s.workload.agents, C.byref(o["raw_result"]), o["raw_trace"], o["n_trace"],
            C.byref(summ))
        assert rc == 0
        row.summary = abi.struct_to_dict(summ)


def run_job(key, tmp_path):
    preset, cmd = key.split("/")
    s = config.scenario_from_dict(load_presets()[preset])
    fn = {"run": experiment.run_command, "compare": experiment.compare_command,
          "sweep": experiment.sweep_command}[cmd]
    text = fn(s, str(tmp_path))
    return text, tree_hashes(os.path.join(tmp_path, GOLD[key]["dir"]))


@pytest.mark.parametrize("key", sorted(GOLD))
def test_commands_with_oracle_rows_match_reference(key, tmp_path, monkeypatch):
    monkeypatch.setattr(experiment, "run_rows", oracle_rows)
    text, files = run_job(key, tmp_path)
    assert files == GOLD[key]["files"]
    assert text.replace(str(tmp_path), "<root>") == GOLD[key]["text"]


def test_render_table_matches_reference_layout():
    t = experiment.render_table([["a", "bb"], ["ccc", "d"]])
    assert t == "a    bb\n-------\nccc  d\n"


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(GOLD))
def test_commands_on_gpu_match_reference(key, tmp_path):
    text, files = run_job(key, tmp_path)
    assert files == GOLD[key]["files"]
    assert text.replace(str(tmp_path), "<root>") == GOLD[key]["text"]
