"""Run artifacts: trace.csv, summary.txt and
phases.csv written from engine results must be BYTE-identical to what the
reference's own writers produce for the same run (execute_run's finalize,
experiment.cpp:161-170; metrics.cpp:89-183, 266-276), so `kvadmit report`
and diff-based determinism checks (acceptance criterion 10) work on them.

CPU suite: the artifact writers in libkvgpu.so are host code; they are fed
the oracle's results (bit-identical to the GPU's, see test_gpu_*). GPU suite:
the same writers fed the device's results."""
import ctypes as C
import os

import pytest

from paper_2601_22705_b200 import abi, engine
from tests.golden_cases import CASES, case_scenario
from tests.helpers import load_presets, oracle_run, ref_artifacts
from tests.offload_cases import OFFLOAD_CASES, offload_scenario

PICKS = ["c1_uncontrolled", "c1_aimd", "preset_thrash_aimd", "preset_smoke_request_cap:1",
         "eng_horizon", "eng_summary", "rand_3", "c3s128_aimd_h03", "off_preset_smoke",
         "off_c3s8", "off_eng_random_2"]


def scenario(cid):
    pres = load_presets()
    for c in CASES:
        if c["id"] == cid:
            return case_scenario(c, pres)
    c = next(c for c in OFFLOAD_CASES if c["id"] == cid)
    return offload_scenario(c, pres)


def files(d):
    return {f: open(os.path.join(d, f), "rb").read()
            for f in ("trace.csv", "summary.txt", "phases.csv")}


@pytest.mark.parametrize("cid", PICKS)
def test_artifacts_from_oracle_results_are_byte_identical(cid, tmp_path):
    s, pol = scenario(cid)
    label = pol or s.policy
    ref_artifacts(s, pol, str(tmp_path / "ref"), label)
    pop = engine.Population(s.workload, s.seed)
    o = oracle_run(s, pol, pop=pop.c)
    out = tmp_path / "ours"
    os.makedirs(out)
    summ = abi.Summary()
    rc = engine.lib().kvg_write_run_artifacts(str(out).encode(), s.name.encode(), label.encode(),
                                              s.seed, s.workload.agents,
                                              C.byref(o["raw_result"]), o["raw_trace"],
                                              o["n_trace"], C.byref(summ))
    assert rc == 0
    assert files(tmp_path / "ref") == files(out)


@pytest.mark.gpu
@pytest.mark.parametrize("cid", PICKS)
def test_artifacts_from_gpu_results_are_byte_identical(cid, tmp_path):
    s, pol = scenario(cid)
    label = pol or s.policy
    ref_artifacts(s, pol, str(tmp_path / "ref"), label)
    b = engine.Batch([engine.SimSpec.from_scenario(s, pol)])
    b.run()
    b.write_artifacts(0, str(tmp_path / "gpu"), s.name, label, s.seed)
    b.close()
    assert files(tmp_path / "ref") == files(tmp_path / "gpu")
