"""The C++ drop-in: the reference's own callers of
kvadmit::run_simulation, unmodified, running on the B200 through the product
adapter include/kvadmit_gpu.hpp (engine.hpp:75-78 seam).

* oracle/_ref/acceptance_gpu — the reference acceptance gate
  (/root/reference/proj/tests/acceptance/acceptance.cpp) linked with every
  run_simulation call wrapped onto kvgpu::run_simulation. Criteria 1-9 must
  print exactly what the unmodified gate prints (tests/golden/acceptance.json):
  the detail strings carry makespans, hit rates and ratios to 6 digits.
* oracle/_ref/libkvadmit_gpu.so — the reference's kva_* C ABI
  (kvadmit.h:56-78: scenario load, kva_cmd_run / compare / sweep, run_rows'
  thread pool) with its simulations on the GPU. Its artifact directories must
  be byte-identical to the reference's (tests/golden/experiments.json), and a
  horizon abort must fail the same way (status, message, partial trace).

Both binaries are built here by oracle/Makefile (they link the reference
sources, so they are test infrastructure) and travel to the GPU box."""
import ctypes as C
import json
import os
import shutil
import subprocess
import tempfile

import pytest

from tests.helpers import GOLDEN
from tests.test_experiment import GOLD as EXP_GOLD, tree_hashes

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_OUT = os.path.join(REPO, "oracle", "_ref")
ACC_GPU = os.path.join(REF_OUT, "acceptance_gpu")
ACC_CPU = os.path.join(REF_OUT, "acceptance_cpu")
KVA_GPU = os.path.join(REF_OUT, "libkvadmit_gpu.so")
CONFIGS = os.path.join(REF_OUT, "configs")
ACC_GOLD = json.load(open(os.path.join(GOLDEN, "acceptance.json")))

need_bins = pytest.mark.skipif(not (os.path.exists(ACC_GPU) and os.path.exists(KVA_GPU)),
                               reason="oracle/_ref drop-in binaries not built (make -C oracle gpuseam)")


def _run_acc(binary, i, **kw):
    return subprocess.run([binary, str(i)], cwd=REPO, capture_output=True, text=True,
                          timeout=600, **kw)


@need_bins
def test_drop_in_links_the_product_library():
    for b in (ACC_GPU, KVA_GPU):
        out = subprocess.run(["ldd", b], capture_output=True, text=True).stdout
        line = next(l for l in out.splitlines() if "libkvgpu.so" in l)
        assert os.path.realpath(line.split("=>")[1].split()[0]) == os.path.realpath(
            os.path.join(REPO, "paper_2601_22705_b200", "libkvgpu.so"))


@need_bins
def test_unmodified_gate_matches_golden():
    if not os.path.exists(ACC_CPU):
        pytest.skip("acceptance_cpu not built")
    for i in (1, 3, 8, 9):  # the quick ones; all nine are in the golden
        assert _run_acc(ACC_CPU, i).stdout == ACC_GOLD[str(i)]


@need_bins
def test_gpu_gate_fails_loudly_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _run_acc(ACC_GPU, 3)
    assert r.returncode != 0 and "no CUDA device" in r.stdout


def test_adapter_header_compiles_against_reference_headers(tmp_path):
    src = "/root/reference/proj/src"
    if not os.path.isdir(src):
        pytest.skip("reference headers only exist in the build container")
    tu = tmp_path / "tu.cpp"
    tu.write_text('#include "kvadmit_gpu.hpp"\n'
                  "kvadmit::SimulationResult (*f)(kvadmit::Population, const kvadmit::Policy&,"
                  " const kvadmit::CostParams&, const kvadmit::EngineParams&,"
                  " kvadmit::SimulationResult*, const kvgpu::Options&) = &kvgpu::run_simulation;\n")
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                        f"-I{src}", f"-I{os.path.join(REPO, 'include')}", str(tu)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
@need_bins
@pytest.mark.parametrize("crit", list(range(1, 10)))
def test_acceptance_gate_on_gpu(crit):
    r = _run_acc(ACC_GPU, crit, env=dict(os.environ, KVGPU_VERIFY="0"))
    assert r.stdout == ACC_GOLD[str(crit)], (r.stdout, r.stderr)
    assert r.returncode == 0


def _kva(path):
    C.CDLL("libstdc++.so.6", mode=C.RTLD_GLOBAL)
    lib = C.CDLL(path)
    lib.kva_scenario_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    lib.kva_scenario_set.argtypes = [C.c_void_p, C.c_char_p]
    for f in ("kva_cmd_compare", "kva_cmd_sweep"):
        getattr(lib, f).argtypes = [C.c_void_p, C.c_char_p, C.c_uint, C.POINTER(C.c_void_p)]
    lib.kva_cmd_run.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]
    lib.kva_text_free.argtypes = [C.c_void_p]
    lib.kva_scenario_free.argtypes = [C.c_void_p]
    lib.kva_last_error.restype = C.c_char_p
    return lib


def _cmd(lib, preset, cmd, root, jobs=1, sets=()):
    sc = C.c_void_p()
    assert lib.kva_scenario_load(os.path.join(CONFIGS, preset + ".toml").encode(),
                                 C.byref(sc)) == 0, lib.kva_last_error()
    for s in sets:
        assert lib.kva_scenario_set(sc, s.encode()) == 0, lib.kva_last_error()
    text = C.c_void_p()
    if cmd == "run":
        rc = lib.kva_cmd_run(sc, root.encode(), C.byref(text))
    else:
        rc = getattr(lib, "kva_cmd_" + cmd)(sc, root.encode(), jobs, C.byref(text))
    err = lib.kva_last_error().decode()
    rendered = C.cast(text, C.c_char_p).value.decode() if text.value else None
    if text.value:
        lib.kva_text_free(text)
    lib.kva_scenario_free(sc)
    return rc, err, rendered


@pytest.mark.gpu
@need_bins
@pytest.mark.parametrize("key", sorted(EXP_GOLD))
def test_kva_commands_on_gpu_match_reference(key):
    preset, cmd = key.split("/")
    lib = _kva(KVA_GPU)
    for jobs in ((1, 4) if cmd != "run" else (1,)):
        root = tempfile.mkdtemp()
        try:
            rc, err, text = _cmd(lib, preset, cmd, root, jobs)
            assert rc == 0, err
            assert tree_hashes(os.path.join(root, EXP_GOLD[key]["dir"])) == EXP_GOLD[key]["files"]
            assert text.replace(root, "<root>") == EXP_GOLD[key]["text"]
        finally:
            shutil.rmtree(root)


@pytest.mark.gpu
@need_bins
def test_horizon_abort_matches_reference():
    """A run past its horizon: kva_cmd_run returns KVA_ERR_HORIZON with the
    reference's HorizonError message and still writes the partial trace
    (kvadmit.h:66-69; engine.cpp:112-119)."""
    outs = []
    for path in (os.path.join(REF_OUT, "libkvref.so"), KVA_GPU):
        lib = _kva(path)
        root = tempfile.mkdtemp()
        try:
            rc, err, _ = _cmd(lib, "thrash", "run", root, sets=("horizon=120",))
            outs.append((rc, err, tree_hashes(root)))
        finally:
            shutil.rmtree(root)
    assert outs[0][0] == 3 and "exceeded horizon" in outs[0][1]
    assert outs[1] == outs[0]


ADAPTER_CHECK = os.path.join(REF_OUT, "adapter_check")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(ADAPTER_CHECK), reason="oracle/_ref/adapter_check not built")
def test_run_simulations_batch_equals_reference_run_simulation():
    """kvgpu::run_simulations (one device batch of 16 jobs: every preset under
    uncontrolled / aimd / agent_cap / request_cap / offload, plus a job the
    reference rejects) against the reference run_simulation in-process:
    SimulationResult field by field, bit for bit, and the same per-job error."""
    r = subprocess.run([ADAPTER_CHECK, CONFIGS], cwd=REPO, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ALL OK"), r.stdout + r.stderr
