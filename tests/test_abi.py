"""The C-ABI boundary (include/kvgpu.h) on a machine without a GPU: the
library loads, exports every declared entry point, validates descriptors
before touching a device, and fails loudly (KVG_ERR_CUDA) instead of falling
back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2601_22705_b200 import abi, config, engine

HEADER = os.path.join(abi.REPO_DIR, "include", "kvgpu.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"KVG_API\s+[\w\s\*]+?\b(kvg_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    names = declared()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (kvg_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert missing == []
    lib = engine.lib()
    for n in names:
        assert getattr(lib, n) is not None


def test_only_kvg_symbols_are_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    funcs = re.findall(r"\bT (\w+)", out)
    assert funcs and all(f.startswith("kvg_") for f in funcs), funcs


def test_version_and_defaults():
    lib = engine.lib()
    assert lib.kvg_version().decode().startswith("0.")
    c = abi.CostParams()
    lib.kvg_cost_params_init(C.byref(c))
    assert c.prefill_linear == 5e-5 and c.bytes_per_token == 6.67e9 / 4096.0
    k = abi.ControllerConfig()
    lib.kvg_controller_config_init(C.byref(k))
    assert (k.alpha, k.beta, k.u_low, k.u_high, k.h_thresh) == (2.0, 0.5, 0.2, 0.5, 0.2)
    e = abi.EngineParams()
    lib.kvg_engine_params_init(C.byref(e))
    assert e.horizon == 1e6 and e.phases.hysteresis == 3


def _spec(**over):
    s = config.c1_toy()
    for k, v in over.items():
        sec, _, name = k.partition(".")
        setattr(getattr(s, sec), name, v)
    return engine.SimSpec.from_scenario(s)


@pytest.mark.parametrize("over,msg", [
    ({"engine.capacity": 0}, "capacity"),
    ({"engine.page_size": 0}, "page_size"),
    ({"engine.hit_window_decay": 1.0}, "hit_window_decay"),
    ({"controller.beta": 1.0}, "beta"),
    ({"controller.u_low": 0.9}, "thresholds"),
])
def test_invalid_descriptors_are_config_errors(over, msg):
    with pytest.raises(engine.EngineError) as e:
        engine.Batch([_spec(**over)])
    assert e.value.status == abi.KVG_ERR_CONFIG
    assert msg in str(e.value)


def test_no_gpu_means_loud_failure_not_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(engine.EngineError) as e:
        engine.Batch([_spec()])
    assert e.value.status == abi.KVG_ERR_CUDA
    assert "no CPU fallback" in str(e.value)
    with pytest.raises(engine.EngineError) as e:
        engine.DeviceCache(64, 16)
    assert e.value.status == abi.KVG_ERR_CUDA


def test_last_error_is_never_null():
    assert engine.lib().kvg_last_error() is not None
