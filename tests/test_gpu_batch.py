"""Batch-level behaviour of the device engine at BASELINE scale."""
import pytest

from paper_2601_22705_b200 import abi, config, engine
from tests.helpers import oracle_run
from tests.parity import diff_all

pytestmark = pytest.mark.gpu


def _det(r: dict) -> dict:
    """Result fields that must be deterministic (drops the timing counter)."""
    return {k: v for k, v in r.items() if k != "device_cycles"}
AGENT_ALL = abi.AGENT_FIELDS + ("finish_time", "finish_ordinal")


@pytest.fixture(scope="module")
def c4_batch():
    pop = engine.Population(config.c1_toy().workload, 42)
    scen = config.c4_sweep(4096)
    specs = [engine.SimSpec.from_scenario(s, population=pop) for s in scen]
    b = engine.Batch(specs)
    b.run()
    yield scen, pop, b
    b.close()


def test_c4_conservation_properties(c4_batch):
    scen, pop, b = c4_batch
    rs = b.results_raw()
    assert len(rs) == 4096
    for r in rs:
        assert r.status == 0
        assert r.agent_steps == 64 * 10          # work conservation
        assert r.decoded_tokens == 64 * 10 * 256
        device = r.ledger.prefill_fresh + r.ledger.prefill_recompute + r.ledger.decode
        assert abs(device - r.device_busy) <= 1e-9 * max(1.0, r.device_busy)
        assert r.device_busy <= r.makespan + 1e-9
        assert r.workload_hash == 0xa0ac2d3c3bc97b20


@pytest.mark.parametrize("k", [0, 1, 63, 64, 255, 256, 1023, 1024, 2047, 4095])
def test_c4_sample_sims_bit_exact_vs_oracle(c4_batch, k):
    scen, pop, b = c4_batch
    g = dict(status=b.result(k)["status"], result=b.result(k), trace=b.trace(k),
             agents=b.agent_stats(k))
    o = oracle_run(scen[k], pop=pop.c)
    assert diff_all(g, o, AGENT_ALL) == []


def test_host_delivery_equals_device_outputs():
    s = config.c1_toy("uncontrolled")
    spec = engine.SimSpec.from_scenario(s)
    a = engine.Batch([spec, spec])
    a.run()
    h = engine.Batch([spec, spec], host_outputs=True)
    h.run()
    for i in range(2):
        assert _det(a.result(i)) == _det(h.result(i))
        assert a.trace(i) == h.trace(i)
        assert a.agent_stats(i) == h.agent_stats(i)


def test_streamed_host_delivery_mixed_batch_with_regrow():
    # rows stream into the pinned host array at cursor-allocated offsets (in
    # finish order); a tiny trace capacity forces the regrow + re-run path
    specs = []
    for pol, seed in [("uncontrolled", 1), ("aimd", 2), ("aimd", 3), ("uncontrolled", 4)]:
        s = config.c1_toy(pol)
        s.seed = seed
        specs.append(engine.SimSpec.from_scenario(s))
    a = engine.Batch(specs)
    a.run()
    h = engine.Batch(specs, host_outputs=True, trace_capacity=8)
    h.run()
    for i in range(len(specs)):
        assert _det(a.result(i)) == _det(h.result(i))
        assert a.trace(i) == h.trace(i) and len(h.trace(i)) > 8
        assert a.agent_stats(i) == h.agent_stats(i)
    h.run()  # rerun reuses the host block
    for i in range(len(specs)):
        assert a.trace(i) == h.trace(i)
        assert (a.trace_array(i) == h.trace_array(i)).all()


def test_host_delivery_packed_fallback(monkeypatch):
    # a host block over the streaming limit falls back to pack + one DMA
    monkeypatch.setenv("KVG_STREAM_MAX", "1024")
    s = config.c1_toy("aimd")
    spec = engine.SimSpec.from_scenario(s)
    a = engine.Batch([spec, spec])
    a.run()
    h = engine.Batch([spec, spec], host_outputs=True)
    h.run()
    for i in range(2):
        assert a.trace(i) == h.trace(i)
        assert (a.trace_array(i) == h.trace_array(i)).all()


def test_trace_overflow_regrows_and_reruns():
    s = config.c1_toy("aimd")
    spec = engine.SimSpec.from_scenario(s)
    small = engine.Batch([spec], trace_capacity=8)
    small.run()
    big = engine.Batch([spec])
    big.run()
    assert small.trace(0) == big.trace(0) and len(big.trace(0)) == 1393


def test_rerun_is_deterministic():
    s = config.c1_toy("uncontrolled")
    b = engine.Batch([engine.SimSpec.from_scenario(s)])
    b.run()
    first = (_det(b.result(0)), b.trace(0))
    b.run()
    assert (_det(b.result(0)), b.trace(0)) == first


def test_horizon_partial_result():
    s = config.c1_toy("uncontrolled")
    s.engine.horizon = 100.0
    b = engine.Batch([engine.SimSpec.from_scenario(s)])
    st = b.run()
    assert st == abi.KVG_ERR_HORIZON
    r = b.result(0)
    assert r["status"] == abi.KVG_ERR_HORIZON
    o = oracle_run(s)
    assert o["status"] == abi.KVG_ERR_HORIZON
    assert r["makespan"] == o["result"]["makespan"]
    assert b.trace(0) == o["trace"]


def test_run_simulation_mirror():
    s = config.c1_toy("aimd")
    out = engine.run_simulation(engine.Population(s.workload, s.seed), *s.resolved()[:1],
                                s.cost.to_abi(), s.resolved()[1].to_abi())
    assert out["result"]["makespan"] == oracle_run(s)["result"]["makespan"]


@pytest.mark.parametrize("verify", [False, True])
def test_c4_sweep_runs_in_one_wave(verify):
    # all 4,096 C4 simulations resident at once (148 SMs x 28 one-warp CTAs):
    # a second wave of even a few simulations doubles the kernel time
    pop = engine.Population(config.c1_toy().workload, 42)
    specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep(4096)]
    b = engine.Batch(specs, verify=verify)
    g = b.geometry()
    b.close()
    assert g["small_sims"] == 4096
    assert g["ctas_per_sm"] >= 28, g
    assert g["waves"] == 1, g


@pytest.mark.parametrize("mode", [1, engine.HOST_OUTPUTS_COPY], ids=["streamed", "dma"])
def test_launch_wait_pipeline_matches_run(mode):
    # kvg_batch_launch / kvg_batch_wait with two batches in flight (the bench's
    # pipelined e2e leg) give the same records as a blocking kvg_batch_run
    pop = engine.Population(config.c1_toy().workload, 42)
    specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep(512)]
    ref = engine.Batch(specs, verify=False, host_outputs=True)
    ref.run()
    want = ref.results_array()
    want_tr = [ref.trace(i) for i in (0, 255, 511)]
    ref.close()
    prev = None
    got = []
    for _ in range(3):
        b = engine.Batch(specs, verify=False, host_outputs=mode)
        b.launch()
        with pytest.raises(Exception):
            b.result(0)  # not readable while in flight
        with pytest.raises(Exception):
            b.launch()   # one launch at a time
        if prev is not None:
            prev.wait()
            got.append((prev.results_array(), [prev.trace(i) for i in (0, 255, 511)]))
            prev.close()
        prev = b
    prev.wait()
    got.append((prev.results_array(), [prev.trace(i) for i in (0, 255, 511)]))
    prev.close()
    skip = {"device_cycles"}
    for arr, tr in got:
        for name in want.dtype.names:
            if name not in skip:
                assert (arr[name] == want[name]).all(), name
        assert tr == want_tr


def test_free_while_in_flight_waits():
    pop = engine.Population(config.c1_toy().workload, 42)
    specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep(64)]
    b = engine.Batch(specs, verify=False)
    b.launch()
    b.close()  # kvg_batch_free synchronises the stream before releasing memory
    c = engine.Batch(specs, verify=False)
    c.run()
    assert all(r.status == 0 for r in c.results_raw())
    c.close()


def test_host_outputs_mode_checked():
    pop = engine.Population(config.c1_toy().workload, 42)
    specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep(4)]
    with pytest.raises(Exception):
        engine.Batch(specs, host_outputs=3)


def test_device_phases_match_host_classifier_over_params():
    # coop_phases (run-by-run scan of the ballot words) against the host
    # classifier kvg_classify_phases, itself pinned to the reference goldens
    # (tests/test_config.py), over thresholds and hysteresis lengths 1-100
    import ctypes as C
    import random
    rng = random.Random(7)
    pop = engine.Population(config.c1_toy().workload, 42)
    scen = config.c4_sweep(256)
    for s in scen:
        s.engine.sat_threshold = rng.choice([0.3, 0.5, 0.8, 0.95])
        s.engine.hit_threshold = rng.choice([0.2, 0.5, 0.9, 1.0])
        s.engine.hysteresis = rng.choice([1, 2, 3, 5, 17, 40, 100])
    specs = [engine.SimSpec.from_scenario(s, population=pop) for s in scen]
    b = engine.Batch(specs, verify=False, host_outputs=True)
    b.run()
    res = b.results_raw()
    seen = set()
    for i, s in enumerate(scen):
        tr = b.trace(i)
        rows = (abi.TraceRow * max(1, len(tr)))()
        for k, r in enumerate(tr):
            rows[k] = abi.TraceRow(**r)
        out = (abi.PhaseLabel * 3)()
        n = C.c_size_t()
        pp = s.engine.to_abi().phases
        assert engine.lib().kvg_classify_phases(rows, len(tr), res[i].makespan, C.byref(pp), out,
                                                3, C.byref(n)) == 0
        want = [(out[k].phase, out[k].start, out[k].end) for k in range(n.value)]
        got = [(res[i].phases[k].phase, res[i].phases[k].start, res[i].phases[k].end)
               for k in range(res[i].n_phases)]
        assert got == want, (i, s.engine.hysteresis, got, want)
        seen.add(len(want))
    b.close()
    assert len(seen) >= 2  # the cases cover more than one phase shape
