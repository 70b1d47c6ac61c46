"""Parity case catalogue shared by the golden generator and the tests.

Every case is a (scenario, policy) pair run identically by the reference
(golden fixtures), the CPU oracle and the GPU engine. They mirror the
reference's own test strategy: the shipped presets and policy
rows (configs/*.toml), the analytic/property engine tests
(tests/test_engine.cpp:97-352), BASELINE configs C1/C2 and scaled C2/C3/C5
shapes, and a seeded randomized sweep like test_engine.cpp:315-352.
"""
from __future__ import annotations

import copy
import random

from paper_2601_22705_b200 import config
from paper_2601_22705_b200.config import (ControllerConfig, CostParams, Distribution,
                                          EngineParams, Scenario, WorkloadConfig)


def test_cost() -> CostParams:  # tests/test_engine.cpp:25-35
    return CostParams(prefill_linear=1e-4, prefill_quadratic=1e-7, decode_base=1e-3,
                      decode_context=1e-8, bytes_per_token=1e6, pcie_bandwidth=1e9,
                      transfer_sync_overhead=0.01)


def constant_workload(agents, prompt, steps, gen, shared=True) -> WorkloadConfig:
    return WorkloadConfig(agents=agents, shared_prompt=shared, prompt_tokens=prompt,
                          steps=steps, gen_tokens=Distribution("constant", gen),
                          obs_tokens=Distribution("constant", 0),
                          tool_latency=Distribution("constant", 0), tool_probability=0.0)


def engine_case(name, wl, seed, policy, capacity, page=1, ctrl=None, horizon=1e6):
    s = Scenario(name=name, seed=seed, policy=policy)
    s.workload = wl
    s.engine = EngineParams(capacity=capacity, page_size=page, horizon=horizon)
    s.controller = ctrl or ControllerConfig()
    s.cost = test_cost()
    return s


def _engine_tests() -> list[tuple[str, Scenario, str]]:
    out = []
    out.append(("eng_analytic", engine_case("a", constant_workload(1, 16, 3, 8), 1,
                                            "uncontrolled", 1024), None))
    wl = constant_workload(1, 16, 2, 8)
    wl.tool_probability = 1.0
    wl.obs_tokens = Distribution("constant", 4)
    wl.tool_latency = Distribution("constant", 0.5)
    out.append(("eng_tools", engine_case("t", wl, 1, "uncontrolled", 1024), None))
    out.append(("eng_empty", engine_case("e", constant_workload(0, 8, 1, 4), 1,
                                         "uncontrolled", 64), None))
    wl = constant_workload(6, 32, 4, 8)
    wl.gen_tokens = Distribution("uniform", 4, 12)
    wl.tool_probability = 0.5
    wl.obs_tokens = Distribution("uniform", 2, 6)
    wl.tool_latency = Distribution("lognormal", 0.1, 0.4)
    out.append(("eng_bitident", engine_case("b", wl, 9, "aimd", 160, page=4,
                                            ctrl=ControllerConfig(initial_window=2, w_max=6)),
                None))
    wl = constant_workload(2, 64, 4, 32, shared=False)
    out.append(("eng_agentcap1", engine_case("c", wl, 3, "agent_cap:1", 256), None))
    out.append(("eng_requestcap1", engine_case("c", wl, 3, "request_cap:1", 256), None))
    out.append(("eng_shared", engine_case("s", constant_workload(4, 64, 1, 8), 2,
                                          "uncontrolled", 1024), None))
    wl = constant_workload(5, 24, 3, 8)
    wl.tool_probability = 0.6
    wl.obs_tokens = Distribution("constant", 4)
    wl.tool_latency = Distribution("lognormal", 0.05, 0.3)
    for iv, tag in ((0.02, "a"), (0.007, "b")):
        out.append((f"eng_cadence_{tag}", engine_case("k", wl, 5, "uncontrolled", 4096,
                                                     ctrl=ControllerConfig(control_interval=iv)),
                    None))
    out.append(("eng_pausing", engine_case(
        "p", constant_workload(8, 16, 10, 16), 6, "aimd", 300,
        ctrl=ControllerConfig(initial_window=8, w_max=8, control_interval=0.05, h_thresh=0.9)),
        None))
    out.append(("eng_stall", engine_case("st", constant_workload(2, 32, 3, 16, shared=False), 8,
                                         "uncontrolled", 96), None))
    out.append(("eng_horizon", engine_case("h", constant_workload(1, 64, 2, 32), 1,
                                           "uncontrolled", 16, horizon=50.0), None))
    out.append(("eng_trace_rows", engine_case("tr", constant_workload(4, 32, 8, 16), 2,
                                              "agent_cap:2", 2048,
                                              ctrl=ControllerConfig(control_interval=0.01)), None))
    out.append(("eng_summary", engine_case("sm", constant_workload(6, 32, 5, 16), 3,
                                           "uncontrolled", 220,
                                           ctrl=ControllerConfig(control_interval=0.05)), None))
    # randomized paranoid rounds (test_engine.cpp:315-352), discard-mode rounds
    for rnd in range(8):
        if rnd % 2 == 0:
            continue  # offload rounds: SURVEY.md §8(f) item 1
        wl = WorkloadConfig(agents=3 + rnd % 4, shared_prompt=rnd % 2 == 0,
                            prompt_tokens=8 + 8 * (rnd % 3), steps=2 + rnd % 3,
                            gen_tokens=Distribution("uniform", 2, 10),
                            obs_tokens=Distribution("uniform", 0, 6),
                            tool_latency=Distribution("lognormal", 0.05, 0.5),
                            tool_probability=0.5)
        pol = ["uncontrolled", f"request_cap:{1 + rnd % 3}", f"agent_cap:{1 + rnd % 3}",
               "aimd"][rnd % 4]
        ctrl = ControllerConfig(control_interval=0.03)
        if pol == "aimd":
            ctrl = ControllerConfig(control_interval=0.03, initial_window=2, w_max=6)
        s = engine_case(f"r{rnd}", wl, 100 + rnd, pol, 96 + 16 * (rnd % 5),
                        page=4 if rnd % 3 == 0 else 1, ctrl=ctrl, horizon=1e5)
        out.append((f"eng_random_{rnd}", s, None))
    return out


def random_scenarios(n: int = 24, seed: int = 0x5eed) -> list[tuple[str, Scenario, str]]:
    """Seeded random small configurations across every policy and page size."""
    rng = random.Random(seed)
    out = []
    for k in range(n):
        agents = rng.randint(1, 12)
        page = rng.choice([1, 2, 4, 16])
        shared = rng.random() < 0.5
        prompt = rng.choice([0, 8, 24, 64, 100])
        steps = rng.randint(1, 6)
        gen = rng.choice([Distribution("constant", rng.randint(1, 64)),
                          Distribution("uniform", 4, rng.randint(8, 96))])
        obs = rng.choice([Distribution("constant", 0), Distribution("uniform", 0, 40),
                          Distribution("lognormal", 20, 0.5)])
        tool = rng.choice([Distribution("constant", 0.05), Distribution("lognormal", 0.3, 0.4)])
        wl = WorkloadConfig(agents=agents, shared_prompt=shared, prompt_tokens=prompt,
                            steps=steps, gen_tokens=gen, obs_tokens=obs, tool_latency=tool,
                            tool_probability=rng.choice([0.0, 0.5, 1.0]))
        worst = prompt + steps * (96 + 80)
        cap_pages = max(4, int(worst / page * rng.uniform(1.1, 3.0)))
        pol = rng.choice(["uncontrolled", "aimd", f"agent_cap:{rng.randint(1, 4)}",
                          f"request_cap:{rng.randint(1, 4)}"])
        ctrl = ControllerConfig(control_interval=rng.choice([0.01, 0.05, 0.25]),
                                initial_window=rng.choice([0, 2]),
                                alpha=rng.choice([1.0, 2.0, 4.0]),
                                beta=rng.choice([0.3, 0.5, 0.9]),
                                u_low=rng.choice([0.1, 0.2]), u_high=rng.choice([0.4, 0.5, 0.8]),
                                h_thresh=rng.choice([0.2, 0.5, 0.9]),
                                signal_smoothing=rng.choice([0.0, 0.0, 0.5]))
        s = Scenario(name=f"rand{k}", seed=rng.randint(1, 10 ** 6), policy=pol)
        s.workload = wl
        s.engine = EngineParams(capacity=cap_pages, page_size=page,
                                hit_window_decay=rng.choice([0.0, 0.5, 0.9]), horizon=1e5)
        s.controller = ctrl
        s.cost = test_cost()
        out.append((f"rand_{k}", s, None))
    return out


def scaled(builder, agents, ratio=1.5, **kw):
    s = builder(agents=agents, capacity=1, **kw)
    pop_peak = _peak_tokens(s)
    s.engine.capacity = config.scaled_capacity(pop_peak, 16, ratio)
    return s


def _peak_tokens(s: Scenario) -> int:
    from tests.helpers import ref_population
    return ref_population(s)[4]


PRESET_ROWS = [
    ("smoke", ["uncontrolled", "aimd", "agent_cap:2", "request_cap:1"]),
    ("thrash", ["uncontrolled", "aimd", "request_cap:16", "agent_cap:8", "agent_cap:4",
                "agent_cap:32"]),
    ("ample", ["aimd", "uncontrolled"]),
    ("sweep-sensitivity", ["aimd"]),
    ("sweep-sensitivity-ulow", ["aimd"]),
]

CASES: list[dict] = []
for _name, _pols in PRESET_ROWS:
    for _p in _pols:
        CASES.append(dict(id=f"preset_{_name}_{_p}", preset=_name, policy=_p))
for _v in (0.4, 0.8):
    CASES.append(dict(id=f"preset_sweep-sensitivity_uhigh{_v}", preset="sweep-sensitivity",
                      policy="aimd", overrides={"controller.u_high": _v}))
for _v in (0.1, 0.5):
    CASES.append(dict(id=f"preset_sweep-sensitivity-ulow_ulow{_v}",
                      preset="sweep-sensitivity-ulow", policy="aimd",
                      overrides={"controller.u_low": _v}))
CASES += [dict(id="c1_uncontrolled", builder="c1", policy="uncontrolled"),
          dict(id="c1_aimd", builder="c1", policy="aimd")]
for _k in (0, 7, 100, 1500, 4095):
    CASES.append(dict(id=f"c4_sim{_k}", builder="c4", index=_k, policy="aimd"))
CASES += [dict(id="c2s64_aimd", builder="c2s", agents=64, policy="aimd"),
          dict(id="c2s64_uncontrolled", builder="c2s", agents=64, policy="uncontrolled",
               digests=False),
          dict(id="c3s128_aimd", builder="c3s", agents=128, policy="aimd"),
          dict(id="c3s128_aimd_h03", builder="c3s", agents=128, policy="aimd",
               overrides={"controller.h_thresh": 0.3}),
          dict(id="c3s128_uncontrolled", builder="c3s", agents=128, policy="uncontrolled",
               digests=False),
          dict(id="c5s256_aimd", builder="c5s", agents=256, policy="aimd", digests=False),
          dict(id="c5s256_cap64", builder="c5s", agents=256, policy="agent_cap:64",
               digests=False),
          dict(id="c2_aimd", builder="c2", policy="aimd", digests=False)]
for _id, _s, _p in _engine_tests() + random_scenarios():
    CASES.append(dict(id=_id, inline=_s, policy=_p))


def case_scenario(case: dict, presets: dict | None = None):
    """(Scenario, policy_text) for a case. `presets`: parsed preset dicts."""
    if "inline" in case:
        s = copy.deepcopy(case["inline"])
    elif "preset" in case:
        if presets is None:
            from tests.helpers import load_presets
            presets = load_presets()
        s = config.scenario_from_dict(presets[case["preset"]])
    else:
        b = case["builder"]
        if b == "c1":
            s = config.c1_toy(case["policy"])
        elif b == "c4":
            s = config.c4_sweep(case["index"] + 1)[case["index"]]
        elif b == "c2":
            s = config.c2_qwen(case["policy"])
        elif b == "c2s":
            s = config.c2_qwen(case["policy"], agents=case["agents"], capacity=1)
            s.engine.capacity = config.scaled_capacity(_peak_or_fixture(case, s))
        elif b == "c3s":
            s = config.c3_dsv3(case["policy"], agents=case["agents"], capacity=1)
            s.engine.capacity = config.scaled_capacity(_peak_or_fixture(case, s))
        elif b == "c5s":
            s = config.c5_stress(case["policy"], agents=case["agents"], capacity=1)
            s.engine.capacity = config.scaled_capacity(_peak_or_fixture(case, s))
        else:
            raise KeyError(b)
    for k, v in case.get("overrides", {}).items():
        section, _, name = k.partition(".")
        setattr(getattr(s, section), name, v)
    return s, case.get("policy")


def _peak_or_fixture(case, s):
    # peak aggregate tokens from the product's population builder (bit-identical
    # to the reference's, see tests/test_population.py); no GPU needed
    from paper_2601_22705_b200 import engine
    return engine.Population(s.workload, s.seed).peak_aggregate_tokens


def cache_fuzz_program(rounds: int = 40, ops: int = 300, seed: int = 0xacce97ed):
    """Randomized CacheTree op sequences in the spirit of acceptance criterion 2
    (acceptance.cpp:133-209) and test_cache_tree.cpp:276-340, over owner-form
    sequences: match/insert with engine-style pin/unpin, explicit evicts and
    suffix discards, small capacities so eviction is constant."""
    rng = random.Random(seed)
    progs = []
    for r in range(rounds):
        page = rng.choice([1, 2, 4, 16])
        agents = rng.randint(1, 6)
        shared = rng.random() < 0.5
        prompt = rng.choice([0, page * rng.randint(1, 4), rng.randint(1, 40)])
        maxlen = prompt + page * rng.randint(2, 12)
        cap = rng.randint(4, 40)
        lens = [prompt] * agents
        pins = {}  # agent -> pinned length (engine discipline: one pin per agent)
        prog_ops = []
        for _ in range(ops):
            a = rng.randrange(agents)
            roll = rng.random()
            if roll < 0.15 and lens[a] < maxlen:
                lens[a] = min(maxlen, lens[a] + rng.randint(1, 3 * page))
            if roll < 0.40:
                prog_ops.append((1, a, lens[a], 0))  # match
            elif roll < 0.70:
                prog_ops.append((2, a, lens[a], 0))  # insert
            elif roll < 0.82:
                prog_ops.append((3, 0, 0, rng.randint(1, 8)))  # evict
            elif roll < 0.90:
                # pin what is resident now: a match gives a node boundary
                prog_ops.append((1, a, lens[a], 0))
                prog_ops.append(("PIN_LAST_MATCH", a, lens[a], 0))
                pins.setdefault(a, []).append(None)
            elif roll < 0.96:
                if pins.get(a):
                    pins[a].pop()
                    prog_ops.append(("UNPIN_ONE", a, 0, 0))
                    continue
                prog_ops.append((1, a, lens[a], 0))
            else:
                prog_ops.append(("DISCARD_IF_UNPINNED", a, lens[a], prompt))
        progs.append(dict(capacity=cap, page_size=page, prompt=prompt, shared=int(shared),
                          agents=agents, ops=prog_ops, seed=r))
    return progs


# Full-size BASELINE configurations the reference finishes in seconds to
# minutes (tests/golden/make_golden_full.py -> full_runs.json). C5 is scaled
# (the full 65,536-agent shape cannot run on the CPU reference: SURVEY.md
# fact 0.3-6): 1,024 and 4,096 agents of the C5 shape, capacity = peak / 1.5.
FULL_CASES: list[dict] = [
    dict(id="c3_aimd_h03", builder="c3", policy="aimd",
         overrides={"controller.h_thresh": 0.3}),
    dict(id="c5s1024_aimd", builder="c5s", agents=1024, policy="aimd"),
    dict(id="c5s4096_aimd", builder="c5s", agents=4096, policy="aimd"),
    dict(id="c5s1024_cap256", builder="c5s", agents=1024, policy="agent_cap:256"),
    dict(id="c5s4096_cap1024", builder="c5s", agents=4096, policy="agent_cap:1024"),
]


def full_case_scenario(case: dict):
    if case["builder"] == "c3":
        s = config.c3_dsv3(case["policy"])
        for k, v in case.get("overrides", {}).items():
            section, _, name = k.partition(".")
            setattr(getattr(s, section), name, v)
        return s, case["policy"]
    return case_scenario(case)
