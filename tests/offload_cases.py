"""Offload-mode parity catalogue (the reference's
EvictionMode::kOffload, cache_tree.cpp:270-368, engine.cpp:156-182, 337-360).

Offload runs exercise the node-level bookkeeping the reference gets wrong in
its own invariant checker: reload self-eviction leaves device nodes below
host nodes (quirk Q1) and re-promotion double-counts children_with_device.
The cases below hit both thousands of times; the golden fixtures come from
the unmodified reference (tests/golden/make_golden_offload.py)."""
from __future__ import annotations

import copy
import random

from paper_2601_22705_b200 import config
from paper_2601_22705_b200.config import ControllerConfig, Distribution, WorkloadConfig
from tests.golden_cases import engine_case, random_scenarios


def _offload(s, policy=None):
    s = copy.deepcopy(s)
    s.engine.eviction = "offload"
    if policy is not None:
        s.policy = policy
    return s


def _cases():
    out = [dict(id="off_preset_smoke", preset="smoke", policy="offload"),
           dict(id="off_preset_thrash", preset="thrash", policy="offload"),
           dict(id="off_preset_ample", preset="ample", policy="offload")]
    # the randomized rounds test_engine.cpp:315-352 runs in offload mode
    for rnd in range(0, 8, 2):
        wl = WorkloadConfig(agents=3 + rnd % 4, shared_prompt=rnd % 2 == 0,
                            prompt_tokens=8 + 8 * (rnd % 3), steps=2 + rnd % 3,
                            gen_tokens=Distribution("uniform", 2, 10),
                            obs_tokens=Distribution("uniform", 0, 6),
                            tool_latency=Distribution("lognormal", 0.05, 0.5),
                            tool_probability=0.5)
        pol = ["uncontrolled", f"request_cap:{1 + rnd % 3}", f"agent_cap:{1 + rnd % 3}",
               "aimd"][rnd % 4]
        ctrl = ControllerConfig(control_interval=0.03)
        s = engine_case(f"r{rnd}", wl, 100 + rnd, pol, 96 + 16 * (rnd % 5),
                        page=4 if rnd % 3 == 0 else 1, ctrl=ctrl, horizon=1e5)
        out.append(dict(id=f"off_eng_random_{rnd}", inline=_offload(s), policy=None))
    for name, s, _ in random_scenarios(16, seed=0x0ff10ad):
        out.append(dict(id=f"off_{name}", inline=_offload(s), policy=None))
    for ag in (8, 16, 32, 64):
        out.append(dict(id=f"off_c3s{ag}", builder="c3s", agents=ag, policy="offload"))
    out.append(dict(id="off_c3s32_aimd", builder="c3s", agents=32, policy="aimd",
                    eviction="offload"))
    out.append(dict(id="off_c1_offload", builder="c1", policy="offload"))
    return out


OFFLOAD_CASES = _cases()


def offload_scenario(case, presets=None):
    from tests.golden_cases import case_scenario
    s, pol = case_scenario(case, presets)
    if case.get("eviction") == "offload":
        s.engine.eviction = "offload"
    return s, pol


def offload_fuzz_programs(rounds: int = 30, ops: int = 250, seed: int = 0x0ff1):
    """Engine-style offload CacheTree programs: match -> pin(matched) ->
    [reload(from=matched, max=host_matched) -> pin/unpin] -> insert ->
    pin(stored)/unpin, with random explicit evicts and suffix discards, over
    small capacities (so reloads self-evict: quirk Q1). Ops that depend on a
    previous result are symbolic; the generator resolves them against the
    reference and records the concrete program."""
    rng = random.Random(seed)
    progs = []
    for r in range(rounds):
        page = rng.choice([1, 2, 4])
        agents = rng.randint(1, 5)
        shared = rng.random() < 0.6
        prompt = rng.choice([page * rng.randint(1, 4), rng.randint(1, 20)])
        maxlen = prompt + page * rng.randint(4, 14)
        cap = rng.randint(6, 40)
        prog = []
        lens = [prompt] * agents
        for _ in range(ops):
            a = rng.randrange(agents)
            roll = rng.random()
            if roll < 0.2 and lens[a] < maxlen:
                lens[a] = min(maxlen, lens[a] + rng.randint(1, 3 * page))
            if roll < 0.70:
                prog.append(("STEP", a, lens[a], 0))        # engine dispatch_member
            elif roll < 0.85:
                prog.append((3, 0, 0, rng.randint(1, 6)))    # evict
            elif roll < 0.93:
                prog.append(("RELEASE", a, 0, 0))            # unpin the agent's pin
            else:
                prog.append(("DISCARD_IF_UNPINNED", a, lens[a], prompt))
        progs.append(dict(capacity=cap, page_size=page, prompt=prompt, shared=int(shared),
                          agents=agents, ops=prog, seed=r))
    return progs
