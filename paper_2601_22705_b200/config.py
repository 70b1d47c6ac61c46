"""Scenario configuration — host-side mirror of the reference config seam.

Mirrors kvadmit::ScenarioConfig (/root/reference/proj/src/config.hpp:44-64)
and the defaults it binds: ControllerConfig (controller.hpp:29-42),
reference_cost_params (cost_model.cpp:49-59), EngineParams (engine.hpp:29-41),
PhaseParams (metrics.hpp:57-63). The preset files are TOML-subset documents
(config.cpp:249-286), which Python's tomllib reads unchanged; unknown keys are
rejected like bind_entry does (config.cpp:533-555).

Also defines the BASELINE.json configurations C1..C5.
"""
from __future__ import annotations

import copy
import math
import tomllib
from dataclasses import dataclass, field

from . import abi


class ConfigError(ValueError):
    """Bad or inconsistent configuration (errors.hpp:21-24)."""


@dataclass
class Distribution:
    kind: str = "constant"  # constant | uniform | lognormal
    a: float = 0.0
    b: float = 0.0

    def to_abi(self) -> abi.Distribution:
        k = {"constant": abi.DIST_CONSTANT, "uniform": abi.DIST_UNIFORM,
             "lognormal": abi.DIST_LOGNORMAL}[self.kind]
        return abi.Distribution(kind=k, a=float(self.a), b=float(self.b))


@dataclass
class WorkloadConfig:
    agents: int = 1
    shared_prompt: bool = True
    prompt_tokens: int = 0
    steps: int = 1
    gen_tokens: Distribution = field(default_factory=Distribution)
    obs_tokens: Distribution = field(default_factory=Distribution)
    tool_latency: Distribution = field(default_factory=Distribution)
    tool_probability: float = 1.0

    def to_abi(self) -> abi.WorkloadConfig:
        return abi.WorkloadConfig(
            agents=self.agents, shared_prompt=int(self.shared_prompt),
            prompt_tokens=self.prompt_tokens, steps=self.steps,
            gen_tokens=self.gen_tokens.to_abi(), obs_tokens=self.obs_tokens.to_abi(),
            tool_latency=self.tool_latency.to_abi(),
            tool_probability=float(self.tool_probability))


@dataclass
class ControllerConfig:
    alpha: float = 2.0
    beta: float = 0.5
    u_low: float = 0.2
    u_high: float = 0.5
    h_thresh: float = 0.2
    w_min: float = 1.0
    w_max: float = 0.0
    initial_window: float = 0.0
    control_interval: float = 0.25
    signal_smoothing: float = 0.0

    def to_abi(self) -> abi.ControllerConfig:
        return abi.ControllerConfig(**{k: float(getattr(self, k)) for k in (
            "alpha", "beta", "u_low", "u_high", "h_thresh", "w_min", "w_max",
            "initial_window", "control_interval", "signal_smoothing")})


@dataclass
class CostParams:
    prefill_linear: float = 5e-5
    prefill_quadratic: float = 5e-8
    decode_base: float = 2e-3
    decode_context: float = 2e-8
    bytes_per_token: float = 6.67e9 / 4096.0
    pcie_bandwidth: float = 25e9
    transfer_sync_overhead: float = 0.05

    def to_abi(self) -> abi.CostParams:
        return abi.CostParams(**{k: float(getattr(self, k)) for k in (
            "prefill_linear", "prefill_quadratic", "decode_base", "decode_context",
            "bytes_per_token", "pcie_bandwidth", "transfer_sync_overhead")})


@dataclass
class EngineParams:
    capacity: int = 0
    page_size: int = 1
    eviction: str = "discard"
    hit_window_decay: float = 0.0
    horizon: float = 1e6
    sat_threshold: float = 0.8
    hit_threshold: float = 0.5
    hysteresis: int = 3

    def to_abi(self) -> abi.EngineParams:
        return abi.EngineParams(
            capacity=self.capacity, page_size=self.page_size,
            eviction=abi.EVICT_OFFLOAD if self.eviction == "offload" else abi.EVICT_DISCARD,
            paranoid=0, hit_window_decay=float(self.hit_window_decay),
            horizon=float(self.horizon),
            phases=abi.PhaseParams(sat_threshold=float(self.sat_threshold),
                                   hit_threshold=float(self.hit_threshold),
                                   hysteresis=int(self.hysteresis)))


def parse_policy(text: str, aimd: ControllerConfig) -> abi.Policy:
    """Mirror of parse_policy (controller.cpp:213-253) returning the ABI struct."""
    head, _, arg = text.partition(":")
    kinds = {"uncontrolled": abi.POLICY_UNCONTROLLED, "request_cap": abi.POLICY_REQUEST_CAP,
             "agent_cap": abi.POLICY_AGENT_CAP, "aimd": abi.POLICY_AIMD}
    if head not in kinds:
        raise ConfigError(f"unknown policy '{text}'")
    kind = kinds[head]
    cap = 1
    if kind in (abi.POLICY_REQUEST_CAP, abi.POLICY_AGENT_CAP):
        if not arg:
            raise ConfigError(f"policy '{head}' needs a cap, e.g. {head}:8")
        if not arg.isdigit() or int(arg) < 1:
            raise ConfigError(f"bad cap in policy '{text}'")
        cap = int(arg)
    elif arg:
        raise ConfigError(f"policy '{head}' takes no argument")
    return abi.Policy(kind=kind, cap=cap, aimd=aimd.to_abi())


@dataclass
class Scenario:
    name: str = "run"
    seed: int = 1
    policy: str = "uncontrolled"
    workload: WorkloadConfig = field(default_factory=WorkloadConfig)
    engine: EngineParams = field(default_factory=EngineParams)
    controller: ControllerConfig = field(default_factory=ControllerConfig)
    cost: CostParams = field(default_factory=CostParams)
    compare: dict | None = None
    sweep: dict | None = None

    def resolved(self, policy_text: str | None = None):
        """(policy, engine) for a row, like resolve_run (experiment.cpp:145-157):
        the pseudo-policy "offload" is uncontrolled admission + offload eviction."""
        text = policy_text or self.policy
        eng = copy.deepcopy(self.engine)
        if text == "offload":
            pol = parse_policy("uncontrolled", self.controller)
            eng.eviction = "offload"
        else:
            pol = parse_policy(text, self.controller)
        return pol, eng

    def with_overrides(self, **kv) -> "Scenario":
        s = copy.deepcopy(self)
        for key, val in kv.items():
            section, _, name = key.rpartition(".")
            obj = s if not section else getattr(s, section)
            if not hasattr(obj, name):
                raise ConfigError(f"unknown key {key}")
            setattr(obj, name, val)
        return s


def _dist(v, path) -> Distribution:
    if isinstance(v, (int, float)) and not isinstance(v, bool):
        return Distribution("constant", float(v))
    if not isinstance(v, dict) or "dist" not in v:
        raise ConfigError(f"{path}: expected a number or {{dist=...}} table")
    d = v["dist"]
    if d == "constant":
        return Distribution("constant", float(v["value"]))
    if d == "uniform":
        return Distribution("uniform", float(v["min"]), float(v["max"]))
    if d == "lognormal":
        return Distribution("lognormal", float(v["mean"]), float(v["sigma"]))
    raise ConfigError(f"{path}: unknown distribution '{d}'")


_WL = {"agents", "shared_prompt", "prompt_tokens", "steps", "gen_tokens",
       "obs_tokens", "tool_latency", "tool_probability"}
_CACHE = {"capacity", "page_size", "eviction", "hit_window_decay"}
_CTRL = {"alpha", "beta", "u_low", "u_high", "h_thresh", "w_min", "w_max",
         "initial_window", "control_interval", "signal_smoothing"}
_COST = {"prefill_linear", "prefill_quadratic", "decode_base", "decode_context",
         "bytes_per_token", "pcie_bandwidth", "transfer_sync_overhead",
         "crossover_concurrency"}
_PHASES = {"sat_threshold", "hit_threshold", "hysteresis"}


def parse_scenario(text: str, origin: str = "<memory>") -> Scenario:
    doc = tomllib.loads(text)
    s = Scenario()
    for key, val in doc.items():
        if isinstance(val, dict) and key in ("workload", "cache", "controller",
                                             "cost", "phases", "compare", "sweep"):
            continue
        if key == "name":
            s.name = str(val)
        elif key == "seed":
            s.seed = int(val)
        elif key == "policy":
            s.policy = str(val)
        elif key == "horizon":
            s.engine.horizon = float(val)
        elif key == "output_dir":
            pass
        else:
            raise ConfigError(f"{origin}: {key}: unknown key")
    for k, v in doc.get("workload", {}).items():
        if k not in _WL:
            raise ConfigError(f"{origin}: workload.{k}: unknown key")
        if k in ("gen_tokens", "obs_tokens", "tool_latency"):
            setattr(s.workload, k, _dist(v, f"workload.{k}"))
        elif k == "shared_prompt":
            s.workload.shared_prompt = bool(v)
        elif k == "tool_probability":
            s.workload.tool_probability = float(v)
        else:
            setattr(s.workload, k, int(v))
    for k, v in doc.get("cache", {}).items():
        if k not in _CACHE:
            raise ConfigError(f"{origin}: cache.{k}: unknown key")
        setattr(s.engine, k, v if k == "eviction" else (float(v) if k == "hit_window_decay" else int(v)))
    for k, v in doc.get("controller", {}).items():
        if k not in _CTRL:
            raise ConfigError(f"{origin}: controller.{k}: unknown key")
        setattr(s.controller, k, float(v))
    for k, v in doc.get("cost", {}).items():
        if k not in _COST:
            raise ConfigError(f"{origin}: cost.{k}: unknown key")
        if k != "crossover_concurrency":
            setattr(s.cost, k, float(v))
    for k, v in doc.get("phases", {}).items():
        if k not in _PHASES:
            raise ConfigError(f"{origin}: phases.{k}: unknown key")
        setattr(s.engine, k, int(v) if k == "hysteresis" else float(v))
    s.compare = doc.get("compare")
    s.sweep = doc.get("sweep")
    return s


def load_scenario(path: str) -> Scenario:
    with open(path, "rb") as f:
        return parse_scenario(f.read().decode(), path)


# ---------------------------------------------------------------------------
# BASELINE.json configurations. Page size 16, decay 0.9,
# controller defaults, reference cost calibration unless stated.

QWEN3_32B_BYTES_PER_TOKEN = 262144.0         # 64 layers x 8 KV heads x 128 x 2 x 2 B
DSV3_BYTES_PER_TOKEN = 1628417.96875         # 6.67 GB / 4096


def c1_toy(policy: str = "aimd") -> Scenario:
    s = Scenario(name="c1_toy", seed=42, policy=policy)
    s.workload = WorkloadConfig(agents=64, shared_prompt=False, prompt_tokens=1024,
                                steps=10, gen_tokens=Distribution("constant", 256),
                                obs_tokens=Distribution("constant", 128),
                                tool_latency=Distribution("lognormal", 2.0, 0.35),
                                tool_probability=1.0)
    s.engine = EngineParams(capacity=12629, page_size=16, hit_window_decay=0.9)
    s.controller = ControllerConfig(initial_window=2, control_interval=0.25)
    s.cost = CostParams(bytes_per_token=QWEN3_32B_BYTES_PER_TOKEN)
    return s


def c2_qwen(policy: str = "aimd", agents: int = 1024, capacity: int = 2038926) -> Scenario:
    s = Scenario(name="c2_qwen3_32b", seed=7, policy=policy)
    s.workload = WorkloadConfig(agents=agents, shared_prompt=True, prompt_tokens=4096,
                                steps=16, gen_tokens=Distribution("uniform", 256, 1024),
                                obs_tokens=Distribution("uniform", 2000, 3000),
                                tool_latency=Distribution("lognormal", 2.0, 0.35),
                                tool_probability=1.0)
    s.engine = EngineParams(capacity=capacity, page_size=16, hit_window_decay=0.9)
    s.controller = ControllerConfig(initial_window=2, control_interval=0.25)
    s.cost = CostParams(bytes_per_token=QWEN3_32B_BYTES_PER_TOKEN)
    return s


def c3_dsv3(policy: str = "aimd", agents: int = 2048, capacity: int = 613697) -> Scenario:
    s = Scenario(name="c3_deepseek_v3", seed=3, policy=policy)
    s.workload = WorkloadConfig(agents=agents, shared_prompt=True, prompt_tokens=2048,
                                steps=10, gen_tokens=Distribution("uniform", 128, 384),
                                obs_tokens=Distribution("lognormal", 512, 0.5),
                                tool_latency=Distribution("lognormal", 2.0, 0.35),
                                tool_probability=1.0)
    s.engine = EngineParams(capacity=capacity, page_size=16, hit_window_decay=0.9)
    s.controller = ControllerConfig(initial_window=2, control_interval=0.25)
    s.cost = CostParams(bytes_per_token=DSV3_BYTES_PER_TOKEN, pcie_bandwidth=25e9)
    return s


C4_U_LOW = (0.05, 0.1, 0.15, 0.2, 0.25, 0.3, 0.35, 0.4)
C4_U_HIGH = (0.4, 0.45, 0.5, 0.55, 0.6, 0.7, 0.8, 0.9)
C4_ALPHA = (1.0, 2.0, 4.0, 8.0)
C4_BETA = (0.3, 0.5, 0.7, 0.9)
C4_H = (0.2, 0.4)


def c4_grid(k: int) -> dict:
    """Controller parameters of sweep sim k."""
    return dict(u_low=C4_U_LOW[k % 8], u_high=C4_U_HIGH[(k // 8) % 8],
                alpha=C4_ALPHA[(k // 64) % 4], beta=C4_BETA[(k // 256) % 4],
                h_thresh=C4_H[(k // 1024) % 2])


def c4_sweep(n: int = 4096, seed: int = 42) -> list[Scenario]:
    out = []
    for k in range(n):
        s = c1_toy("aimd")
        s.name = f"c4_{k}"
        s.seed = seed
        for key, v in c4_grid(k).items():
            setattr(s.controller, key, v)
        out.append(s)
    return out


def c5_stress(policy: str = "aimd", seed: int = 5, agents: int = 65536,
              capacity: int = 16777216) -> Scenario:
    s = Scenario(name="c5_stress", seed=seed, policy=policy)
    s.workload = WorkloadConfig(agents=agents, shared_prompt=True, prompt_tokens=8192,
                                steps=16, gen_tokens=Distribution("uniform", 512, 1536),
                                obs_tokens=Distribution("uniform", 3000, 6000),
                                tool_latency=Distribution("lognormal", 2.0, 0.35),
                                tool_probability=1.0)
    s.engine = EngineParams(capacity=capacity, page_size=16, hit_window_decay=0.9)
    s.controller = ControllerConfig(initial_window=2, control_interval=0.25)
    s.cost = CostParams(bytes_per_token=QWEN3_32B_BYTES_PER_TOKEN)
    return s


def scaled_capacity(peak_tokens: int, page: int = 16, ratio: float = 1.5) -> int:
    return int(math.floor(peak_tokens / page / ratio))


def scenario_to_dict(s: Scenario) -> dict:
    from dataclasses import asdict
    return asdict(s)


def scenario_from_dict(d: dict) -> Scenario:
    s = Scenario(name=d["name"], seed=d["seed"], policy=d["policy"],
                 compare=d.get("compare"), sweep=d.get("sweep"))
    w = dict(d["workload"])
    for k in ("gen_tokens", "obs_tokens", "tool_latency"):
        w[k] = Distribution(**w[k])
    s.workload = WorkloadConfig(**w)
    s.engine = EngineParams(**d["engine"])
    s.controller = ControllerConfig(**d["controller"])
    s.cost = CostParams(**d["cost"])
    return s
