"""Multi-GPU plumbing for independent simulations.

Simulations never exchange data while they run, so GPUs shard them with no
data-path collective: rank r of N owns its own slice of the sweep and, at the
end, ONE all_gather moves fixed-size per-simulation summary records to every
rank (NCCL over NVLink on the GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

from . import config

RECORD_FIELDS = ("makespan", "agent_steps", "lookups", "status", "decoded_tokens",
                 "recompute_tokens", "stall_events", "ticks")


def weak_shard(workload: str, rank: int, sims: int):
    """Weak scaling: every rank runs a full sweep of `sims` simulations; rank r
    draws its workload with seed base + r (rank 0 = the BASELINE config)."""
    if workload == "c4":
        return config.c4_sweep(sims, seed=42 + rank)
    if workload == "c2":
        s = config.c2_qwen("aimd")
        s.seed = 7 + rank
        return [s]
    if workload == "c3":  # DeepSeek-V3 MLA sizing, the controlled AIMD row (h_thresh 0.3)
        s = config.c3_dsv3("aimd")
        s.controller.h_thresh = 0.3
        s.seed = 3 + rank
        return [s]
    if workload == "c3off":  # offload tier on the 32-agent C3 shape (the reference's
        # offload runs take minutes from 128 agents on; the full size exceeds the horizon)
        s = config.c3_dsv3("offload", agents=32, capacity=1)
        s.seed = 3 + rank  # before the capacity: it is this rank's population peak
        from . import engine
        s.engine.capacity = config.scaled_capacity(
            engine.Population(s.workload, s.seed).peak_aggregate_tokens)
        return [s]
    s = config.c1_toy("aimd")
    s.seed = 42 + rank
    return [s]


def strong_shard(scenarios: list, rank: int, world: int) -> list:
    """Strong scaling: a fixed list split into contiguous slices (sim i -> rank
    i * world // len)."""
    n = len(scenarios)
    lo, hi = rank * n // world, (rank + 1) * n // world
    return scenarios[lo:hi]


def records(results) -> list[list[float]]:
    """Fixed-size summary record per simulation (what the final gather moves)."""
    out = []
    for r in results:
        get = (lambda k: r[k]) if isinstance(r, dict) else (lambda k: getattr(r, k))
        out.append([float(get(k)) for k in RECORD_FIELDS])
    return out


def gather_records(recs: list[list[float]], dist=None, device="cpu"):
    """All-gather the per-sim records of every rank (one collective)."""
    import torch
    t = torch.tensor(recs, dtype=torch.float64, device=device).reshape(-1, len(RECORD_FIELDS))
    if dist is None:
        return t
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(sizes, n)
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros((mx, t.shape[1]), dtype=t.dtype, device=device)
    pad[: t.shape[0]] = t
    bufs = [torch.zeros_like(pad) for _ in sizes]
    dist.all_gather(bufs, pad)
    return torch.cat([b[: int(s.item())] for b, s in zip(bufs, sizes)])
