#!/usr/bin/env python
"""Benchmark of the B200 engine for the kvadmit simulator hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c4|c2|c1]

Default workload (BASELINE.json metric "simulated agent-steps/s & prefix-block
lookups/s at 1/2/4/8 B200 vs CPU ref"): C4, the 4096-simulation controller
sweep over the C1 toy trace (64 agents x 10 steps, Qwen3-32B KV sizing; grid
u_low x u_high x alpha x beta x h_thresh). One STEP = every
simulation of the sweep run to completion. Weak scaling: every rank runs its
own full 4096-sim sweep (workload seed 42 + rank); no data-path collective, one
NCCL gather of per-sim summary records at the end.

--impl reference runs the UNMODIFIED reference run_simulation (oracle/_ref,
compiled from /root/reference sources) on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

PEAKS_PATH = os.path.join(REPO, "MEASURED_PEAKS.json")
PROFILE_SUMMARY = os.path.join(REPO, "profiles", "ncu_summary.json")
METRIC = "simulated agent-steps/s & prefix-block lookups/s at 1/2/4/8 B200 vs CPU ref"
HBM_FALLBACK_GBS = 6650.0


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="c4", choices=["c4", "c2", "c3", "c3off", "c1"])
    p.add_argument("--sims", type=int, default=4096)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=2)
    return p.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# --------------------------------------------------------------------------- workloads

def build_scenarios(workload: str, rank: int, sims: int):
    from paper_2601_22705_b200 import sweep
    scen = sweep.weak_shard(workload, rank, sims)
    if workload == "c4":
        desc = (f"C4 controller sweep: {sims} sims of C1 (64 agents x 10 steps, private 1024-token "
                f"prompts, 12,629-page cache, Qwen3-32B KV sizing), workload seed {42 + rank}")
    elif workload == "c2":
        desc = "C2: 1024 agents x 16 steps, 4K->55.7K contexts, 2,038,926-page cache, aimd"
    elif workload == "c3":
        desc = ("C3: DeepSeek-V3 MLA sizing, 2048 agents x 10 steps, 613,697-page cache, "
                "aimd h_thresh=0.3")
    elif workload == "c3off":
        desc = ("C3 shape, offload tier: 32 agents x 10 steps, scaled cache (peak/1.5), "
                "uncontrolled admission + offload eviction (PCIe 25 GB/s link model)")
    else:
        desc = "C1 toy: 64 agents x 10 steps, aimd"
    return scen, desc


def make_specs(scen):
    from paper_2601_22705_b200 import engine
    cache = {}
    specs = []
    for s in scen:
        key = (s.seed, repr(s.workload))
        if key not in cache:
            cache[key] = engine.Population(s.workload, s.seed)
        specs.append(engine.SimSpec.from_scenario(s, population=cache[key]))
    return specs, cache


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for name, flag in zip(names, r[4:8]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        under = [x for x in sm if mx and x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(under) if under else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------------------- helpers

def algorithmic_bytes(results, tree: bool = False) -> dict:
    """SURVEY.md §8(d) / BASELINE.md §2 per-unit byte counts. Offload mode
    (tree=True): an eviction select reads one 64 B node record per pool entry."""
    look = sum(16 * r.lookups + 8 * r.hit_pages for r in results)
    ins = sum(16 * r.created_pages + 8 * r.refreshed_pages for r in results)
    ev = sum((64 if tree else 8) * r.evict_scanned + 16 * r.evicted_pages for r in results)
    state = sum(192 * r.agent_events for r in results)
    tick = sum(88 * r.ticks for r in results)
    return dict(lookup=look, insert=ins, evict=ev, state=state, tick=tick,
                total=look + ins + ev + state + tick)


def load_peak():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def load_traffic(workload):
    try:
        with open(PROFILE_SUMMARY) as fh:
            d = json.load(fh)
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_sample(workload: str, scen):
    """Bounded CPU sample of a workload (all current workloads run whole)."""
    return scen, None


def cpu_reference(scen, threads: int, sample_every: int = 1):
    """The reference's own run_simulation on host cores (oracle/_ref)."""
    import ctypes as C

    from paper_2601_22705_b200 import abi
    from tests.helpers import ref_lib
    lib = ref_lib()
    chosen = scen[::sample_every]
    n = len(chosen)
    wls = (abi.WorkloadConfig * n)()
    seeds = (C.c_uint64 * n)()
    pols = (abi.Policy * n)()
    costs = (abi.CostParams * n)()
    engs = (abi.EngineParams * n)()
    for i, s in enumerate(chosen):
        pol, eng = s.resolved()
        wls[i] = s.workload.to_abi()
        seeds[i] = s.seed
        pols[i] = pol
        costs[i] = s.cost.to_abi()
        engs[i] = eng.to_abi()
    mk = (C.c_double * n)()
    dec = (C.c_uint64 * n)()
    wall = C.c_double()
    rc = lib.kvr_run_many(n, wls, seeds, pols, costs, engs, threads, mk, dec, C.byref(wall))
    if rc != 0:
        raise RuntimeError(lib.kvr_last_error().decode())
    steps = sum(s.workload.agents * s.workload.steps for s in chosen)
    return steps, wall.value, n


# --------------------------------------------------------------------------- arms

def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    scen, desc = build_scenarios(args.workload, 0, args.sims)
    scen, note = cpu_sample(args.workload, scen)
    threads = os.cpu_count() or 1
    # bounded sample per step so --steps K --warmup W finishes within minutes
    every = {"c4": 8}.get(args.workload, 1)
    for _ in range(args.warmup if args.workload in ("c4", "c1") else 0):
        cpu_reference(scen, threads, every)
    vals, walls = [], []
    steps = n = 0
    for _ in range(args.steps):
        steps, wall, n = cpu_reference(scen, threads, every)
        vals.append(steps / wall)
        walls.append(wall)
    value = sum(steps for _ in walls) / sum(walls)
    sample = (f"{n} of the {len(scen)} simulations (every {every}th) per step, reference "
              f"run_simulation on {threads} threads" if every > 1 else
              f"all {n} simulation(s) per step on {threads} threads")
    if note:
        sample = note + "; " + sample
    line = {"metric": METRIC, "value": value, "unit": "agent-steps/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.mean(walls), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64/u64",
            "data": "synthetic (reference seeded workload generator)",
            "config": {"workload": desc},
            "cpu_baseline": {"value": value, "unit": "agent-steps/s", "cores": threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "agent-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import ctypes as C

    import torch

    from paper_2601_22705_b200 import abi, engine
    rank, world, local = env_rank()
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    scen, desc = build_scenarios(args.workload, rank, args.sims)
    specs, pops = make_specs(scen)
    batch = engine.Batch(specs, device=device)
    for _ in range(max(args.warmup, 1)):
        batch.run()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(device)).split(",")[0])
                           if os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[0].isdigit()
                           else device)
    sampler.start()
    step_ms = kern_ms = 0.0
    per_step = []
    for _ in range(args.steps):
        batch.run()
        a, k = batch.timing()
        step_ms += a
        kern_ms += k
        per_step.append(a)
    torch.cuda.synchronize()
    sampler.stop()
    results = batch.results_raw()
    units = sum(r.agent_steps for r in results)          # per step, this rank
    lookups = sum(r.lookups for r in results)
    bad = [i for i, r in enumerate(results) if r.status != 0]
    tot = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device="cuda")
    cnt = torch.tensor([units, lookups], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    max_ms, max_kms = tot.tolist()
    all_units, all_lookups = cnt.tolist()
    value = all_units * args.steps / (max_ms / 1e3)
    # ---- NCCL final metric gather: per-sim summary records of every rank
    from paper_2601_22705_b200 import sweep
    summary = sweep.gather_records(sweep.records(results), dist, device="cuda")
    makespans = summary[:, 0].cpu().tolist()
    # ---- roofline of the engine kernel
    ab = algorithmic_bytes(results, tree=args.workload == "c3off")
    kernel_s = (kern_ms / args.steps) / 1e3
    peak, peak_kind = load_peak()
    achieved = ab["total"] / kernel_s / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": load_traffic(args.workload),
            "peak_source": peak_kind, "kernel": "kvg::engine_kernel_small" if len(specs) >= 296
            else "kvg::engine_kernel_big",
            "algorithmic_bytes_per_launch": ab,
            "kernel_ms_per_launch": kern_ms / args.steps}
    # ---- end to end through the C ABI with host buffers: every step creates
    # the batch from host populations (H2D), runs it, and the kernel streams
    # results / trace rows / agent stats into pinned host memory (D2H)
    # the device-resident batch goes back to the workspace cache first, so the
    # e2e batches reuse its HBM arena (and, after one untimed step, the pinned
    # host block) like any repeated caller would
    batch.close()
    e2e_ms = []
    n_agents = sum(s.population.c.agents for s in specs)
    h2d = sum(p.c.agents * p.c.steps * C.sizeof(abi.StepPlan) for p in pops.values()) + \
        len(specs) * 512
    d2h = 0
    phases = {"create_ms": 0.0, "run_ms": 0.0, "results_ms": 0.0, "kernel_ms": 0.0}
    for k in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b2 = engine.Batch(specs, device=device, host_outputs=True)
        t1 = time.perf_counter()
        b2.run()
        t2 = time.perf_counter()
        kern_e2e = b2.timing()[1]  # the run's kernel span (rows stream out inside it)
        res2 = b2.results_array()
        d2h = int(res2["ticks"].sum()) * C.sizeof(abi.TraceRow) + \
            n_agents * C.sizeof(abi.AgentStats) + len(res2) * C.sizeof(abi.SimResult)
        b2.close()
        t3 = time.perf_counter()
        if k > 0:  # step 0 is the untimed warm-up (first pinned allocation)
            e2e_ms.append(1e3 * (t3 - t0))
            phases["create_ms"] += 1e3 * (t1 - t0) / args.e2e_steps
            phases["run_ms"] += 1e3 * (t2 - t1) / args.e2e_steps
            phases["results_ms"] += 1e3 * (t3 - t2) / args.e2e_steps
            phases["kernel_ms"] += kern_e2e / args.e2e_steps
    e2e_t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = all_units * len(e2e_ms) / (e2e_t.item() / 1e3)
    # ---- CPU baseline (rank 0, N=1): the reference on the host cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        every = 8 if args.workload == "c4" else 1
        try:
            cscen, note = cpu_sample(args.workload, scen)
            steps_cpu, wall, n = cpu_reference(cscen, threads, every)
            cpu = {"value": steps_cpu / wall, "unit": "agent-steps/s", "cores": threads,
                   "kind": "reference",
                   "sample": (note + "; " if note else "") +
                   f"{n} of {len(cscen)} simulations (every {every}th), unmodified "
                   f"reference run_simulation, {threads} threads, {wall:.2f} s"}
        except Exception as e:  # the reference build travels with the repo; report if absent
            cpu = {"value": None, "unit": "agent-steps/s", "cores": threads,
                   "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "agent-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64/u64", "data": "synthetic (seeded reference workload generator)",
            "config": {"workload": desc, "sims_per_gpu": len(specs),
                       "parallelism": f"independent sims sharded over {world} GPU(s)",
                       "l2": "inputs larger than L2: per-sim hash tables total "
                             f"{batch_bytes(specs) / 2**30:.1f} GiB, re-initialised every step"},
            "lookups_per_s": all_lookups * args.steps / (max_ms / 1e3),
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "agent-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "phases_ms": {k: round(v, 2) for k, v in phases.items()}},
            "gpu_launches": args.steps * launches_per_step(specs),
            "clocks": sampler.summary(),
            "parity": {"sims": len(summary), "nonzero_status": len(bad),
                       "makespan_min": min(makespans), "makespan_max": max(makespans)},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def batch_bytes(specs):
    from paper_2601_22705_b200.abi import table_bytes
    return sum(table_bytes(s.engine.capacity, s.population.c.agents) for s in specs)


def launches_per_step(specs):
    # one engine-kernel launch per warps-per-sim group (uniform workloads: 1)
    return 1


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
