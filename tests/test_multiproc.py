"""World-size-2 gloo run of the multi-GPU plumbing on CPU: each rank owns its
shard of a sweep (weak and strong splits), computes it (here with the CPU
oracle standing in for the device), and the single all_gather of summary
records reproduces the serial run exactly on every rank."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_22705_b200 import config, engine, sweep


def _small_sweep(n=6):
    out = []
    for k in range(n):
        s = config.c1_toy("aimd")
        s.workload.agents = 6
        s.workload.steps = 3
        s.engine.capacity = 600
        for key, v in config.c4_grid(k * 37).items():
            setattr(s.controller, key, v)
        out.append(s)
    return out


def _run(scen):
    from tests.helpers import oracle_run
    res = []
    for s in scen:
        pop = engine.Population(s.workload, s.seed)
        res.append(oracle_run(s, pop=pop.c)["result"])
    return sweep.records(res)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = sweep.strong_shard(_small_sweep(), rank, world)
        strong = sweep.gather_records(_run(mine), dist)
        weak = sweep.gather_records(_run([_shrink(sweep.weak_shard("c1", rank, 1)[0])]), dist)
        q.put((rank, strong.tolist(), weak.tolist()))
    finally:
        dist.destroy_process_group()


def _shrink(s):
    s.workload.agents = 4
    s.workload.steps = 2
    s.engine.capacity = 400
    return s


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
def test_gloo_world2_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict()
    for _ in procs:
        r, strong, weak = q.get(timeout=240)
        got[r] = (strong, weak)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    serial = _run(_small_sweep())
    assert got[0][0] == serial and got[1][0] == serial
    weak_serial = _run([_shrink(sweep.weak_shard("c1", r, 1)[0]) for r in range(2)])
    assert got[0][1] == weak_serial and got[1][1] == weak_serial
    # rank 1's weak shard is a different workload (seed 43), not a copy of rank 0's
    assert weak_serial[0] != weak_serial[1]


def test_bench_strong_split_partitions_the_c4_sweep():
    import bench
    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            args = bench.parse_args(["--split", "strong", "--gpus", str(world)])
            scen, desc = bench.build_scenarios(args, r, world)
            seen += [s.name for s in scen]
            assert len(scen) == 4096 // world and f"[{r * 4096 // world}," in desc
        assert seen == [f"c4_{k}" for k in range(4096)]


def test_bench_c5_replicas_one_per_rank():
    import bench
    args = bench.parse_args(["--workload", "c5"])
    got = [(s.policy, s.seed) for r in range(8) for s in bench.build_scenarios(args, r, 8)[0]]
    assert got == bench.C5_REPLICAS and len(set(got)) == 8


@pytest.mark.timeout(600)
def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun re-executes itself as a 2-rank
    torch.distributed job (the path the driver's --gpus N takes); the CPU
    reference arm needs no GPU, rank 0 prints the line with n_gpus = 2."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--workload", "c1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, env=env, timeout=540)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def _gpu_worker(rank, world, port, q):
    """One rank of the strong split, computed by the DEVICE engine (both ranks
    share cuda:0 here: the pool hands out one GPU), gathered over gloo."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = sweep.strong_shard(config.c4_sweep(64, seed=42), rank, world)
        b = engine.Batch([engine.SimSpec.from_scenario(s) for s in mine], device=0, verify=False)
        b.run()
        recs = sweep.records(b.results_raw())
        b.close()
        q.put((rank, sweep.gather_records(recs, dist).tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_gloo_world2_device_engine_shards_match_one_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    b = engine.Batch([engine.SimSpec.from_scenario(s) for s in config.c4_sweep(64, seed=42)],
                     verify=False)
    b.run()
    serial = sweep.records(b.results_raw())
    b.close()
    assert got[0] == serial and got[1] == serial


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_bench_multi_rank_path_on_one_gpu():
    """`bench.py --gpus 2` end to end through the device engine — re-exec
    under torchrun, per-rank shards, barriers, max-over-ranks timing, the
    record all_gather — with the gloo backend so both ranks can share the one
    GPU this suite runs on (KVG_DIST_BACKEND; NCCL needs a GPU per rank)."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env["KVG_DIST_BACKEND"] = "gloo"
    for split in ("weak", "strong"):
        r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2",
                            "--split", split, "--sims", "256", "--steps", "1", "--warmup", "3",
                            "--no-probe-mode", "--no-cpu-baseline", "--e2e-steps", "1"],
                           capture_output=True, text=True, env=env, timeout=540)
        assert r.returncode == 0, r.stderr[-2000:]
        lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
        assert len(lines) == 1 and lines[0]["n_gpus"] == 2
        d = lines[0]
        assert d["scaling"] == split and d["value"] > 0 and d["parity"]["bad_status"] == 0
        assert d["parity"]["sims"] == (512 if split == "weak" else 256)
