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
