"""Quick device-time probe of the engine on the BASELINE shapes (dev tool)."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import config, engine  # noqa: E402


def run(name, specs, reps=3, **kw):
    t0 = time.perf_counter()
    b = engine.Batch(specs, **kw)
    t1 = time.perf_counter()
    b.run()
    ms = []
    for _ in range(reps):
        b.run()
        ms.append(b.last_ms())
    rs = b.results_raw()
    steps = sum(r.agent_steps for r in rs)
    look = sum(r.lookups for r in rs)
    ev = sum(r.events for r in rs)
    best = min(ms)
    cyc = sorted(r.device_cycles for r in rs)
    if len(cyc) > 1:
        print(f"  per-sim device ms @1.965GHz: p50={cyc[len(cyc)//2]/1.965e6:.1f} "
              f"p90={cyc[int(len(cyc)*0.9)]/1.965e6:.1f} max={cyc[-1]/1.965e6:.1f}")
    print(f"{name}: sims={len(specs)} create={1e3*(t1-t0):.1f}ms run={best:.2f}ms "
          f"agent_steps/s={steps/best*1e3:.3e} lookups/s={look/best*1e3:.3e} "
          f"events={ev} evict_calls={sum(r.evict_calls for r in rs)} "
          f"makespan0={rs[0].makespan:.6g}", flush=True)
    b.close()


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c4", "c2"]
    if "c1" in which:
        for p in ("aimd", "uncontrolled"):
            s = config.c1_toy(p)
            run(f"c1_{p}", [engine.SimSpec.from_scenario(s)])
    if "c4" in which:
        pop = engine.Population(config.c1_toy().workload, 42)
        specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]
        run("c4", specs)
    if "c2" in which:
        s = config.c2_qwen("aimd")
        for w in (8, 32):
            run(f"c2_aimd_w{w}", [engine.SimSpec.from_scenario(s)], reps=1, warps_per_sim=w)
