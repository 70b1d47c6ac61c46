"""dev probe: C4 kernel time of the first run of a fresh batch vs later runs,
with / without streamed host delivery."""
import sys, time
sys.path.insert(0, ".")
from paper_2601_22705_b200 import config, engine
pop = engine.Population(config.c1_toy().workload, 42)
specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]
for ho in (True, False, True):
    for it in range(3):
        t0 = time.perf_counter()
        b = engine.Batch(specs, verify=False, host_outputs=ho)
        t1 = time.perf_counter()
        b.run(); k1 = b.timing()
        t2 = time.perf_counter()
        b.run(); k2 = b.timing()
        t3 = time.perf_counter()
        b.close()
        print(f"host_outputs={ho} it={it} create {1e3*(t1-t0):.2f} ms | run1 wall {1e3*(t2-t1):.2f} step/kernel {k1[0]:.2f}/{k1[1]:.2f} | run2 wall {1e3*(t3-t2):.2f} step/kernel {k2[0]:.2f}/{k2[1]:.2f}", flush=True)
