"""dev probe: C4 kernel time with / without streamed host delivery."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2601_22705_b200 import config, engine
pop = engine.Population(config.c1_toy().workload, 42)
specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]
for ho in (False, True, False, True):
    b = engine.Batch(specs, verify=False, host_outputs=ho)
    b.run()
    ks, ws = [], []
    for _ in range(3):
        t = time.perf_counter(); b.run(); w = time.perf_counter() - t
        a, k = b.timing(); ks.append(k); ws.append(w * 1e3)
    print("host_outputs", ho, "kernel ms", [round(x, 2) for x in ks], "wall ms", [round(x, 2) for x in ws], flush=True)
    b.close()
