"""Dev probe: e2e step phases as bench.py runs them."""
import ctypes as C
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import abi, config, engine  # noqa: E402

pop = engine.Population(config.c1_toy().workload, 42)
specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]
main = engine.Batch(specs)
main.run()
main.close()
for rep in range(4):
    t = [time.perf_counter()]
    b = engine.Batch(specs, host_outputs=True); t.append(time.perf_counter())
    b.run(); t.append(time.perf_counter())
    r = b.results_array(); t.append(time.perf_counter())
    x = int(r["ticks"].sum()); t.append(time.perf_counter())
    b.close(); t.append(time.perf_counter())
    d = [1e3 * (t[i + 1] - t[i]) for i in range(len(t) - 1)]
    print("create %.1f run %.1f results %.1f sum %.1f close %.1f" % tuple(d), flush=True)
