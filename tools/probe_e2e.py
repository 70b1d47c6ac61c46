"""Dev probe: e2e phase breakdown and per-sim device-time distribution (C4)."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402

from paper_2601_22705_b200 import config, engine  # noqa: E402

pop = engine.Population(config.c1_toy().workload, 42)
scen = config.c4_sweep()
t0 = time.perf_counter()
specs = [engine.SimSpec.from_scenario(s, population=pop) for s in scen]
t1 = time.perf_counter()
print(f"specs: {1e3*(t1-t0):.1f} ms")
for rep in range(3):
    t0 = time.perf_counter()
    b = engine.Batch(specs, host_outputs=True)
    t1 = time.perf_counter()
    b.run()
    t2 = time.perf_counter()
    rs = b.results_raw()
    t3 = time.perf_counter()
    b.close()
    t4 = time.perf_counter()
    print(f"e2e rep{rep}: create={1e3*(t1-t0):.1f} run={1e3*(t2-t1):.1f} "
          f"results={1e3*(t3-t2):.1f} close={1e3*(t4-t3):.1f} timing={b.timing() if b.h else ''}")
b = engine.Batch(specs)
for _ in range(3):
    b.run()
print("device step/kernel ms:", b.timing())
rs = b.results_raw()
cyc = np.array([r.device_cycles for r in rs], dtype=np.float64) / 1.965e6
ev = np.array([r.events for r in rs])
evc = np.array([r.evict_calls for r in rs])
evs = np.array([r.evict_scanned for r in rs])
evp = np.array([r.evicted_pages for r in rs])
tk = np.array([r.ticks for r in rs])
look = np.array([r.lookups for r in rs])
print("per-sim ms quantiles (0,10,50,90,99,100):", np.percentile(cyc, [0, 10, 50, 90, 99, 100]).round(2))
order = np.argsort(cyc)
for name, arr in [("events", ev), ("evict_calls", evc), ("evict_scanned", evs),
                  ("evicted_pages", evp), ("ticks", tk), ("lookups", look)]:
    print(f"{name}: mean={arr.mean():.1f} slowest10%={arr[order[-len(arr)//10:]].mean():.1f} "
          f"fastest10%={arr[order[:len(arr)//10]].mean():.1f}")
# correlation of time with components
X = np.stack([ev, evc, evs / 1000, look / 100, np.ones_like(ev)], 1).astype(np.float64)
coef, *_ = np.linalg.lstsq(X, cyc, rcond=None)
print("lstsq ms ~ events, evict_calls, evict_scanned/1e3, lookups/100, 1:", coef)
print("sum cyc ms", cyc.sum(), "kernel ms x 148*24", b.timing()[1] * 148 * 24)
b.close()
