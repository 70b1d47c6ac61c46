"""Dev probe (KVG_LIB=var_libs/libkvgpu_gt.so, a -DKVG_GTIMER build): where each
C4 simulation sits in wall-clock time inside one launch, its effective SM clock,
and per-SM load."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import config, engine  # noqa: E402

pop = engine.Population(config.c1_toy().workload, 42)
specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]
b = engine.Batch(specs, verify=False)
for _ in range(3):
    b.run()
print("timing", b.timing())
rs = [b.result(i) for i in range(len(specs))]
g0 = np.array([r["abort_time"] for r in rs])
g1 = np.array([r["device_cycles"] for r in rs], dtype=np.float64)
cyc = np.array([r["evict_scanned"] for r in rs], dtype=np.float64)
sm = np.array([r["evicted_pages"] for r in rs])
t0 = g0.min()
s, e = (g0 - t0) / 1e6, (g1 - t0) / 1e6
print("start ms pct", np.percentile(s, [0, 50, 90, 99, 100]))
print("end ms pct", np.percentile(e, [0, 10, 50, 90, 99, 100]))
print("dur ms pct", np.percentile(e - s, [0, 10, 50, 90, 100]))
print("eff MHz pct", np.percentile(cyc / ((g1 - g0) / 1e3), [0, 50, 100]))
cnt = np.bincount(sm, minlength=148)
print("sims per SM min/max", cnt.min(), cnt.max(), "n SMs used", (cnt > 0).sum())
# is the longest simulation on an SM with more residents?
last = np.argsort(-e)[:5]
for i in last:
    print("late sim", i, "sm", sm[i], "residents", cnt[sm[i]], "start", s[i], "end", e[i])
