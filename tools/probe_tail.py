"""Dev probe: per-simulation device cycles and events of one C4 launch (is the
kernel bound by the longest simulations' chains or by the average?)."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import config, engine  # noqa: E402

pop = engine.Population(config.c1_toy().workload, 42)
specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]
b = engine.Batch(specs, verify=False)
for _ in range(3):
    b.run()
print("kernel ms", b.timing())
rs = [b.result(i) for i in range(len(specs))]
cyc = np.array([r["device_cycles"] for r in rs], dtype=np.float64)
ev = np.array([r["events"] for r in rs], dtype=np.float64)
ae = np.array([r["agent_events"] for r in rs], dtype=np.float64)
st = np.array([r["stall_events"] for r in rs], dtype=np.float64)
tk = np.array([r["ticks"] for r in rs], dtype=np.float64)
for name, a in [("cycles", cyc), ("events", ev), ("agent_events", ae), ("stalls", st), ("ticks", tk),
                ("cyc/event", cyc / np.maximum(ev, 1))]:
    q = np.percentile(a, [0, 10, 50, 90, 99, 100])
    print(f"{name:14s} " + " ".join(f"{x:12.1f}" for x in q) + f"  mean {a.mean():.1f}")
print("corr(cycles, events)", np.corrcoef(cyc, ev)[0, 1])
order = np.argsort(-cyc)[:10]
for i in order:
    print(i, specs[i].name if hasattr(specs[i], "name") else "", cyc[i], ev[i], st[i], tk[i])
# by sweep axis (k % 8 = u_low etc.)
for m in (8, 64):
    g = [cyc[np.arange(len(cyc)) % m == k].mean() for k in range(m)]
    print(f"mean cycles by k%{m}:", " ".join(f"{x/1e6:.1f}" for x in g[:16]))
