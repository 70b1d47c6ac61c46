"""One engine launch for ncu capture: python tools/profile_run.py c4 [n_sims]."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import config, engine  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if which == "c4":
    pop = engine.Population(config.c1_toy().workload, 42)
    specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep(n)]
elif which == "c2":
    specs = [engine.SimSpec.from_scenario(config.c2_qwen("aimd"))]
else:
    specs = [engine.SimSpec.from_scenario(config.c1_toy(which))]
b = engine.Batch(specs, trace_capacity=4096)
for _ in range(reps):
    b.run()
    print(which, n, b.timing(), flush=True)
