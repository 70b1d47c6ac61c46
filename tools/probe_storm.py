"""dev probe: find C5-shape configs that storm (stalls) quickly."""
import sys, time
sys.path.insert(0, ".")
from paper_2601_22705_b200 import config, engine
for agents, pol, cap, hz in [(8192, "uncontrolled", 1500, 200.0), (8192, "uncontrolled", 4000, 500.0),
                             (16384, "uncontrolled", 3000, 300.0), (8192, "aimd", 3000, 2000.0),
                             (16384, "agent_cap:4096", 20000, 1000.0)]:
    s = config.c5_stress(pol, agents=agents, capacity=cap)
    s.engine.horizon = hz
    b = engine.Batch([engine.SimSpec.from_scenario(s)], verify=False)
    t = time.perf_counter(); b.run(); w = time.perf_counter() - t
    r = b.result(0)
    print(agents, pol, cap, hz, f"{w:.2f}s", "status", r["status"], "steps", r["agent_steps"], "stalls", r["stall_events"], "events", r["events"], flush=True)
    b.close()
