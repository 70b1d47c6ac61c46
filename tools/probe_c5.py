"""dev probe: C5 stress replicas under short simulated horizons — device time,
events, evict calls, scanned pages (what bounds the full-size run)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2601_22705_b200 import config, engine  # noqa: E402

for pol in sys.argv[1].split(","):
    for hz in [float(x) for x in sys.argv[2].split(",")]:
        s = config.c5_stress(pol)
        s.engine.horizon = hz
        spec = engine.SimSpec.from_scenario(s)
        b = engine.Batch([spec], verify=False)
        t0 = time.perf_counter()
        b.run()
        wall = time.perf_counter() - t0
        r = b.result(0)
        print(f"{pol:16s} horizon={hz:8.0f} status={r['status']} wall={wall:7.2f}s dev={b.last_ms():9.1f}ms "
              f"steps={r['agent_steps']} events={r['events']} evicts={r['evict_calls']} "
              f"evicted={r['evicted_pages']} scanned={r['evict_scanned']} stalls={r['stall_events']} "
              f"ticks={r['ticks']} used={r['pool_used']}", flush=True)
        b.close()
