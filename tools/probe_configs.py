"""Dev probe: device time of each BASELINE config at full size (one sim each)."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import config, engine  # noqa: E402


def go(name, s, pol=None, warps=0):
    t0 = time.perf_counter()
    spec = engine.SimSpec.from_scenario(s, pol)
    b = engine.Batch([spec], warps_per_sim=warps)
    t1 = time.perf_counter()
    st = b.run()
    r = b.result(0)
    print(f"{name}: status={st} create={t1-t0:.2f}s run_ms={b.timing()[1]:.1f} makespan={r['makespan']:.6g} "
          f"events={r['events']} agent_steps={r['agent_steps']} lookups={r['lookups']} "
          f"evict_calls={r['evict_calls']} stalls={r['stall_events']} offl={r['offloaded_tokens']} "
          f"rel={r['reloaded_tokens']} wall={time.perf_counter()-t1:.1f}s", flush=True)
    b.close()


which = sys.argv[1:]
for w in which:
    if w == "c2":
        go("c2_aimd", config.c2_qwen("aimd"))
    elif w == "c2u":
        go("c2_uncontrolled", config.c2_qwen("uncontrolled"))
    elif w.startswith("c3"):
        pol = w[3:] or "aimd"
        s = config.c3_dsv3("offload" if pol == "offload" else ("aimd" if pol == "h03" else pol))
        if pol == "h03":
            s.controller.h_thresh = 0.3
        go(f"c3_{pol}", s)
    elif w.startswith("c5"):
        pol = w[3:] or "aimd"
        go(f"c5_{pol}", config.c5_stress(pol if pol else "aimd"))
