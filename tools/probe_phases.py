"""Dev probe: where a C4 launch spends its cycles (needs a -DKVG_PROFILE build:
KVG_LIB=var_libs/libkvgpu_prof.so python tools/probe_phases.py)."""
import ctypes as C
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import config, engine  # noqa: E402

PH = ["EVENT", "MEMBER", "M_MATCHED", "M_INSERT", "M_EVICTED", "M_COMMIT", "M_CREATED", "M_FAIL",
      "M_RESTORED", "BATCH_END", "GEN_DISCARDED", "GROUP_DONE", "O_MEMBER", "O_RELOAD_CHUNK",
      "O_RELOAD_EVICTED", "O_RELOAD_END", "O_INSERT_START", "O_INSERT_COUNT",
      "O_INSERT_EVICTED", "O_INSERT_FAIL", "O_EVICT_POP", "DONE", "FINAL", "EXITED"]
names = {i: "leader:" + n for i, n in enumerate(PH)}
names.update({32 + k: "coop:" + n for k, n in enumerate(
    ["NONE", "EXIT", "RANGE", "EVICT", "REBUILD", "SCANFREE", "FRONTIER", "TICKS", "PHASES",
     "GROUP", "STORM", "FLUSH"])})
names.update({24: "fast_housekeeping", 25: "member_loop (chain form)", 26: "agent event handler",
              27: "admission_pass", 46: "leader_step entry+sync", 47: "init/finalize"})
which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c4":
    pop = engine.Population(config.c1_toy().workload, 42)
    specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]
elif which == "c2":
    specs = [engine.SimSpec.from_scenario(config.c2_qwen("aimd"))]
elif which == "c5":
    specs = [engine.SimSpec.from_scenario(config.c5_stress("aimd"))]
elif which == "c5h":  # the bench's C5 line: full size to a 5e4 s horizon
    s = config.c5_stress("aimd")
    s.engine.horizon = 5e4
    specs = [engine.SimSpec.from_scenario(s)]
elif which.startswith("c5s"):  # scaled C5 shape: c5s<agents>
    ag = int(which[3:])
    s = config.c5_stress("aimd", agents=ag, capacity=1)
    s.engine.capacity = config.scaled_capacity(engine.Population(s.workload, s.seed).peak_aggregate_tokens)
    specs = [engine.SimSpec.from_scenario(s)]
elif which == "c3off":
    from paper_2601_22705_b200 import sweep
    specs = [engine.SimSpec.from_scenario(s) for s in sweep.weak_shard("c3off", 0, 1)]
elif which == "c3h":
    s = config.c3_dsv3("aimd")
    s.controller.h_thresh = 0.3
    specs = [engine.SimSpec.from_scenario(s)]
else:
    s = config.c3_dsv3("aimd", agents=int(which[3:]) if which[3:] else 2048)
    specs = [engine.SimSpec.from_scenario(s)]
lib = engine.lib()
prof = hasattr(lib, "kvg_debug_profile")  # only in -DKVG_PROFILE builds
b = engine.Batch(specs, verify=False)
buf = (C.c_ulonglong * 48)()
if prof:
    lib.kvg_debug_profile.argtypes = [C.POINTER(C.c_ulonglong)]
    lib.kvg_debug_profile(buf)  # clear
b.run()
if prof:
    lib.kvg_debug_profile(buf)
tot = max(1, sum(buf))
r = b.result(0)
print(which, "kernel ms", b.timing()[1], "total sim-cycles", tot, "events", r["events"], "stalls", r["stall_events"], "evict_calls", r["evict_calls"], "agent_steps", r["agent_steps"], "status", r["status"])
for i in sorted(range(48), key=lambda i: -buf[i]):
    if buf[i]:
        print(f"{100 * buf[i] / tot:6.2f}%  {names.get(i, i)}")
